// Load-balancing plan of the f32 n-row operator pass (ancka_row_split): row
// cost = structural + KNN nonzeros; rows by descending cost (stable, the
// order the fused narrow-block kernel deals rows to its lane groups); "long"
// rows (cost > thr, KNN or graph hubs), which the SpMM gives a whole warp.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include "common.cuh"

namespace ancka {

__global__ void plan_cost_kernel(const int64_t* __restrict__ srp, const int64_t* __restrict__ krp,
                                 int64_t n, double thr, uint32_t* __restrict__ cost,
                                 int32_t* __restrict__ iota, uint8_t* __restrict__ is_long) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = (srp[i + 1] - srp[i]) + (krp[i + 1] - krp[i]);
    cost[i] = (uint32_t)c;
    iota[i] = (int32_t)i;
    is_long[i] = (double)c > thr ? 1 : 0;
  }
}

struct PlanScratch {
  size_t sort_bytes, select_bytes;
};

static PlanScratch plan_scratch(int64_t n) {
  PlanScratch s{0, 0};
  const int m = (int)std::max<int64_t>(n, 1);
  cub::DeviceRadixSort::SortPairsDescending(nullptr, s.sort_bytes, (const uint32_t*)nullptr,
                                            (uint32_t*)nullptr, (const int32_t*)nullptr,
                                            (int32_t*)nullptr, m);
  cub::DeviceSelect::Flagged(nullptr, s.select_bytes, (const int32_t*)nullptr,
                             (const uint8_t*)nullptr, (int32_t*)nullptr, (int64_t*)nullptr, m);
  return s;
}

}  // namespace ancka

using namespace ancka;

extern "C" size_t ancka_row_split_workspace_size(int64_t n) {
  const PlanScratch s = plan_scratch(n);
  Carver cv(nullptr, 0);
  cv.take<uint32_t>(n);                         // cost
  cv.take<uint32_t>(n);                         // sorted cost (discarded)
  cv.take<int32_t>(n);                          // iota
  cv.take<unsigned char>(std::max(s.sort_bytes, s.select_bytes));
  return cv.used;
}

extern "C" int ancka_row_split_plan(const int64_t* srp, const int64_t* krp, int64_t n, double thr,
                                    int32_t* order_out, uint8_t* is_long_out,
                                    int32_t* long_rows_out, int64_t* n_long_out, void* workspace,
                                    size_t workspace_bytes, ancka_stream_t stream) {
  ANCKA_REQUIRE(n >= 1 && n < (int64_t)INT32_MAX, ANCKA_ERR_ARG, "row_split_plan: bad size n=%lld",
                (long long)n);
  const PlanScratch s = plan_scratch(n);
  Carver cv(workspace, workspace_bytes);
  uint32_t* cost = cv.take<uint32_t>(n);
  uint32_t* cost_sorted = cv.take<uint32_t>(n);
  int32_t* iota = cv.take<int32_t>(n);
  const size_t tb = std::max(s.sort_bytes, s.select_bytes);
  void* tmp = cv.take<unsigned char>(tb);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "row_split_plan: workspace too small");
  auto st = as_stream(stream);
  const int grid = (int)std::min<int64_t>(ceil_div(n, 256), 4 * kNumSMs);
  plan_cost_kernel<<<grid, 256, 0, st>>>(srp, krp, n, thr, cost, iota, is_long_out);
  ANCKA_LAUNCHED();
  // stable descending order of cost (ties keep ascending row index)
  size_t b = tb;
  ANCKA_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp, b, cost, cost_sorted, iota, order_out,
                                                       (int)n, 0, 32, st));
  b = tb;   // long rows in ascending order, their count -> *n_long_out
  ANCKA_CUDA(cub::DeviceSelect::Flagged(tmp, b, iota, is_long_out, long_rows_out, n_long_out,
                                        (int)n, st));
  return ANCKA_OK;
}
