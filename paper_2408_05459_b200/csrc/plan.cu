// Load-balancing plan of the f32 n-row operator pass (ancka_row_split): row
// cost = structural + KNN nonzeros; rows by descending cost (stable, the
// order the fused narrow-block kernel deals rows to its lane groups); "long"
// rows (cost > thr, KNN or graph hubs) cut into pieces of at most `piece`
// nonzeros of one segment (structural pieces first).  Two calls around one
// read-back of (n_long, n_pieces), which size the caller's piece arrays.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include "common.cuh"

namespace ancka {

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void plan_cost_kernel(const int64_t* __restrict__ srp, const int64_t* __restrict__ krp,
                                 int64_t n, double thr, int piece, uint32_t* __restrict__ cost,
                                 int32_t* __restrict__ iota, uint8_t* __restrict__ is_long,
                                 unsigned long long* __restrict__ counts) {
  unsigned long long pieces = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ls = srp[i + 1] - srp[i], lk = krp[i + 1] - krp[i];
    const int64_t c = ls + lk;
    cost[i] = (uint32_t)c;
    iota[i] = (int32_t)i;
    const bool lg = (double)c > thr;
    is_long[i] = lg ? 1 : 0;
    if (lg) pieces += (unsigned long long)((ls + piece - 1) / piece + (lk + piece - 1) / piece);
  }
  pieces = warp_sum_u64(pieces);
  if ((threadIdx.x & 31) == 0 && pieces) atomicAdd(counts + 1, pieces);   // integer: order-free
}

__global__ void plan_per_row_kernel(const int64_t* __restrict__ srp, const int64_t* __restrict__ krp,
                                    const int32_t* __restrict__ long_rows, int64_t n_long, int piece,
                                    int64_t* __restrict__ per) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_long;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = long_rows[j];
    per[j] = (srp[r + 1] - srp[r] + piece - 1) / piece + (krp[r + 1] - krp[r] + piece - 1) / piece;
  }
}

__global__ void plan_fill_kernel(const int64_t* __restrict__ srp, const int64_t* __restrict__ krp,
                                 const int32_t* __restrict__ long_rows, int64_t n_long, int piece,
                                 const int64_t* __restrict__ ptr, int32_t* __restrict__ seg,
                                 int64_t* __restrict__ begin, int64_t* __restrict__ end) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_long;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = long_rows[j];
    int64_t q = ptr[j];
    for (int s = 0; s < 2; ++s) {
      const int64_t b = s == 0 ? srp[r] : krp[r], e = s == 0 ? srp[r + 1] : krp[r + 1];
      for (int64_t p = b; p < e; p += piece, ++q) {
        seg[q] = s;
        begin[q] = p;
        end[q] = p + piece < e ? p + piece : e;
      }
    }
  }
}

struct PlanScratch {
  size_t sort_bytes, select_bytes, scan_bytes;
};

static PlanScratch plan_scratch(int64_t n) {
  PlanScratch s{0, 0, 0};
  const int m = (int)std::max<int64_t>(n, 1);
  cub::DeviceRadixSort::SortPairsDescending(nullptr, s.sort_bytes, (const uint32_t*)nullptr,
                                            (uint32_t*)nullptr, (const int32_t*)nullptr,
                                            (int32_t*)nullptr, m);
  cub::DeviceSelect::Flagged(nullptr, s.select_bytes, (const int32_t*)nullptr,
                             (const uint8_t*)nullptr, (int32_t*)nullptr, (int64_t*)nullptr, m);
  cub::DeviceScan::InclusiveSum(nullptr, s.scan_bytes, (const int64_t*)nullptr, (int64_t*)nullptr, m);
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
  cv.take<int64_t>(n);                          // per-long-row piece counts
  cv.take<unsigned char>(std::max(s.sort_bytes, std::max(s.select_bytes, s.scan_bytes)));
  return cv.used;
}

extern "C" int ancka_row_split_plan(const int64_t* srp, const int64_t* krp, int64_t n, double thr,
                                    int32_t piece, int32_t* order_out, uint8_t* is_long_out,
                                    int32_t* long_rows_out, int64_t* counts_out, void* workspace,
                                    size_t workspace_bytes, ancka_stream_t stream) {
  ANCKA_REQUIRE(n >= 1 && piece >= 1 && n < (int64_t)INT32_MAX, ANCKA_ERR_ARG,
                "row_split_plan: bad sizes (n=%lld, piece=%d)", (long long)n, piece);
  const PlanScratch s = plan_scratch(n);
  Carver cv(workspace, workspace_bytes);
  uint32_t* cost = cv.take<uint32_t>(n);
  uint32_t* cost_sorted = cv.take<uint32_t>(n);
  int32_t* iota = cv.take<int32_t>(n);
  cv.take<int64_t>(n);
  size_t tb = std::max(s.sort_bytes, std::max(s.select_bytes, s.scan_bytes));
  void* tmp = cv.take<unsigned char>(tb);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "row_split_plan: workspace too small");
  auto st = as_stream(stream);
  ANCKA_CUDA(cudaMemsetAsync(counts_out, 0, 2 * sizeof(int64_t), st));
  const int grid = (int)std::min<int64_t>(ceil_div(n, 256), 4 * kNumSMs);
  plan_cost_kernel<<<grid, 256, 0, st>>>(srp, krp, n, thr, piece, cost, iota, is_long_out,
                                         reinterpret_cast<unsigned long long*>(counts_out));
  ANCKA_LAUNCHED();
  // stable descending order of cost (ties keep ascending row index)
  size_t b = tb;
  ANCKA_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp, b, cost, cost_sorted, iota, order_out,
                                                       (int)n, 0, 32, st));
  b = tb;   // long rows in ascending order; their count -> counts_out[0]
  ANCKA_CUDA(cub::DeviceSelect::Flagged(tmp, b, iota, is_long_out, long_rows_out, counts_out,
                                        (int)n, st));
  return ANCKA_OK;
}

extern "C" int ancka_row_split_pieces(const int64_t* srp, const int64_t* krp,
                                      const int32_t* long_rows, int64_t n, int64_t n_long,
                                      int32_t piece, int64_t* piece_ptr, int32_t* piece_seg,
                                      int64_t* piece_begin, int64_t* piece_end, void* workspace,
                                      size_t workspace_bytes, ancka_stream_t stream) {
  ANCKA_REQUIRE(n_long >= 1 && n_long <= n && piece >= 1, ANCKA_ERR_ARG,
                "row_split_pieces: bad sizes (n_long=%lld)", (long long)n_long);
  const PlanScratch s = plan_scratch(n);
  Carver cv(workspace, workspace_bytes);
  cv.take<uint32_t>(n);
  cv.take<uint32_t>(n);
  cv.take<int32_t>(n);
  int64_t* per = cv.take<int64_t>(n);
  size_t tb = std::max(s.sort_bytes, std::max(s.select_bytes, s.scan_bytes));
  void* tmp = cv.take<unsigned char>(tb);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "row_split_pieces: workspace too small");
  auto st = as_stream(stream);
  const int grid = (int)std::min<int64_t>(ceil_div(n_long, 256), 4 * kNumSMs);
  plan_per_row_kernel<<<grid, 256, 0, st>>>(srp, krp, long_rows, n_long, piece, per);
  ANCKA_LAUNCHED();
  ANCKA_CUDA(cudaMemsetAsync(piece_ptr, 0, sizeof(int64_t), st));
  size_t b = tb;
  ANCKA_CUDA(cub::DeviceScan::InclusiveSum(tmp, b, per, piece_ptr + 1, (int)n_long, st));
  plan_fill_kernel<<<grid, 256, 0, st>>>(srp, krp, long_rows, n_long, piece, piece_ptr, piece_seg,
                                         piece_begin, piece_end);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}
