// KNN-graph assembly (K2): A_K = M + M^T and P_K = D_K^-1 A_K from the padded
// neighbour lists (knn.py:294-324).  Both directions of every selected pair
// are emitted as 64-bit (row, col) keys, radix-sorted, and equal keys (a
// mutual pair) are summed -- exactly scipy's csr + csr for two addends.  Row
// sums replicate numpy's pairwise reduction so P_K in f64 is bit-identical
// to the reference's for the same lists.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>

#include "common.cuh"

namespace ancka {

__global__ void knn_emit_kernel(const int32_t* __restrict__ ids, const double* __restrict__ scores,
                                int64_t n, int K, uint64_t* __restrict__ keys,
                                double* __restrict__ vals) {
  const int64_t total = n * K;
  const uint64_t sentinel = (uint64_t)n << 32;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < total;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = p / K;
    const int32_t j = ids[p];
    if (j >= 0) {
      const double s = scores[p];
      keys[2 * p] = ((uint64_t)i << 32) | (uint32_t)j;
      keys[2 * p + 1] = ((uint64_t)j << 32) | (uint32_t)i;
      vals[2 * p] = s;
      vals[2 * p + 1] = s;
    } else {
      keys[2 * p] = keys[2 * p + 1] = sentinel;
      vals[2 * p] = vals[2 * p + 1] = 0.0;
    }
  }
}

struct SumOp {
  __device__ __forceinline__ double operator()(double a, double b) const { return __dadd_rn(a, b); }
};

__global__ void knn_rowptr_kernel(const uint64_t* __restrict__ ukeys, const int64_t* __restrict__ nruns,
                                  int64_t n, int64_t* __restrict__ rowptr, int64_t* __restrict__ nnz_out) {
  // the last run may be the sentinel row n
  int64_t runs = *nruns;
  int64_t nnz = runs;
  if (runs > 0 && (ukeys[runs - 1] >> 32) >= (uint64_t)n) nnz = runs - 1;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t target = (uint64_t)r << 32;
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (ukeys[mid] < target) lo = mid + 1; else hi = mid;
    }
    rowptr[r] = lo;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *nnz_out = nnz;
}

__global__ void knn_finish_kernel(const uint64_t* __restrict__ ukeys, const double* __restrict__ agg,
                                  const int64_t* __restrict__ rowptr, int64_t n,
                                  int32_t* __restrict__ colidx, double* __restrict__ a_k,
                                  double* __restrict__ p64, float* __restrict__ p32,
                                  uint8_t* __restrict__ zero_rows) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = rowptr[r], e = rowptr[r + 1];
    for (int64_t p = b; p < e; ++p) {
      colidx[p] = (int32_t)(ukeys[p] & 0xffffffffu);
      a_k[p] = agg[p];
    }
    double rs = 0.0;
    if (e > b) rs = __dadd_rn(agg[b], np_pairwise_sum(agg + b + 1, e - b - 1));
    zero_rows[r] = rs == 0.0;
    const double inv = rs != 0.0 ? 1.0 / rs : 0.0;
    for (int64_t p = b; p < e; ++p) {
      const double v = __dmul_rn(inv, agg[p]);
      p64[p] = v;
      p32[p] = (float)v;
    }
  }
}

__global__ void knn_coo_keys_kernel(const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                                    const double* __restrict__ vals, int64_t E,
                                    uint64_t* __restrict__ keys, double* __restrict__ kv) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < E;
       p += (int64_t)gridDim.x * blockDim.x) {
    keys[p] = ((uint64_t)(uint32_t)rows[p] << 32) | (uint32_t)cols[p];
    kv[p] = vals[p];
  }
}

// thread per row: two (score desc, id asc) lists -> first K of the union
__global__ void knn_merge_lists_kernel(int32_t* __restrict__ ia, double* __restrict__ sa,
                                       const int32_t* __restrict__ ib, const double* __restrict__ sb,
                                       int64_t nq, int K) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nq;
       r += (int64_t)gridDim.x * blockDim.x) {
    int32_t oi[32];
    double os[32];
    const int32_t* A = ia + r * K;
    const double* As = sa + r * K;
    const int32_t* B = ib + r * K;
    const double* Bs = sb + r * K;
    int pa = 0, pb = 0, m = 0;
    while (m < K) {
      const bool va = pa < K && A[pa] >= 0, vb = pb < K && B[pb] >= 0;
      if (!va && !vb) break;
      bool takeA;
      if (!vb) takeA = true;
      else if (!va) takeA = false;
      else takeA = As[pa] > Bs[pb] || (As[pa] == Bs[pb] && A[pa] < B[pb]);
      const int32_t id = takeA ? A[pa] : B[pb];
      const double sc = takeA ? As[pa] : Bs[pb];
      if (takeA) ++pa; else ++pb;
      bool dup = false;
      for (int q = 0; q < m; ++q) dup |= oi[q] == id;
      if (dup) continue;
      oi[m] = id;
      os[m] = sc;
      ++m;
    }
    for (int q = 0; q < K; ++q) {
      ia[r * K + q] = q < m ? oi[q] : -1;
      sa[r * K + q] = q < m ? os[q] : 0.0;
    }
  }
}

struct GraphWs {
  uint64_t *k0, *k1, *ukeys;
  double *v0, *v1, *agg;
  int64_t* nruns;
  void* cub_tmp;
  size_t cub_bytes;
};

static int bits_for(int64_t n) {
  int b = 1;
  while (((int64_t)1 << b) <= n) ++b;
  return b;
}

static int carve_graph(Carver& cv, GraphWs& w, int64_t n, int K) {
  const int64_t E = 2 * n * (int64_t)K;
  w.k0 = cv.take<uint64_t>(E);
  w.k1 = cv.take<uint64_t>(E);
  w.ukeys = cv.take<uint64_t>(E);
  w.v0 = cv.take<double>(E);
  w.v1 = cv.take<double>(E);
  w.agg = cv.take<double>(E);
  w.nruns = cv.take<int64_t>(1);
  size_t sort_bytes = 0, red_bytes = 0;
  cub::DoubleBuffer<uint64_t> kb(nullptr, nullptr);
  cub::DoubleBuffer<double> vb(nullptr, nullptr);
  if (cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, kb, vb, E, 0, 32 + bits_for(n)) !=
      cudaSuccess)
    return ANCKA_ERR_CUDA;
  if (cub::DeviceReduce::ReduceByKey(nullptr, red_bytes, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                     (double*)nullptr, (double*)nullptr, (int64_t*)nullptr, SumOp(),
                                     E) != cudaSuccess)
    return ANCKA_ERR_CUDA;
  w.cub_bytes = std::max(sort_bytes, red_bytes);
  w.cub_tmp = cv.take<char>(w.cub_bytes);
  return ANCKA_OK;
}

}  // namespace ancka

using namespace ancka;

extern "C" size_t ancka_knn_graph_workspace_size(int64_t n, int32_t K) {
  Carver cv(nullptr, 0);
  GraphWs w;
  if (carve_graph(cv, w, n, K) != ANCKA_OK) return 0;
  return cv.used;
}

extern "C" int ancka_knn_graph(const int32_t* ids, const double* scores, int64_t n, int32_t K,
                               int64_t* rowptr, int32_t* colidx, double* a_k, double* p_k64,
                               float* p_k32, uint8_t* zero_rows, int64_t* nnz_out,
                               void* workspace, size_t workspace_bytes, ancka_stream_t stream) {
  ANCKA_REQUIRE(n >= 1 && K >= 1, ANCKA_ERR_ARG, "knn_graph: bad sizes");
  ANCKA_REQUIRE(n < (1ll << 31), ANCKA_ERR_UNSUPPORTED, "knn_graph: n must fit int32 column ids");
  Carver cv(workspace, workspace_bytes);
  GraphWs w;
  ANCKA_TRY(carve_graph(cv, w, n, K));
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "knn_graph: workspace too small");
  auto st = as_stream(stream);
  const int64_t E = 2 * n * (int64_t)K;
  const int g = (int)std::min<int64_t>(ceil_div(n * K, 256), 16 * kNumSMs);
  knn_emit_kernel<<<std::max(g, 1), 256, 0, st>>>(ids, scores, n, K, w.k0, w.v0);
  ANCKA_LAUNCHED();
  cub::DoubleBuffer<uint64_t> kb(w.k0, w.k1);
  cub::DoubleBuffer<double> vb(w.v0, w.v1);
  size_t bytes = w.cub_bytes;
  ANCKA_CUDA(cub::DeviceRadixSort::SortPairs(w.cub_tmp, bytes, kb, vb, E, 0, 32 + bits_for(n), st));
  bytes = w.cub_bytes;
  ANCKA_CUDA(cub::DeviceReduce::ReduceByKey(w.cub_tmp, bytes, kb.Current(), w.ukeys, vb.Current(),
                                            w.agg, w.nruns, SumOp(), E, st));
  const int gr = (int)std::min<int64_t>(ceil_div(n + 1, 256), 16 * kNumSMs);
  knn_rowptr_kernel<<<std::max(gr, 1), 256, 0, st>>>(w.ukeys, w.nruns, n, rowptr, nnz_out);
  ANCKA_LAUNCHED();
  knn_finish_kernel<<<std::max(gr, 1), 256, 0, st>>>(w.ukeys, w.agg, rowptr, n, colidx, a_k,
                                                     p_k64, p_k32, zero_rows);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

extern "C" int ancka_knn_merge_lists(int32_t* ids_a, double* scores_a, const int32_t* ids_b,
                                     const double* scores_b, int64_t nq, int32_t K,
                                     ancka_stream_t stream) {
  ANCKA_REQUIRE(K >= 1 && K <= 32, ANCKA_ERR_UNSUPPORTED, "merge_lists: K must be in [1, 32]");
  if (nq <= 0) return ANCKA_OK;
  const int g = (int)std::min<int64_t>(ceil_div(nq, 128), 16 * kNumSMs);
  knn_merge_lists_kernel<<<g, 128, 0, as_stream(stream)>>>(ids_a, scores_a, ids_b, scores_b, nq, K);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

static int carve_graph_coo(Carver& cv, GraphWs& w, int64_t E, int64_t nrows) {
  w.k0 = cv.take<uint64_t>(E);
  w.k1 = cv.take<uint64_t>(E);
  w.ukeys = cv.take<uint64_t>(E);
  w.v0 = cv.take<double>(E);
  w.v1 = cv.take<double>(E);
  w.agg = cv.take<double>(E);
  w.nruns = cv.take<int64_t>(1);
  size_t sort_bytes = 0, red_bytes = 0;
  cub::DoubleBuffer<uint64_t> kb(nullptr, nullptr);
  cub::DoubleBuffer<double> vb(nullptr, nullptr);
  if (cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, kb, vb, E, 0, 32 + bits_for(nrows)) !=
      cudaSuccess)
    return ANCKA_ERR_CUDA;
  if (cub::DeviceReduce::ReduceByKey(nullptr, red_bytes, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                     (double*)nullptr, (double*)nullptr, (int64_t*)nullptr, SumOp(),
                                     E) != cudaSuccess)
    return ANCKA_ERR_CUDA;
  w.cub_bytes = std::max(sort_bytes, red_bytes);
  w.cub_tmp = cv.take<char>(w.cub_bytes);
  return ANCKA_OK;
}

extern "C" size_t ancka_knn_graph_coo_workspace_size(int64_t E) {
  Carver cv(nullptr, 0);
  GraphWs w;
  if (carve_graph_coo(cv, w, std::max<int64_t>(E, 1), 1ll << 31) != ANCKA_OK) return 0;
  return cv.used;
}

extern "C" int ancka_knn_graph_coo(const int32_t* rows, const int32_t* cols, const double* vals,
                                   int64_t E, int64_t nrows, int64_t ncols, int64_t* rowptr,
                                   int32_t* colidx, double* a_k, double* p_k64, float* p_k32,
                                   uint8_t* zero_rows, int64_t* nnz_out, void* workspace,
                                   size_t workspace_bytes, ancka_stream_t stream) {
  ANCKA_REQUIRE(nrows >= 1 && E >= 0, ANCKA_ERR_ARG, "knn_graph_coo: bad sizes");
  ANCKA_REQUIRE(ncols < (1ll << 31) && nrows < (1ll << 31), ANCKA_ERR_UNSUPPORTED,
                "knn_graph_coo: ids must fit int32");
  auto st = as_stream(stream);
  const int gr = (int)std::min<int64_t>(ceil_div(nrows + 1, 256), 16 * kNumSMs);
  if (E == 0) {
    ANCKA_CUDA(cudaMemsetAsync(rowptr, 0, sizeof(int64_t) * (nrows + 1), st));
    ANCKA_CUDA(cudaMemsetAsync(zero_rows, 1, nrows, st));
    ANCKA_CUDA(cudaMemsetAsync(nnz_out, 0, sizeof(int64_t), st));
    return ANCKA_OK;
  }
  Carver cv(workspace, workspace_bytes);
  GraphWs w;
  ANCKA_TRY(carve_graph_coo(cv, w, E, 1ll << 31));
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "knn_graph_coo: workspace too small");
  const int g = (int)std::min<int64_t>(ceil_div(E, 256), 16 * kNumSMs);
  knn_coo_keys_kernel<<<std::max(g, 1), 256, 0, st>>>(rows, cols, vals, E, w.k0, w.v0);
  ANCKA_LAUNCHED();
  cub::DoubleBuffer<uint64_t> kb(w.k0, w.k1);
  cub::DoubleBuffer<double> vb(w.v0, w.v1);
  size_t bytes = w.cub_bytes;
  ANCKA_CUDA(cub::DeviceRadixSort::SortPairs(w.cub_tmp, bytes, kb, vb, E, 0, 32 + bits_for(nrows), st));
  bytes = w.cub_bytes;
  ANCKA_CUDA(cub::DeviceReduce::ReduceByKey(w.cub_tmp, bytes, kb.Current(), w.ukeys, vb.Current(),
                                            w.agg, w.nruns, SumOp(), E, st));
  knn_rowptr_kernel<<<std::max(gr, 1), 256, 0, st>>>(w.ukeys, w.nruns, nrows, rowptr, nnz_out);
  ANCKA_LAUNCHED();
  knn_finish_kernel<<<std::max(gr, 1), 256, 0, st>>>(w.ukeys, w.agg, rowptr, nrows, colidx, a_k,
                                                     p_k64, p_k32, zero_rows);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}
