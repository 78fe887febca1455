// Exact cosine KNN on CUDA cores in f64 (general real-valued attributes).
// knn.py:54-65 (row normalisation) and knn.py:83-140 (blocked scan + ordered
// top-K).  Query-stationary: a CTA owns 64 query rows and streams every key
// tile of 64 rows; the 64 x 64 similarity tile lives only in shared memory and
// each query row's running top-K list is owned by one thread, updated in
// ascending key order so (value desc, index asc) needs only a strict compare.
// The n x n similarity matrix never reaches HBM.
#include "common.cuh"
#include "knn.cuh"

namespace ancka {

constexpr int BM = 64, BN = 64, BK = 16;

// xn = X / ||X||_2 row-wise, zero rows stay zero; norms out.  (knn.py:62-65)
__global__ void normalize_rows_f64_kernel(const double* __restrict__ X, int64_t n, int64_t d,
                                          int64_t ldx, double* __restrict__ xn, int64_t ldn,
                                          double* __restrict__ norms) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nwarps) {
    double s = 0.0;
    for (int64_t c = lane; c < d; c += 32) {
      const double v = X[i * ldx + c];
      s = fma(v, v, s);
    }
    s = warp_sum(s);
    const double nrm = sqrt(s);
    const double inv = nrm > 0 ? 1.0 / nrm : 0.0;
    for (int64_t c = lane; c < ldn; c += 32) xn[i * ldn + c] = c < d ? X[i * ldx + c] * inv : 0.0;
    if (lane == 0) norms[i] = nrm;
  }
}

__global__ void __launch_bounds__(256)
knn_simt_kernel(const double* __restrict__ xn, int64_t n, int64_t ldn, const double* __restrict__ norms,
                int K, int64_t q_begin, int64_t q_end, int32_t* __restrict__ ids,
                double* __restrict__ scores) {
  extern __shared__ __align__(16) unsigned char smraw[];
  double* As = reinterpret_cast<double*>(smraw);           // BM x BK
  double* Bs = As + BM * BK;                                // BN x BK
  double* S = Bs + BN * BK;                                 // BM x (BN+1)
  double* lv = S + BM * (BN + 1);                           // BM x K values
  int32_t* li = reinterpret_cast<int32_t*>(lv + (size_t)BM * K);  // BM x K ids
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;  // 16 x 16 threads, 4 x 4 each
  const int64_t q0 = q_begin + (int64_t)blockIdx.x * BM;
  int fill = 0;                            // list length (owner threads)
  for (int e = tid; e < BM * K; e += blockDim.x) { lv[e] = 0.0; li[e] = -1; }
  const int64_t qi = q0 + tid;
  const bool owner = tid < BM && qi < q_end;
  const bool qzero = owner ? norms[qi] == 0.0 : true;
  __syncthreads();
  for (int64_t k0 = 0; k0 < n; k0 += BN) {
    double acc[4][4] = {};
    for (int64_t d0 = 0; d0 < ldn; d0 += BK) {
      for (int e = tid; e < BM * BK; e += blockDim.x) {
        const int r = e / BK, c = e % BK;
        const int64_t qr = q0 + r, kr = k0 + r;
        As[e] = qr < q_end ? xn[qr * ldn + d0 + c] : 0.0;
        Bs[e] = kr < n ? xn[kr * ldn + d0 + c] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int c = 0; c < BK; ++c) {
        double a[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { a[u] = As[(ty * 4 + u) * BK + c]; b[u] = Bs[(tx * 4 + u) * BK + c]; }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) S[(ty * 4 + u) * (BN + 1) + tx * 4 + v] = acc[u][v];
    __syncthreads();
    if (owner && !qzero) {
      double* myv = lv + (size_t)tid * K;
      int32_t* myi = li + (size_t)tid * K;
      const int jn = (int)lmin(BN, n - k0);
      for (int jj = 0; jj < jn; ++jj) {
        const int64_t j = k0 + jj;
        const double s = S[tid * (BN + 1) + jj];
        if (j == qi || !(s > 0.0)) continue;
        if (fill == K && !(s > myv[K - 1])) continue;
        int pos = fill < K ? fill : K - 1;
        while (pos > 0 && myv[pos - 1] < s) {
          myv[pos] = myv[pos - 1];
          myi[pos] = myi[pos - 1];
          --pos;
        }
        myv[pos] = s;
        myi[pos] = (int32_t)j;
        if (fill < K) ++fill;
      }
    }
    __syncthreads();
  }
  if (tid < BM && qi < q_end) {
    for (int t = 0; t < K; ++t) {
      const bool ok = !qzero && t < fill;
      ids[(qi - q_begin) * K + t] = ok ? li[tid * K + t] : -1;
      scores[(qi - q_begin) * K + t] = ok ? fmin(lv[tid * K + t], 1.0) : 0.0;
    }
  }
}

size_t knn_simt_smem(int K) {
  return sizeof(double) * (BM * BK + BN * BK + BM * (BN + 1) + (size_t)BM * K) +
         sizeof(int32_t) * (size_t)BM * K;
}

int knn_simt(const double* xn, int64_t n, int64_t ldn, const double* norms, int K,
             int64_t q_begin, int64_t q_end, int32_t* ids, double* scores, cudaStream_t st) {
  const size_t smem = knn_simt_smem(K);
  ANCKA_REQUIRE(smem <= 220 * 1024, ANCKA_ERR_UNSUPPORTED, "knn_simt: K=%d too large", K);
  ANCKA_CUDA(cudaFuncSetAttribute(knn_simt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  knn_simt_kernel<<<(unsigned)ceil_div(q_end - q_begin, BM), 256, smem, st>>>(
      xn, n, ldn, norms, K, q_begin, q_end, ids, scores);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

int normalize_rows_f64(const double* X, int64_t n, int64_t d, int64_t ldx, double* xn, int64_t ldn,
                       double* norms, cudaStream_t st) {
  const int g = (int)std::min<int64_t>(ceil_div(n * 32, 256), 16 * kNumSMs);
  normalize_rows_f64_kernel<<<std::max(g, 1), 256, 0, st>>>(X, n, d, ldx, xn, ldn, norms);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

}  // namespace ancka
