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

// Query rows are q_begin + local (qlist == nullptr) or qlist[local] for
// local < *qcount (the uncertified rows of the tensor-core real path); CTAs
// stride over chunks of BM query rows.
__global__ void __launch_bounds__(256)
knn_simt_kernel(const double* __restrict__ xn, int64_t n, int64_t ldn, const double* __restrict__ norms,
                int K, int64_t q_begin, int64_t q_end, const int32_t* __restrict__ qlist,
                const int* __restrict__ qcount, int32_t* __restrict__ ids,
                double* __restrict__ scores, int64_t seg_len, double* __restrict__ part_v,
                int32_t* __restrict__ part_i, int64_t seg_cap) {
  extern __shared__ __align__(16) unsigned char smraw[];
  // seg_cap > 0: the segmented launch, which runs only when *qcount <= seg_cap;
  // seg_cap < 0: the single-segment launch, which runs only when *qcount > -seg_cap
  if (seg_cap != 0 && qlist) {
    const int64_t c = *qcount;
    if (seg_cap > 0 ? c > seg_cap : c <= -seg_cap) return;
  }
  double* As = reinterpret_cast<double*>(smraw);           // BM x BK
  double* Bs = As + BM * BK;                                // BN x BK
  double* S = Bs + BN * BK;                                 // BM x (BN+1)
  double* lv = S + BM * (BN + 1);                           // BM x K values
  int32_t* li = reinterpret_cast<int32_t*>(lv + (size_t)BM * K);  // BM x K ids
  int64_t* qrow = reinterpret_cast<int64_t*>(li + (size_t)BM * K + 2);  // BM query rows
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;  // 16 x 16 threads, 4 x 4 each
  const int64_t nq = qlist ? (int64_t)*qcount : q_end - q_begin;
  for (int64_t chunk = blockIdx.x; chunk * BM < nq; chunk += gridDim.x) {
    const int64_t base = chunk * BM;
    for (int r = tid; r < BM; r += blockDim.x)
      qrow[r] = base + r < nq ? (qlist ? (int64_t)qlist[base + r] : q_begin + base + r) : -1;
    int fill = 0;                            // list length (owner threads)
    for (int e = tid; e < BM * K; e += blockDim.x) { lv[e] = 0.0; li[e] = -1; }
    __syncthreads();
    const int64_t qi = tid < BM ? qrow[tid] : -1;
    const bool owner = qi >= 0;
    const bool qzero = owner ? norms[qi] == 0.0 : true;
    // key range of this CTA (blockIdx.y segments; one segment = all keys)
    const int64_t kbeg = (int64_t)blockIdx.y * seg_len;
    const int64_t kend = lmin(n, kbeg + seg_len);
    for (int64_t k0 = kbeg; k0 < kend; k0 += BN) {
      double acc[4][4] = {};
      for (int64_t d0 = 0; d0 < ldn; d0 += BK) {
        for (int e = tid; e < BM * BK; e += blockDim.x) {
          const int r = e / BK, c = e % BK;
          const int64_t qr = qrow[r], kr = k0 + r;
          As[e] = qr >= 0 ? xn[qr * ldn + d0 + c] : 0.0;
          Bs[e] = kr < kend ? xn[kr * ldn + d0 + c] : 0.0;
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
        const int jn = (int)lmin(BN, kend - k0);
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
    if (owner && part_v) {                   // partial list of this key segment
      const int64_t o = ((base + tid) * gridDim.y + blockIdx.y) * K;
      for (int t = 0; t < K; ++t) {
        const bool ok = !qzero && t < fill;
        part_i[o + t] = ok ? li[tid * K + t] : -1;
        part_v[o + t] = ok ? lv[tid * K + t] : 0.0;
      }
    } else if (owner) {
      const int64_t o = qi - q_begin;
      for (int t = 0; t < K; ++t) {
        const bool ok = !qzero && t < fill;
        ids[o * K + t] = ok ? li[tid * K + t] : -1;
        scores[o * K + t] = ok ? fmin(lv[tid * K + t], 1.0) : 0.0;
      }
    }
    __syncthreads();
  }
}

size_t knn_simt_smem(int K) {
  return sizeof(double) * (BM * BK + BN * BK + BM * (BN + 1) + (size_t)BM * K) +
         sizeof(int32_t) * ((size_t)BM * K + 2) + sizeof(int64_t) * BM;
}

int knn_simt(const double* xn, int64_t n, int64_t ldn, const double* norms, int K,
             int64_t q_begin, int64_t q_end, int32_t* ids, double* scores, cudaStream_t st) {
  const size_t smem = knn_simt_smem(K);
  ANCKA_REQUIRE(smem <= 220 * 1024, ANCKA_ERR_UNSUPPORTED, "knn_simt: K=%d too large", K);
  ANCKA_CUDA(cudaFuncSetAttribute(knn_simt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  knn_simt_kernel<<<(unsigned)ceil_div(q_end - q_begin, BM), 256, smem, st>>>(
      xn, n, ldn, norms, K, q_begin, q_end, nullptr, nullptr, ids, scores, n, nullptr, nullptr, 0);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

// Exact f64 rescan of the rows in qlist[0 .. *qcount) -- the count stays on
// the device, so the host does not wait for the search: up to kSegCap rows
// (the usual case: a handful) are spread over kSegs key segments so the
// rescan uses the whole GPU, then merged; more rows take one launch that
// strides over row chunks.  Each launch returns at once when the count
// selects the other.
constexpr int kSegs = 16;
constexpr int64_t kSegCap = 4 * BM * kNumSMs / kSegs * 4;

size_t knn_simt_list_workspace(int K) {
  return (size_t)kSegCap * kSegs * K * (sizeof(double) + sizeof(int32_t)) + 1024;
}

__global__ void knn_simt_merge_gate(const double* part_v, const int32_t* part_i, const int* qcount,
                                    int nseg, int K, const int32_t* qlist, int64_t q_begin,
                                    int32_t* ids, double* scores) {
  const int64_t c = *qcount;
  if (c == 0 || c > kSegCap) return;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < c;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = (qlist[r] - q_begin) * K;
    const double* v = part_v + r * nseg * K;
    const int32_t* id = part_i + r * nseg * K;
    int head[kSegs];
    for (int s2 = 0; s2 < nseg; ++s2) head[s2] = 0;
    for (int t = 0; t < K; ++t) {
      int best = -1;
      for (int s2 = 0; s2 < nseg; ++s2) {
        const int h = head[s2];
        if (h >= K || id[s2 * K + h] < 0) continue;
        if (best < 0) { best = s2; continue; }
        const double a = v[s2 * K + h], b = v[best * K + head[best]];
        if (a > b || (a == b && id[s2 * K + h] < id[best * K + head[best]])) best = s2;
      }
      if (best < 0) { ids[o + t] = -1; scores[o + t] = 0.0; continue; }
      ids[o + t] = id[best * K + head[best]];
      scores[o + t] = fmin(v[best * K + head[best]], 1.0);
      ++head[best];
    }
  }
}

int knn_simt_list(const double* xn, int64_t n, int64_t ldn, const double* norms, int K,
                  int64_t q_begin, const int32_t* qlist, const int* qcount, int32_t* ids,
                  double* scores, void* ws, size_t wsb, cudaStream_t st) {
  const size_t smem = knn_simt_smem(K);
  ANCKA_REQUIRE(smem <= 220 * 1024, ANCKA_ERR_UNSUPPORTED, "knn_simt: K=%d too large", K);
  ANCKA_CUDA(cudaFuncSetAttribute(knn_simt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t nseg = std::max<int64_t>(1, std::min<int64_t>(kSegs, ceil_div(n, 4 * BN)));
  const int64_t seg_len = ceil_div(ceil_div(n, nseg), BN) * BN;
  const int64_t nseg2 = ceil_div(n, seg_len);
  Carver cv(ws, wsb);
  double* pv = cv.take<double>((size_t)kSegCap * nseg2 * K);
  int32_t* pi = cv.take<int32_t>((size_t)kSegCap * nseg2 * K);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "knn_simt_list: workspace too small");
  // few rows: (row chunks x key segments), partial lists, merge
  const unsigned gx = (unsigned)std::max<int64_t>(1, 2 * kNumSMs / nseg2);
  knn_simt_kernel<<<dim3(gx, (unsigned)nseg2), 256, smem, st>>>(
      xn, n, ldn, norms, K, q_begin, 0, qlist, qcount, ids, scores, seg_len, pv, pi, kSegCap);
  ANCKA_LAUNCHED();
  knn_simt_merge_gate<<<2 * kNumSMs, 128, 0, st>>>(pv, pi, qcount, (int)nseg2, K, qlist, q_begin,
                                                   ids, scores);
  ANCKA_LAUNCHED();
  // many rows: one segment, CTAs stride over row chunks
  knn_simt_kernel<<<2 * kNumSMs, 256, smem, st>>>(xn, n, ldn, norms, K, q_begin, 0, qlist, qcount,
                                                  ids, scores, n, nullptr, nullptr, -kSegCap);
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
