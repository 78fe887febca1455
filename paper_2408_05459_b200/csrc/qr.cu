// Subsystem 3: per-iteration re-orthonormalisation (engine.py:130-149).
//
// f32 fast path = Cholesky-QR: deterministic f64 Gram partials over fixed row
// ranges, one-CTA f64 Cholesky + triangular inverse, then Q = Z R^-1 fused
// with the ||Q - Q_prev||_F^2 partials.  The unique QR with diag(R) > 0 is
// the reference's sign-fixed Householder QR (engine.py:148-149).
//
// f64 path = classical Gram-Schmidt with one re-orthogonalisation pass
// (CGS2), used for the parity-critical first step whose block is rank
// deficient by construction: it reports |R_jj| so the host
// applies the reference's rank test (engine.py:141-142) exactly.
#include "common.cuh"
#include "spmm.cuh"

namespace ancka {

constexpr int kGramThreads = 256;
constexpr int kGramBlocks = 2 * kNumSMs;
constexpr int kGramTile = 32;
constexpr int kApplyBlocks = 8 * kNumSMs;

__device__ __forceinline__ int packed_idx(int a, int b, int c) {  // a <= b
  return a * c - (a * (a - 1)) / 2 + (b - a);
}

// Each thread owns up to PP upper-triangle pairs; groups of threads split the
// rows of a tile when there are fewer pairs than threads.
template <int PP>
__global__ void __launch_bounds__(kGramThreads)
gram_partial_kernel(const float* __restrict__ Z, int64_t n, int64_t ld, int c,
                    double* __restrict__ partial) {
  extern __shared__ float tile[];  // kGramTile x c
  const int npairs = c * (c + 1) / 2;
  const int groups = npairs >= kGramThreads ? 1 : kGramThreads / npairs;
  const int slots = npairs >= kGramThreads ? kGramThreads : npairs;
  const int g = threadIdx.x / slots, slot = threadIdx.x % slots;
  const bool active = g < groups;

  int pa[PP], pb[PP];
  float acc32[PP];
  double acc64[PP];
#pragma unroll
  for (int q = 0; q < PP; ++q) {
    pa[q] = pb[q] = -1;
    acc64[q] = 0.0;
    int p = slot + q * slots;
    if (active && p < npairs) {
      int a = 0, rem = p;
      while (rem >= c - a) { rem -= c - a; ++a; }
      pa[q] = a;
      pb[q] = a + rem;
    }
  }
  const int64_t rows_per_block = ceil_div(n, gridDim.x);
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = lmin(n, r0 + rows_per_block);
  for (int64_t t0 = r0; t0 < r1; t0 += kGramTile) {
    const int tr = (int)lmin(kGramTile, r1 - t0);
    __syncthreads();
    for (int e = threadIdx.x; e < tr * c; e += blockDim.x) {
      int r = e / c, col = e % c;
      tile[r * c + col] = Z[(t0 + r) * ld + col];
    }
    __syncthreads();
    if (!active) continue;
#pragma unroll
    for (int q = 0; q < PP; ++q) acc32[q] = 0.f;
    for (int r = g; r < tr; r += groups) {
      const float* row = tile + r * c;
#pragma unroll
      for (int q = 0; q < PP; ++q)
        if (pa[q] >= 0) acc32[q] = fmaf(row[pa[q]], row[pb[q]], acc32[q]);
    }
#pragma unroll
    for (int q = 0; q < PP; ++q) acc64[q] += (double)acc32[q];
  }
  // combine groups in fixed order through shared memory
  __syncthreads();
  double* red = reinterpret_cast<double*>(tile);  // reuse (>= groups*slots doubles)
  if (groups > 1) {
    if (active) red[g * slots + slot] = acc64[0];
    __syncthreads();
    if (threadIdx.x < npairs) {
      double s = 0.0;
      for (int gg = 0; gg < groups; ++gg) s += red[gg * slots + threadIdx.x];
      partial[(int64_t)blockIdx.x * npairs + threadIdx.x] = s;
    }
  } else {
#pragma unroll
    for (int q = 0; q < PP; ++q) {
      int p = slot + q * slots;
      if (p < npairs) partial[(int64_t)blockIdx.x * npairs + p] = acc64[q];
    }
  }
}

// One CTA: reduce Gram partials (fixed order), Cholesky G = R^T R in packed
// upper storage (f64), pivot diagnostics, R^-1 (f32 copy for the apply).
__global__ void __launch_bounds__(256)
chol_kernel(const double* __restrict__ partial, int nblocks, int c, float* __restrict__ rinv32,
            double* __restrict__ rdiag, double* __restrict__ stats) {
  extern __shared__ double sm[];
  const int npairs = c * (c + 1) / 2;
  double* R = sm;               // packed upper, npairs
  double* X = sm + npairs;      // packed upper inverse, npairs
  __shared__ double s_minratio;
  __shared__ int s_bad;
  __shared__ double gsum[256];
  if (npairs >= (int)blockDim.x / 2) {
    for (int p = threadIdx.x; p < npairs; p += blockDim.x) {
      double s0 = 0.0, s1 = 0.0;
      int b = 0;
      for (; b + 1 < nblocks; b += 2) {
        s0 += partial[(int64_t)b * npairs + p];
        s1 += partial[(int64_t)(b + 1) * npairs + p];
      }
      if (b < nblocks) s0 += partial[(int64_t)b * npairs + p];
      R[p] = s0 + s1;
    }
  } else {  // G groups of threads sum interleaved block subsets; fixed-order combine
    const int G = blockDim.x / npairs, g = threadIdx.x / npairs, p = threadIdx.x % npairs;
    if (g < G) {
      double s = 0.0;
      for (int b = g; b < nblocks; b += G) s += partial[(int64_t)b * npairs + p];
      gsum[g * npairs + p] = s;
    }
    __syncthreads();
    if ((int)threadIdx.x < npairs) {
      double s = 0.0;
      for (int gg = 0; gg < G; ++gg) s += gsum[gg * npairs + threadIdx.x];
      R[threadIdx.x] = s;
    }
  }
  if (threadIdx.x == 0) { s_minratio = 1.0; s_bad = 0; }
  __syncthreads();
  for (int j = 0; j < c; ++j) {
    // diagonal
    if (threadIdx.x == 0) {
      const double g = R[packed_idx(j, j, c)];
      double piv = g;
      for (int l = 0; l < j; ++l) { double v = R[packed_idx(l, j, c)]; piv -= v * v; }
      double ratio = g > 0 ? piv / g : 0.0;
      if (ratio < s_minratio) s_minratio = ratio;
      if (!(ratio > 1e-9)) {
        s_bad += 1;
        piv = fmax(piv, 1e-30 + 1e-9 * fmax(g, 0.0));
      }
      R[packed_idx(j, j, c)] = sqrt(piv);
    }
    __syncthreads();
    const double rjj = R[packed_idx(j, j, c)];
    for (int k = j + 1 + threadIdx.x; k < c; k += blockDim.x) {
      double v = R[packed_idx(j, k, c)];
      for (int l = 0; l < j; ++l) v -= R[packed_idx(l, j, c)] * R[packed_idx(l, k, c)];
      R[packed_idx(j, k, c)] = v / rjj;
    }
    __syncthreads();
  }
  // inverse of upper-triangular R, one column per thread
  for (int b = threadIdx.x; b < c; b += blockDim.x) {
    X[packed_idx(b, b, c)] = 1.0 / R[packed_idx(b, b, c)];
    for (int a = b - 1; a >= 0; --a) {
      double s = 0.0;
      for (int l = a + 1; l <= b; ++l) s += R[packed_idx(a, l, c)] * X[packed_idx(l, b, c)];
      X[packed_idx(a, b, c)] = -s / R[packed_idx(a, a, c)];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < c * c; e += blockDim.x) {
    int a = e / c, b = e % c;
    rinv32[e] = a <= b ? (float)X[packed_idx(a, b, c)] : 0.f;
  }
  for (int j = threadIdx.x; j < c; j += blockDim.x) rdiag[j] = R[packed_idx(j, j, c)];
  if (threadIdx.x == 0) {  // accumulated across steps until the host resets them
    stats[1] = fmin(stats[1], s_minratio);
    stats[2] += (double)s_bad;
  }
}

// Q = Z R^-1 with ||Q - Q_prev||^2 block partials.
__global__ void __launch_bounds__(256)
apply_rinv_kernel(const float* __restrict__ Z, const float* __restrict__ Qprev,
                  float* __restrict__ Q, int64_t n, int64_t ld, int c,
                  const float* __restrict__ rinv, double* __restrict__ dq_partial) {
  extern __shared__ float rs[];  // c x c
  __shared__ double red[32];
  for (int e = threadIdx.x; e < c * c; e += blockDim.x) rs[e] = rinv[e];
  __syncthreads();
  const int nchunk = (int)((ld + 3) / 4);
  const int64_t total = n * nchunk;
  double dq = 0.0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / nchunk;
    const int j0 = (int)(t - row * nchunk) * 4;
    const float* z = Z + row * ld;
    float o[4] = {0.f, 0.f, 0.f, 0.f};
    const int jmax = min(c, j0 + 4);
    for (int l = 0; l < jmax; ++l) {
      const float zl = z[l];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0 + u;
        if (j < c && l <= j) o[u] = fmaf(zl, rs[l * c + j], o[u]);
      }
    }
    const float4 prev = *reinterpret_cast<const float4*>(Qprev + row * ld + j0);
    const float pv[4] = {prev.x, prev.y, prev.z, prev.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double d = (double)o[u] - (double)pv[u];
      if (j0 + u < c) dq += d * d;
    }
    *reinterpret_cast<float4*>(Q + row * ld + j0) = make_float4(o[0], o[1], o[2], o[3]);
  }
  dq = block_sum(dq, red);
  if (threadIdx.x == 0) dq_partial[blockIdx.x] = dq;
}

__global__ void reduce_partials_kernel(const double* __restrict__ partial, int nblocks,
                                       double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) s += partial[b];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

struct OrthWs {
  float* rinv32;
  double* rdiag;
  double* gram_partial;
  double* dq_partial;
  float* scratch;
};

static size_t carve_orth(Carver& cv, OrthWs& w, const ancka_operator* op, int c) {
  const int64_t ld = (c + 3) / 4 * 4;
  w.rinv32 = cv.take<float>((size_t)c * c);
  w.rdiag = cv.take<double>(c);
  w.gram_partial = cv.take<double>((size_t)kGramBlocks * c * (c + 1) / 2);
  w.dq_partial = cv.take<double>(kApplyBlocks);
  w.scratch = cv.take<float>(op && op->kind == ANCKA_HYPERGRAPH ? (size_t)op->m * ld : 1);
  return cv.used;
}

static int launch_gram(const float* Z, int64_t n, int64_t ld, int c, double* partial,
                       cudaStream_t st) {
  const int npairs = c * (c + 1) / 2;
  const int pp = (npairs + kGramThreads - 1) / kGramThreads;
  const size_t smem = std::max<size_t>((size_t)kGramTile * c * sizeof(float),
                                       (size_t)kGramThreads * sizeof(double));
#define GRAM_CASE(P)                                                                    \
  if (pp <= P) {                                                                        \
    if (smem > 48 * 1024)                                                               \
      cudaFuncSetAttribute(gram_partial_kernel<P>,                                      \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
    gram_partial_kernel<P><<<kGramBlocks, kGramThreads, smem, st>>>(Z, n, ld, c, partial); \
    ANCKA_LAUNCHED();                                                                   \
    return ANCKA_OK;                                                                    \
  }
  GRAM_CASE(1)
  GRAM_CASE(4)
  GRAM_CASE(16)
  GRAM_CASE(64)
#undef GRAM_CASE
  set_error("gram: block width c=%d too large", c);
  return ANCKA_ERR_UNSUPPORTED;
}

int cholqr_f32(const float* Z, const float* Qprev, float* Qout, int64_t n, int64_t ld, int c,
               double* stats, OrthWs& w, cudaStream_t st) {
  ANCKA_REQUIRE(c >= 1 && c <= 256 && ld % 4 == 0, ANCKA_ERR_ARG, "cholqr: bad c/ld");
  ANCKA_TRY(launch_gram(Z, n, ld, c, w.gram_partial, st));
  const int npairs = c * (c + 1) / 2;
  const size_t csm = 2 * (size_t)npairs * sizeof(double);
  ANCKA_REQUIRE(csm <= 227 * 1024, ANCKA_ERR_UNSUPPORTED, "cholqr: c=%d too large", c);
  if (csm > 48 * 1024)
    cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm);
  chol_kernel<<<1, 256, csm, st>>>(w.gram_partial, kGramBlocks, c, w.rinv32, w.rdiag, stats);
  ANCKA_LAUNCHED();
  const size_t asm_ = (size_t)c * c * sizeof(float);
  if (asm_ > 48 * 1024)
    cudaFuncSetAttribute(apply_rinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)asm_);
  apply_rinv_kernel<<<kApplyBlocks, 256, asm_, st>>>(Z, Qprev, Qout, n, ld, c, w.rinv32,
                                                     w.dq_partial);
  ANCKA_LAUNCHED();
  reduce_partials_kernel<<<1, 256, 0, st>>>(w.dq_partial, kApplyBlocks, stats);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

// ------------------------------------------------------------- f64 CGS2 ---
constexpr int kQrBlocks = 2 * kNumSMs;

// partial[l * nblk + b] = sum_{i in block b} Q[i, l] * Z[i, j]   for l < j
// (j == -1 denotes the norm of column `col`: partial[b] = sum Z[i,col]^2)
__global__ void __launch_bounds__(256)
cgs_dots_kernel(const double* __restrict__ Z, int64_t n, int64_t ld, int j,
                double* __restrict__ partial, int norm) {
  __shared__ double red[32];
  const int l = norm ? j : (int)blockIdx.y;  // l < j: projection; norm: ||Z[:,j]||^2
  const int64_t rows_per_block = ceil_div(n, gridDim.x);
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = lmin(n, r0 + rows_per_block);
  double s = 0.0;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    const double a = Z[i * ld + l], b = Z[i * ld + j];
    s = fma(a, b, s);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) partial[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
}

__global__ void cgs_reduce_kernel(const double* __restrict__ partial, int nblk, int cnt,
                                  double* __restrict__ out) {
  __shared__ double red[32];
  for (int l = 0; l < cnt; ++l) {
    double s = 0.0;
    for (int b = threadIdx.x; b < nblk; b += blockDim.x) s += partial[(int64_t)l * nblk + b];
    s = block_sum(s, red);
    if (threadIdx.x == 0) out[l] = s;
  }
}

// Z[:, j] -= Q[:, :j] proj   (mode 0)   or   Z[:, j] /= norm (mode 1)
__global__ void cgs_update_kernel(double* __restrict__ Z, int64_t n, int64_t ld, int j,
                                  const double* __restrict__ proj, int mode,
                                  double* __restrict__ rdiag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double* row = Z + i * ld;
    if (mode == 0) {
      double v = row[j];
      for (int l = 0; l < j; ++l) v -= row[l] * proj[l];
      row[j] = v;
    } else {
      const double nrm = sqrt(proj[j]);
      row[j] = nrm > 0 ? row[j] / nrm : 0.0;
      if (i == 0) rdiag[j] = nrm;
    }
  }
}

}  // namespace ancka

using namespace ancka;

extern "C" size_t ancka_orth_workspace_size(const ancka_operator* op, int32_t c) {
  Carver cv(nullptr, 0);
  OrthWs w;
  return carve_orth(cv, w, op, c);
}

extern "C" int ancka_orth_step_f32(const ancka_operator* op32, const float* Q_prev, float* Q_out,
                                   float* Z, int64_t ld, int32_t c, double* stats,
                                   void* workspace, size_t workspace_bytes,
                                   ancka_stream_t stream) {
  ANCKA_REQUIRE(op32 && op32->dtype == ANCKA_F32, ANCKA_ERR_ARG, "orth_step_f32 needs an f32 operator");
  Carver cv(workspace, workspace_bytes);
  OrthWs w;
  carve_orth(cv, w, op32, c);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "orth_step: workspace too small");
  auto st = as_stream(stream);
  ANCKA_TRY(op_apply_t<float>(op32, Q_prev, ld, c, Z, ld, w.scratch, st, nullptr));
  return cholqr_f32(Z, Q_prev, Q_out, op32->n, ld, c, stats, w, st);
}

extern "C" size_t ancka_qr_f64_workspace_size(int64_t n, int32_t c) {
  (void)n;
  Carver cv(nullptr, 0);
  cv.take<double>((size_t)kQrBlocks * (c + 1));
  cv.take<double>(c + 1);
  return cv.used;
}

extern "C" int ancka_qr_f64(double* Z, int64_t n, int64_t ld, int32_t c, double* rdiag,
                            void* workspace, size_t workspace_bytes, ancka_stream_t stream) {
  Carver cv(workspace, workspace_bytes);
  double* partial = cv.take<double>((size_t)kQrBlocks * (c + 1));
  double* proj = cv.take<double>(c + 1);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "qr_f64: workspace too small");
  auto st = as_stream(stream);
  const int ub = 256;
  const int ug = (int)std::min<int64_t>(ceil_div(n, ub), 4 * kNumSMs);
  for (int j = 0; j < c; ++j) {
    for (int pass = 0; pass < 2 && j > 0; ++pass) {
      cgs_dots_kernel<<<dim3(kQrBlocks, j), 256, 0, st>>>(Z, n, ld, j, partial, 0);
      cgs_reduce_kernel<<<1, 256, 0, st>>>(partial, kQrBlocks, j, proj);
      cgs_update_kernel<<<ug, ub, 0, st>>>(Z, n, ld, j, proj, 0, rdiag);
      note_launch();
      note_launch();
      ANCKA_LAUNCHED();
    }
    // norm: dots of column j with itself, stored at proj[j]
    cgs_dots_kernel<<<dim3(kQrBlocks, 1), 256, 0, st>>>(Z, n, ld, j, partial, 1);
    ANCKA_LAUNCHED();
    cgs_reduce_kernel<<<1, 256, 0, st>>>(partial, kQrBlocks, 1, proj + j);
    cgs_update_kernel<<<ug, ub, 0, st>>>(Z, n, ld, j, proj, 1, rdiag);
    note_launch();
    ANCKA_LAUNCHED();
  }
  return ANCKA_OK;
}

// ------------------------------------------- split CholQR (multi-GPU path) ---
// partial Gram of the local rows -> G (packed upper, f64); the caller
// all-reduces G across ranks, then ancka_cholqr_apply_f32 factors it.
namespace ancka {
__global__ void gram_reduce_kernel(const double* __restrict__ partial, int nblocks, int npairs,
                                   double* __restrict__ G) {
  for (int p = threadIdx.x; p < npairs; p += blockDim.x) {
    double s0 = 0.0, s1 = 0.0;
    int b = 0;
    for (; b + 1 < nblocks; b += 2) {
      s0 += partial[(int64_t)b * npairs + p];
      s1 += partial[(int64_t)(b + 1) * npairs + p];
    }
    if (b < nblocks) s0 += partial[(int64_t)b * npairs + p];
    G[p] = s0 + s1;
  }
}
}  // namespace ancka

extern "C" int ancka_gram_f32(const float* Z, int64_t n, int64_t ld, int32_t c, double* G,
                              void* workspace, size_t workspace_bytes, ancka_stream_t stream) {
  Carver cv(workspace, workspace_bytes);
  OrthWs w;
  carve_orth(cv, w, nullptr, c);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "gram: workspace too small");
  auto st = as_stream(stream);
  ANCKA_TRY(launch_gram(Z, n, ld, c, w.gram_partial, st));
  gram_reduce_kernel<<<1, 256, 0, st>>>(w.gram_partial, kGramBlocks, c * (c + 1) / 2, G);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

extern "C" int ancka_cholqr_apply_f32(const float* Z, const float* Q_prev, float* Q_out, int64_t n,
                                      int64_t ld, int32_t c, const double* G, double* stats,
                                      void* workspace, size_t workspace_bytes,
                                      ancka_stream_t stream) {
  Carver cv(workspace, workspace_bytes);
  OrthWs w;
  carve_orth(cv, w, nullptr, c);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "cholqr_apply: workspace too small");
  auto st = as_stream(stream);
  const int npairs = c * (c + 1) / 2;
  const size_t csm = 2 * (size_t)npairs * sizeof(double);
  ANCKA_REQUIRE(csm <= 227 * 1024, ANCKA_ERR_UNSUPPORTED, "cholqr: c=%d too large", c);
  if (csm > 48 * 1024)
    cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm);
  chol_kernel<<<1, 256, csm, st>>>(G, 1, c, w.rinv32, w.rdiag, stats);
  ANCKA_LAUNCHED();
  const size_t asm_ = (size_t)c * c * sizeof(float);
  if (asm_ > 48 * 1024)
    cudaFuncSetAttribute(apply_rinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)asm_);
  apply_rinv_kernel<<<kApplyBlocks, 256, asm_, st>>>(Z, Q_prev, Q_out, n, ld, c, w.rinv32,
                                                     w.dq_partial);
  ANCKA_LAUNCHED();
  reduce_partials_kernel<<<1, 256, 0, st>>>(w.dq_partial, kApplyBlocks, stats);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}
