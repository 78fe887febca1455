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
#include <cooperative_groups.h>
#include <cstdlib>

#include "common.cuh"
#include "spmm.cuh"

namespace cg = cooperative_groups;

namespace ancka {

constexpr int kGramThreads = 256;
constexpr int kGramBlocks = 2 * kNumSMs;
constexpr int kApplyBlocks = 8 * kNumSMs;
constexpr int kMaxC = 256;     // widest block (Papers100M: c = 173)

__device__ __forceinline__ int packed_idx(int a, int b, int c) {  // a <= b
  return a * c - (a * (a - 1)) / 2 + (b - a);
}

// Register-blocked Gram partials: thread = one 4 x 4 block (bi <= bj) of the
// upper triangle of Z^T Z; a tile of kGT rows is staged in shared memory with
// float4 loads (rows of Z are contiguous at stride ld), every row contributes
// 16 FMAs per two LDS.128.  f32 sums per tile, promoted to f64 per tile; row
// groups (when there are fewer block pairs than threads) combine in fixed
// order.  blockIdx.y splits the block pairs for wide blocks (c > 88).
constexpr int kGT = 64;
__global__ void __launch_bounds__(kGramThreads)
gram_blocked_kernel(const float* __restrict__ Z, int64_t n, int64_t ld, int c,
                    double* __restrict__ partial) {
  extern __shared__ __align__(16) float gtile[];   // kGT x ld, then reduction scratch
  const int nb4 = (c + 3) / 4;
  const int nbp = nb4 * (nb4 + 1) / 2;
  const int npairs = c * (c + 1) / 2;
  const int per_y = (nbp + gridDim.y - 1) / gridDim.y;
  const int q0 = blockIdx.y * per_y, q1 = min(nbp, q0 + per_y);
  const int nq = q1 - q0;
  const int groups = nq >= kGramThreads ? 1 : kGramThreads / nq;
  const int g = threadIdx.x / nq, q = q0 + threadIdx.x % nq;
  const bool active = g < groups && threadIdx.x % nq + q0 < q1 && nq > 0;
  int bi = 0, bj = 0;
  if (active) {
    int rem = q;
    while (rem >= nb4 - bi) { rem -= nb4 - bi; ++bi; }
    bj = bi + rem;
  }
  float acc32[16];
  double acc64[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) acc64[u] = 0.0;
  const int64_t rows_per_block = ceil_div(n, gridDim.x);
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = lmin(n, r0 + rows_per_block);
  const int ld4 = (int)(ld / 4);
  // double-buffered tiles: the copy of tile t + 1 runs under tile t's FMAs
  auto stage = [&](int64_t t0, int b) {
    const int tr = (int)lmin(kGT, r1 - t0);
    const float4* src = reinterpret_cast<const float4*>(Z + t0 * ld);
    float* dst = gtile + (size_t)b * kGT * ld;
    for (int e = threadIdx.x; e < tr * ld4; e += blockDim.x)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(dst + 4 * e)),
                   "l"(src + e)
                   : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (r0 < r1) stage(r0, 0);
  int buf = 0;
  for (int64_t t0 = r0; t0 < r1; t0 += kGT, buf ^= 1) {
    const int tr = (int)lmin(kGT, r1 - t0);
    if (t0 + kGT < r1) {
      stage(t0 + kGT, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const float* tile = gtile + (size_t)buf * kGT * ld;
    if (active) {
#pragma unroll
      for (int u = 0; u < 16; ++u) acc32[u] = 0.f;
      for (int r = g; r < tr; r += groups) {
        const float4 a = *reinterpret_cast<const float4*>(tile + r * ld + 4 * bi);
        const float4 b = *reinterpret_cast<const float4*>(tile + r * ld + 4 * bj);
        const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc32[u * 4 + v] = fmaf(av[u], bv[v], acc32[u * 4 + v]);
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) acc64[u] += (double)acc32[u];
    }
    __syncthreads();                          // buffer free for the copy after next
  }
  __syncthreads();
  double* red = reinterpret_cast<double*>(gtile);  // groups x nq x 16 doubles
  if (active) {
#pragma unroll
    for (int u = 0; u < 16; ++u) red[((size_t)g * nq + (threadIdx.x % nq)) * 16 + u] = acc64[u];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nq * 16; e += blockDim.x) {
    const int qq = e / 16, u = e % 16;
    double s2 = 0.0;
    for (int gg = 0; gg < groups; ++gg) s2 += red[((size_t)gg * nq + qq) * 16 + u];
    int a0 = 0, rem = q0 + qq;
    while (rem >= nb4 - a0) { rem -= nb4 - a0; ++a0; }
    const int a = 4 * a0 + u / 4, b = 4 * (a0 + rem) + u % 4;
    if (a < c && b < c && a <= b) partial[(int64_t)blockIdx.x * npairs + packed_idx(a, b, c)] = s2;
  }
}

// Q = Z R^-1 with ||Q - Q_prev||^2 block partials.  A tile of kAT rows is
// staged transposed in shared memory (zt[l][r]); a thread computes a 4 x 4
// block (4 rows x 4 columns) per pass, so one LDS.128 of Z and one of R^-1
// feed 16 FMAs.
constexpr int kAT = 64;
constexpr int kATS = kAT + 4;                     // padded stride of the transposed tile
__global__ void __launch_bounds__(256)
apply_rinv_tiled_kernel(const float* __restrict__ Z, const float* __restrict__ Qprev,
                        float* __restrict__ Q, int64_t n, int64_t ld, int c,
                        const float* __restrict__ rinv, double* __restrict__ dq_partial) {
  extern __shared__ __align__(16) float asm_[];
  float* rs = asm_;                               // c x ld (row l, col j), zero padded
  float* zt = asm_ + (size_t)c * ld;              // ld x kATS (column l, row r)
  __shared__ double red[32];
  for (int e = threadIdx.x; e < c * (int)ld; e += blockDim.x) {
    const int l = e / (int)ld, j = e % (int)ld;
    rs[e] = j < c ? rinv[l * c + j] : 0.f;
  }
  const int nchunk = (int)(ld / 4);
  const int npair = (kAT / 4) * nchunk;           // (row group, column chunk) pairs
  const int ld4 = (int)(ld / 4);
  double dq = 0.0;
  for (int64_t t0 = (int64_t)blockIdx.x * kAT; t0 < n; t0 += (int64_t)gridDim.x * kAT) {
    const int tr = (int)lmin(kAT, n - t0);
    __syncthreads();
    const float4* src = reinterpret_cast<const float4*>(Z + t0 * ld);
    for (int e = threadIdx.x; e < tr * ld4; e += blockDim.x) {
      const int r = e / ld4, q = e - r * ld4;
      const float4 v = __ldg(src + e);
      zt[(4 * q + 0) * kATS + r] = v.x;
      zt[(4 * q + 1) * kATS + r] = v.y;
      zt[(4 * q + 2) * kATS + r] = v.z;
      zt[(4 * q + 3) * kATS + r] = v.w;
    }
    __syncthreads();
    for (int pp = threadIdx.x; pp < npair; pp += blockDim.x) {
      const int rg = pp / nchunk, ch = pp - rg * nchunk;
      const int r0 = rg * 4, j0 = ch * 4;
      if (r0 >= tr) continue;
      float o[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) o[u][v] = 0.f;
      const int lmax = min(c, j0 + 4);            // R^-1 is upper triangular
      for (int l = 0; l < lmax; ++l) {
        const float4 z = *reinterpret_cast<const float4*>(zt + l * kATS + r0);
        const float4 w = *reinterpret_cast<const float4*>(rs + l * ld + j0);
        const float zv[4] = {z.x, z.y, z.z, z.w}, wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) o[u][v] = fmaf(zv[u], wv[v], o[u][v]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (r0 + u >= tr) break;
        const int64_t row = t0 + r0 + u;
        const float4 prev = *reinterpret_cast<const float4*>(Qprev + row * ld + j0);
        const float pv[4] = {prev.x, prev.y, prev.z, prev.w};
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const double d = (double)o[u][v] - (double)pv[v];
          if (j0 + v < c) dq += d * d;
        }
        *reinterpret_cast<float4*>(Q + row * ld + j0) = make_float4(o[u][0], o[u][1], o[u][2], o[u][3]);
      }
    }
  }
  dq = block_sum(dq, red);
  if (threadIdx.x == 0) dq_partial[blockIdx.x] = dq;
}

// Q = Z R^-1 for c <= 64: a thread per row, the row and its c outputs in
// registers, R^-1 in shared memory (every lane reads the same entry:
// broadcast); Z, Q_prev and Q rows move as float4s.  The same f32 sums in
// the same l order as apply_rinv_tiled_kernel (R^-1 is upper triangular, the
// skipped terms are exact zeros).
template <int CM>
__global__ void __launch_bounds__(256)
apply_rinv_rows_kernel(const float* __restrict__ Z, const float* __restrict__ Qprev,
                       float* __restrict__ Q, int64_t n, int64_t ld, int c,
                       const float* __restrict__ rinv, double* __restrict__ dq_partial) {
  __shared__ __align__(16) float rs[CM * CM];     // R^-1 (row l, col j), zero outside c
  __shared__ double red[32];
  for (int e = threadIdx.x; e < CM * CM; e += blockDim.x) {
    const int l = e / CM, j = e % CM;
    rs[e] = (l < c && j < c) ? rinv[l * c + j] : 0.f;
  }
  __syncthreads();
  const int ld4 = (int)(ld / 4);
  double dq = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float z[CM], o[CM];
    const float4* zr = reinterpret_cast<const float4*>(Z + i * ld);
#pragma unroll
    for (int q = 0; q < CM / 4; ++q) {
      const float4 v = q < ld4 ? __ldg(zr + q) : make_float4(0.f, 0.f, 0.f, 0.f);
      z[4 * q] = v.x; z[4 * q + 1] = v.y; z[4 * q + 2] = v.z; z[4 * q + 3] = v.w;
    }
#pragma unroll
    for (int j = 0; j < CM; ++j) o[j] = 0.f;
#pragma unroll
    for (int l = 0; l < CM; ++l) {
      if (l < c) {
        const float zl = z[l];
        const float4* rl = reinterpret_cast<const float4*>(rs + l * CM);
#pragma unroll
        for (int q = l / 4; q < CM / 4; ++q) {
          const float4 w = rl[q];
          o[4 * q] = fmaf(zl, w.x, o[4 * q]);
          o[4 * q + 1] = fmaf(zl, w.y, o[4 * q + 1]);
          o[4 * q + 2] = fmaf(zl, w.z, o[4 * q + 2]);
          o[4 * q + 3] = fmaf(zl, w.w, o[4 * q + 3]);
        }
      }
    }
    const float4* pr = reinterpret_cast<const float4*>(Qprev + i * ld);
    float4* qr = reinterpret_cast<float4*>(Q + i * ld);
#pragma unroll
    for (int q = 0; q < CM / 4; ++q) {
      if (q < ld4) {
        const float4 pv = __ldg(pr + q);
        const float pvv[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const double d = (double)o[4 * q + v] - (double)pvv[v];
          if (4 * q + v < c) dq += d * d;
        }
        qr[q] = make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
      }
    }
  }
  dq = block_sum(dq, red);
  if (threadIdx.x == 0) dq_partial[blockIdx.x] = dq;
}

// Fixed-order reduction of per-block Gram partials, one thread per packed
// pair (several CTAs), so the single-CTA Cholesky reads one G.
__global__ void __launch_bounds__(256)
gram_sum_kernel(const double* __restrict__ partial, int nblocks, int npairs,
                double* __restrict__ G) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npairs) return;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int b = 0;
  for (; b + 3 < nblocks; b += 4) {
    s0 += partial[(int64_t)b * npairs + p];
    s1 += partial[(int64_t)(b + 1) * npairs + p];
    s2 += partial[(int64_t)(b + 2) * npairs + p];
    s3 += partial[(int64_t)(b + 3) * npairs + p];
  }
  for (; b < nblocks; ++b) s0 += partial[(int64_t)b * npairs + p];
  G[p] = (s0 + s1) + (s2 + s3);
}

// One CTA: reduce Gram partials (fixed order), Cholesky G = R^T R in packed
// upper storage (f64), pivot diagnostics, R^-1 (f32 copy for the apply).
__global__ void __launch_bounds__(256)
chol_kernel(const double* __restrict__ partial, int nblocks, int c, float* __restrict__ rinv32,
            double* __restrict__ rdiag, double* __restrict__ stats) {
  extern __shared__ double sm[];
  const int npairs = c * (c + 1) / 2;
  double* R = sm;               // packed upper, npairs
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
  // inverse of upper-triangular R, one column per thread (the column lives in
  // a per-thread local array, so only R occupies shared memory)
  for (int b = threadIdx.x; b < c; b += blockDim.x) {
    double xc[kMaxC];
    xc[b] = 1.0 / R[packed_idx(b, b, c)];
    for (int a = b - 1; a >= 0; --a) {
      double s = 0.0;
      for (int l = a + 1; l <= b; ++l) s += R[packed_idx(a, l, c)] * xc[l];
      xc[a] = -s / R[packed_idx(a, a, c)];
    }
    for (int a = 0; a < c; ++a) rinv32[a * c + b] = a <= b ? (float)xc[a] : 0.f;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < c; j += blockDim.x) rdiag[j] = R[packed_idx(j, j, c)];
  if (threadIdx.x == 0) {  // accumulated across steps until the host resets them
    stats[1] = fmin(stats[1], s_minratio);
    stats[2] += (double)s_bad;
  }
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
  double* gsum;
};

static size_t carve_orth(Carver& cv, OrthWs& w, const ancka_operator* op, int c) {
  const int64_t ld = (c + 3) / 4 * 4;
  w.rinv32 = cv.take<float>((size_t)c * c);
  w.rdiag = cv.take<double>(c);
  w.gram_partial = cv.take<double>((size_t)kGramBlocks * c * (c + 1) / 2);
  w.dq_partial = cv.take<double>(kApplyBlocks);
  w.scratch = cv.take<float>(op && op->kind == ANCKA_HYPERGRAPH ? (size_t)op->m * ld : 1);
  w.gsum = cv.take<double>((size_t)c * (c + 1) / 2);
  return cv.used;
}

static int launch_gram(const float* Z, int64_t n, int64_t ld, int c, double* partial,
                       cudaStream_t st) {
  const int nb4 = (c + 3) / 4;
  const int nbp = nb4 * (nb4 + 1) / 2;
  const int ny = (nbp + kGramThreads - 1) / kGramThreads;
  const int nq = (nbp + ny - 1) / ny;
  const int groups = nq >= kGramThreads ? 1 : kGramThreads / nq;
  const size_t smem = std::max<size_t>((size_t)2 * kGT * ld * sizeof(float),
                                       (size_t)groups * nq * 16 * sizeof(double));
  if (smem > 48 * 1024)
    ANCKA_CUDA(cudaFuncSetAttribute(gram_blocked_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
  gram_blocked_kernel<<<dim3(kGramBlocks, ny), kGramThreads, smem, st>>>(Z, n, ld, c, partial);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

static int launch_apply(const float* Z, const float* Qprev, float* Qout, int64_t n, int64_t ld,
                        int c, const float* rinv, double* dq_partial, cudaStream_t st) {
  if (c <= 64 && !getenv("ANCKA_QR_TILED_APPLY")) {
    const int cm = c <= 16 ? 16 : c <= 32 ? 32 : c <= 48 ? 48 : 64;
    if (cm == 16) apply_rinv_rows_kernel<16><<<kApplyBlocks, 256, 0, st>>>(Z, Qprev, Qout, n, ld, c, rinv, dq_partial);
    else if (cm == 32) apply_rinv_rows_kernel<32><<<kApplyBlocks, 256, 0, st>>>(Z, Qprev, Qout, n, ld, c, rinv, dq_partial);
    else if (cm == 48) apply_rinv_rows_kernel<48><<<kApplyBlocks, 256, 0, st>>>(Z, Qprev, Qout, n, ld, c, rinv, dq_partial);
    else apply_rinv_rows_kernel<64><<<kApplyBlocks, 256, 0, st>>>(Z, Qprev, Qout, n, ld, c, rinv, dq_partial);
    ANCKA_LAUNCHED();
    return ANCKA_OK;
  }
  const size_t smem = ((size_t)c * ld + (size_t)ld * kATS) * sizeof(float);
  ANCKA_REQUIRE(smem <= 227 * 1024 && ld / 4 <= 256, ANCKA_ERR_UNSUPPORTED, "apply: c=%d too large", c);
  if (smem > 48 * 1024)
    ANCKA_CUDA(cudaFuncSetAttribute(apply_rinv_tiled_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  apply_rinv_tiled_kernel<<<kApplyBlocks, 256, smem, st>>>(Z, Qprev, Qout, n, ld, c, rinv, dq_partial);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

int cholqr_f32(const float* Z, const float* Qprev, float* Qout, int64_t n, int64_t ld, int c,
               double* stats, OrthWs& w, cudaStream_t st) {
  ANCKA_REQUIRE(c >= 1 && c <= 256 && ld % 4 == 0, ANCKA_ERR_ARG, "cholqr: bad c/ld");
  ANCKA_TRY(launch_gram(Z, n, ld, c, w.gram_partial, st));
  const int npairs = c * (c + 1) / 2;
  const size_t csm = (size_t)npairs * sizeof(double);
  ANCKA_REQUIRE(csm <= 227 * 1024, ANCKA_ERR_UNSUPPORTED, "cholqr: c=%d too large", c);
  if (csm > 48 * 1024)
    cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm);
  gram_sum_kernel<<<(npairs + 255) / 256, 256, 0, st>>>(w.gram_partial, kGramBlocks, npairs, w.gsum);
  ANCKA_LAUNCHED();
  chol_kernel<<<1, 256, csm, st>>>(w.gsum, 1, c, w.rinv32, w.rdiag, stats);
  ANCKA_LAUNCHED();
  ANCKA_TRY(launch_apply(Z, Qprev, Qout, n, ld, c, w.rinv32, w.dq_partial, st));
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

// One cooperative kernel for the whole f64 CGS2 (the step-1 QR): CTA b owns
// rows [b*rpb, (b+1)*rpb).  Per column j: two projection passes and the
// norm, each a CTA-local partial -> grid barrier -> fixed-order reduction of
// the partials by every CTA (identical, deterministic) -> local update.
// Rows are read warp-wide (lane = column), so every pass streams the
// row-major block coalesced.
constexpr int kCgsWarps = 8;
__global__ void __launch_bounds__(32 * kCgsWarps)
cgs2_fused_kernel(double* __restrict__ Z, int64_t n, int64_t ld, int c,
                  double* __restrict__ partial, double* __restrict__ rdiag) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double wpart[kCgsWarps][kMaxC];
  __shared__ double proj[kMaxC];
  const int nb = gridDim.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t rpb = ceil_div(n, (int64_t)nb);
  const int64_t r0 = (int64_t)blockIdx.x * rpb, r1 = lmin(n, r0 + rpb);
  int buf = 0;
  auto reduce_cols = [&](int cnt, double* part) {   // warp partials -> CTA partial[blk]
    __syncthreads();
    for (int l = threadIdx.x; l < cnt; l += blockDim.x) {
      double s = 0.0;
      for (int ww = 0; ww < kCgsWarps; ++ww) s += wpart[ww][l];
      part[(size_t)blockIdx.x * kMaxC + l] = s;
    }
  };
  // all CTAs' partials -> proj: per column, the CTA's threads load the
  // partials in parallel and sum them with the fixed block tree
  // (deterministic, and no serial chain of L2 loads)
  auto total_cols = [&](int cnt, const double* part) {
    __shared__ double tred[32];
    for (int l = 0; l < cnt; ++l) {
      double v = 0.0;
      for (int b = threadIdx.x; b < nb; b += blockDim.x) v += __ldcg(part + (size_t)b * kMaxC + l);
      v = block_sum(v, tred);
      if (threadIdx.x == 0) proj[l] = v;
    }
    __syncthreads();
  };
  for (int j = 0; j < c; ++j) {
    for (int pass = 0; pass < 2 && j > 0; ++pass) {
      double* part = partial + (size_t)buf * nb * kMaxC;
      // thread per row (independent loads in flight across the CTA); the
      // j products of a 32-row batch are summed across the warp per column
      for (int l = threadIdx.x; l < kCgsWarps * kMaxC; l += blockDim.x) (&wpart[0][0])[l] = 0.0;
      __syncthreads();
      // per-thread partial dots in registers over 16-column blocks, one warp
      // reduction per block (fixed order: rows by thread, lanes by tree)
      for (int lb = 0; lb < j; lb += 16) {
        double acc[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) acc[u] = 0.0;
        for (int64_t i = r0 + (int64_t)w * 32 + lane; i < r1; i += 32 * kCgsWarps) {
          const double* row = Z + i * ld;
          const double zj = row[j];
#pragma unroll
          for (int u = 0; u < 16; ++u)
            if (lb + u < j) acc[u] = fma(row[lb + u], zj, acc[u]);
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          if (lb + u >= j) break;
          const double v = warp_sum(acc[u]);
          if (lane == 0) wpart[w][lb + u] = v;
        }
      }
      reduce_cols(j, part);
      grid.sync();
      total_cols(j, part);
      for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {   // Z[:,j] -= Q[:, :j] proj
        double* row = Z + i * ld;
        double v = row[j];
        for (int l = 0; l < j; ++l) v -= row[l] * proj[l];
        row[j] = v;
      }
      buf ^= 1;
      __syncthreads();
    }
    double* part = partial + (size_t)buf * nb * kMaxC;
    double s = 0.0;
    for (int64_t i = r0 + w * 32 + lane; i < r1; i += 32 * kCgsWarps) {
      const double v = Z[i * ld + j];
      s = fma(v, v, s);
    }
    s = warp_sum(s);
    if (lane == 0) wpart[w][0] = s;
    reduce_cols(1, part);
    grid.sync();
    total_cols(1, part);
    const double nrm = sqrt(proj[0]);
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x)
      Z[i * ld + j] = nrm > 0 ? Z[i * ld + j] / nrm : 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) rdiag[j] = nrm;
    buf ^= 1;
    __syncthreads();
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
  cv.take<double>((size_t)2 * 2 * kNumSMs * kMaxC);   // fused CGS2 partials
  return cv.used;
}

extern "C" int ancka_qr_f64(double* Z, int64_t n, int64_t ld, int32_t c, double* rdiag,
                            void* workspace, size_t workspace_bytes, ancka_stream_t stream) {
  Carver cv(workspace, workspace_bytes);
  double* partial = cv.take<double>((size_t)kQrBlocks * (c + 1));
  double* proj = cv.take<double>(c + 1);
  double* fpart = cv.take<double>((size_t)2 * 2 * kNumSMs * kMaxC);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "qr_f64: workspace too small");
  auto st = as_stream(stream);
  if (c <= kMaxC && !getenv("ANCKA_QR_UNFUSED")) {    // one cooperative launch
    int per_sm = 0, dev = 0, sms = 0;
    ANCKA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cgs2_fused_kernel,
                                                             32 * kCgsWarps, 0));
    ANCKA_CUDA(cudaGetDevice(&dev));
    ANCKA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int grid = (int)std::min<int64_t>(ceil_div(n, 256), std::min(per_sm, 2) * (int64_t)sms);
    grid = std::max(grid, 1);
    void* args[] = {&Z, &n, &ld, &c, &fpart, &rdiag};
    note_launch();
    ANCKA_CUDA(cudaLaunchCooperativeKernel((void*)cgs2_fused_kernel, dim3(grid),
                                           dim3(32 * kCgsWarps), args, 0, st));
    return ANCKA_OK;
  }
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

extern "C" int ancka_gram_f32(const float* Z, int64_t n, int64_t ld, int32_t c, double* G,
                              void* workspace, size_t workspace_bytes, ancka_stream_t stream) {
  Carver cv(workspace, workspace_bytes);
  OrthWs w;
  carve_orth(cv, w, nullptr, c);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "gram: workspace too small");
  auto st = as_stream(stream);
  ANCKA_TRY(launch_gram(Z, n, ld, c, w.gram_partial, st));
  gram_sum_kernel<<<(c * (c + 1) / 2 + 255) / 256, 256, 0, st>>>(w.gram_partial, kGramBlocks,
                                                                 c * (c + 1) / 2, G);
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
  const size_t csm = (size_t)npairs * sizeof(double);
  ANCKA_REQUIRE(csm <= 227 * 1024, ANCKA_ERR_UNSUPPORTED, "cholqr: c=%d too large", c);
  if (csm > 48 * 1024)
    cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm);
  chol_kernel<<<1, 256, csm, st>>>(G, 1, c, w.rinv32, w.rdiag, stats);
  ANCKA_LAUNCHED();
  ANCKA_TRY(launch_apply(Z, Q_prev, Q_out, n, ld, c, w.rinv32, w.dq_partial, st));
  reduce_partials_kernel<<<1, 256, 0, st>>>(w.dq_partial, kApplyBlocks, stats);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}
