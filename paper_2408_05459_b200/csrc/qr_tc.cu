// Cholesky-QR on the tensor cores for blocks wider than the fused kernel
// (engine.py:130-149; 12 n c bytes, 3 n c^2 FLOP).
//
// Both dense contractions run as warp-level TF32 MMAs (m16n8k8) in three
// products, x = hi + lo with hi = rna_tf32(x), lo = x - hi truncated by the
// MMA: hi.hi + hi.lo + lo.hi carries ~2^-21 relative error per product,
// the f32 accumulation error of the SIMT kernels they replace.
//
// * gram_tc_kernel   per CTA a contiguous row range staged in 128-row tiles;
//                    each warp owns up to four 16 x 8 blocks of the upper
//                    triangle of Z^T Z; a tile's f32 sums are promoted to f64
//                    per block, and the CTA partials are summed in a fixed
//                    order afterwards (gram_sum_kernel): deterministic.
// * apply_tc_kernel  Q = Z R^-1 per 128-row tile (a warp per 16 rows, all c
//                    columns; R^-1 upper triangular, so k-steps below the
//                    diagonal block are skipped) fused with the
//                    ||Q - Q_prev||^2 partials.
#include "common.cuh"

namespace ancka {

namespace {
constexpr int kTR = 128;             // rows per staged tile
constexpr int kTW = 8;               // warps per CTA
constexpr int kTileBlocks = 4;       // 16 x 8 Gram blocks per warp

__device__ __forceinline__ uint32_t tf32_rna_q(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void mma_tf32_q(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                           uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// x -> (hi, lo) tf32 bit patterns
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = tf32_rna_q(x);
  lo = __float_as_uint(x - __uint_as_float(hi));
}
// three-product MMA on split operands
__device__ __forceinline__ void mma3(float (&d)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4],
                                     uint32_t bh0, uint32_t bh1, uint32_t bl0, uint32_t bl1) {
  mma_tf32_q(d, ah[0], ah[1], ah[2], ah[3], bh0, bh1);
  mma_tf32_q(d, ah[0], ah[1], ah[2], ah[3], bl0, bl1);
  mma_tf32_q(d, al[0], al[1], al[2], al[3], bh0, bh1);
}

__host__ __device__ inline int tc_ldz(int64_t ld) {       // smem row stride: == 8 (mod 32)
  int s = (int)((ld + 7) / 8 * 8);
  while (s % 32 != 8) s += 8;
  return s;
}
__device__ __forceinline__ int packed_ix(int a, int b, int c) {  // a <= b
  return a * c - (a * (a - 1)) / 2 + (b - a);
}
}  // namespace

// Gram partials.  Block list: (ma, nb) with 16 ma <= 8 nb + 7 (touches the
// upper triangle); warp w of CTA column y owns blocks (y * kTW + w) * kTileBlocks + i.
__global__ void __launch_bounds__(32 * kTW)
gram_tc_kernel(const float* __restrict__ Z, int64_t n, int64_t ld, int c,
               double* __restrict__ partial) {
  extern __shared__ __align__(16) float zt[];            // kTR x ldz
  const int ldz = tc_ldz(ld);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int mb16 = (c + 15) / 16, nb8 = (c + 7) / 8;
  const int npairs = c * (c + 1) / 2;
  // my blocks
  int bm[kTileBlocks], bn[kTileBlocks];
  int nmine = 0;
  {
    int idx = 0;
    const int first = (blockIdx.y * kTW + warp) * kTileBlocks;
    for (int ma = 0; ma < mb16; ++ma)
      for (int nb = 0; nb < nb8; ++nb) {
        if (16 * ma > 8 * nb + 7) continue;              // entirely below the diagonal
        if (idx >= first && idx < first + kTileBlocks) { bm[nmine] = ma; bn[nmine] = nb; ++nmine; }
        ++idx;
      }
  }
  double acc64[kTileBlocks][4];
#pragma unroll
  for (int i = 0; i < kTileBlocks; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc64[i][q] = 0.0;
  const int64_t rows_per_block = ceil_div(n, gridDim.x);
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = lmin(n, r0 + rows_per_block);
  const int ld4 = (int)(ld / 4);
  for (int64_t t0 = r0; t0 < r1; t0 += kTR) {
    const int tr = (int)lmin(kTR, r1 - t0);
    __syncthreads();
    for (int e = threadIdx.x; e < kTR * ld4; e += blockDim.x) {
      const int r = e / ld4, q = e - r * ld4;
      const float4 v = r < tr ? __ldg(reinterpret_cast<const float4*>(Z + (t0 + r) * ld) + q)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(zt + r * ldz + 4 * q) = v;
    }
    __syncthreads();
    if (nmine == 0) continue;
    float acc[kTileBlocks][4];
#pragma unroll
    for (int i = 0; i < kTileBlocks; ++i)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[i][q] = 0.f;
    const int ksteps = (tr + 7) / 8;
    for (int ks = 0; ks < ksteps; ++ks) {
      const float* zr0 = zt + (ks * 8 + t) * ldz;       // row ks*8 + t
      const float* zr1 = zr0 + 4 * ldz;                 // row ks*8 + t + 4
#pragma unroll
      for (int i = 0; i < kTileBlocks; ++i) {
        if (i >= nmine) break;
        const int ca = bm[i] * 16 + g, cb = bn[i] * 8 + g;
        uint32_t ah[4], al[4];
        // A = Z^T (16 columns of Z x 8 rows): a0 (g, t), a1 (g+8, t), a2 (g, t+4), a3 (g+8, t+4)
        split_tf32(ca < c ? zr0[ca] : 0.f, ah[0], al[0]);
        split_tf32(ca + 8 < c ? zr0[ca + 8] : 0.f, ah[1], al[1]);
        split_tf32(ca < c ? zr1[ca] : 0.f, ah[2], al[2]);
        split_tf32(ca + 8 < c ? zr1[ca + 8] : 0.f, ah[3], al[3]);
        uint32_t bh0, bl0, bh1, bl1;                     // B = Z (8 rows x 8 columns)
        split_tf32(cb < c ? zr0[cb] : 0.f, bh0, bl0);
        split_tf32(cb < c ? zr1[cb] : 0.f, bh1, bl1);
        mma3(acc[i], ah, al, bh0, bh1, bl0, bl1);
      }
    }
#pragma unroll
    for (int i = 0; i < kTileBlocks; ++i)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc64[i][q] += (double)acc[i][q];
  }
  // C fragment: (g, 2t), (g, 2t+1), (g+8, 2t), (g+8, 2t+1)
#pragma unroll
  for (int i = 0; i < kTileBlocks; ++i) {
    if (i >= nmine) break;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int a = bm[i] * 16 + g + ((q & 2) ? 8 : 0), b = bn[i] * 8 + 2 * t + (q & 1);
      if (a < c && b < c && a <= b) partial[(int64_t)blockIdx.x * npairs + packed_ix(a, b, c)] = acc64[i][q];
    }
  }
}

// Q = Z R^-1 (R^-1 upper triangular, f32 c x c row-major in rinv), dQ partials.
__global__ void __launch_bounds__(32 * kTW)
apply_tc_kernel(const float* __restrict__ Z, const float* __restrict__ Qprev, float* __restrict__ Q,
                int64_t n, int64_t ld, int c, const float* __restrict__ rinv,
                double* __restrict__ dq_partial) {
  extern __shared__ __align__(16) float sm[];
  const int ldz = tc_ldz(ld);
  const int cr = (c + 7) / 8 * 8;                       // R^-1 padded to n-blocks
  float* rs = sm;                                       // cr x (cr + 8): row l, col j
  const int ldr = cr + 8;
  float* zt = sm + (size_t)cr * ldr;                    // kTR x ldz
  __shared__ double red[32];
  for (int e = threadIdx.x; e < cr * ldr; e += blockDim.x) {
    const int l = e / ldr, j = e % ldr;
    rs[e] = (l < c && j < c) ? rinv[l * c + j] : 0.f;
  }
  // tile columns [ld, cr) are read by the last k-step: zero once (staging writes [0, ld))
  for (int e = threadIdx.x; e < kTR * (cr > ld ? cr - (int)ld : 0); e += blockDim.x) {
    const int w = cr - (int)ld;
    zt[(e / w) * ldz + ld + e % w] = 0.f;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int nb8 = cr / 8;
  const int ld4 = (int)(ld / 4);
  double dq = 0.0;
  for (int64_t t0 = (int64_t)blockIdx.x * kTR; t0 < n; t0 += (int64_t)gridDim.x * kTR) {
    const int tr = (int)lmin(kTR, n - t0);
    __syncthreads();
    for (int e = threadIdx.x; e < kTR * ld4; e += blockDim.x) {
      const int r = e / ld4, q = e - r * ld4;
      const float4 v = r < tr ? __ldg(reinterpret_cast<const float4*>(Z + (t0 + r) * ld) + q)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(zt + r * ldz + 4 * q) = v;
    }
    __syncthreads();
    const int rw = warp * 16;                           // this warp's 16 rows
    if (rw >= tr) continue;
    const float* za = zt + (rw + g) * ldz;
    const float* zb = za + 8 * ldz;
    for (int nb = 0; nb < nb8; ++nb) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      for (int ks = 0; ks <= nb; ++ks) {                // R^-1[l][j] = 0 for l > j
        uint32_t ah[4], al[4];
        split_tf32(za[ks * 8 + t], ah[0], al[0]);
        split_tf32(zb[ks * 8 + t], ah[1], al[1]);
        split_tf32(za[ks * 8 + t + 4], ah[2], al[2]);
        split_tf32(zb[ks * 8 + t + 4], ah[3], al[3]);
        uint32_t bh0, bl0, bh1, bl1;
        split_tf32(rs[(ks * 8 + t) * ldr + nb * 8 + g], bh0, bl0);
        split_tf32(rs[(ks * 8 + t + 4) * ldr + nb * 8 + g], bh1, bl1);
        mma3(acc, ah, al, bh0, bh1, bl0, bl1);
      }
      // rows rw+g and rw+g+8, columns nb*8 + 2t, +1 (columns >= c are exact
      // zeros: the padding of R^-1 is zero)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = rw + g + 8 * h;
        const int j = nb * 8 + 2 * t;
        if (r >= tr || j >= ld) continue;
        const int64_t row = t0 + r;
        const float o0 = acc[2 * h], o1 = acc[2 * h + 1];
        if (j < c) {
          const double d0 = (double)o0 - (double)Qprev[row * ld + j];
          dq += d0 * d0;
        }
        if (j + 1 < c) {
          const double d1 = (double)o1 - (double)Qprev[row * ld + j + 1];
          dq += d1 * d1;
        }
        if (j + 1 < ld) *reinterpret_cast<float2*>(Q + row * ld + j) = make_float2(o0, o1);
        else Q[row * ld + j] = o0;
      }
    }
    // zero the padding columns past the last n-block
    if (ld > cr)
      for (int e = lane; e < 16 * (int)(ld - cr); e += 32) {
        const int r = rw + e / (int)(ld - cr), j = cr + e % (int)(ld - cr);
        if (r < tr) Q[(t0 + r) * ld + j] = 0.f;
      }
  }
  dq = block_sum(dq, red);
  if (threadIdx.x == 0) dq_partial[blockIdx.x] = dq;
}

int gram_tc(const float* Z, int64_t n, int64_t ld, int c, double* partial, int nblocks,
            cudaStream_t st) {
  const int mb16 = (c + 15) / 16, nb8 = (c + 7) / 8;
  int nblk = 0;
  for (int ma = 0; ma < mb16; ++ma)
    for (int nb = 0; nb < nb8; ++nb) nblk += 16 * ma <= 8 * nb + 7;
  const int ny = (int)ceil_div(nblk, kTW * kTileBlocks);
  const size_t smem = (size_t)kTR * tc_ldz(ld) * sizeof(float);
  ANCKA_REQUIRE(smem <= 227 * 1024, ANCKA_ERR_UNSUPPORTED, "gram_tc: c too large");
  ANCKA_CUDA(cudaFuncSetAttribute(gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  // CTA columns y split the block list; every (x, y) writes disjoint packed entries
  gram_tc_kernel<<<dim3(nblocks, ny), 32 * kTW, smem, st>>>(Z, n, ld, c, partial);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

int apply_tc(const float* Z, const float* Qprev, float* Qout, int64_t n, int64_t ld, int c,
             const float* rinv, double* dq_partial, int nblocks, cudaStream_t st) {
  const int cr = (c + 7) / 8 * 8;
  const size_t smem = ((size_t)cr * (cr + 8) + (size_t)kTR * tc_ldz(ld)) * sizeof(float);
  ANCKA_REQUIRE(smem <= 227 * 1024, ANCKA_ERR_UNSUPPORTED, "apply_tc: c too large");
  ANCKA_CUDA(cudaFuncSetAttribute(apply_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  apply_tc_kernel<<<nblocks, 32 * kTW, smem, st>>>(Z, Qprev, Qout, n, ld, c, rinv, dq_partial);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

}  // namespace ancka
