// Discretisation for wide blocks (k > 16, up to Papers100M's k = 172):
// engine.py:183-263 with the per-round n-sized work on the device and the
// k x k Procrustes step (SVD) on the host, exactly as the reference
// computes it (numpy's SVD of Y~^T Q~).
//
//   ancka_disc_normalize   q~ = q / ||q|| (numpy's pairwise norm), f32 copy
//   ancka_disc_score       scores = q~ R (64-row tiles, 4x4 register blocks),
//                          first-max argmax and second-best margin per row
//   ancka_disc_accumulate  S[l][j] = sum_{i: lab_i = l} q~[i][j] and the
//                          cluster sizes, in 64-bit fixed point: integer sums
//                          are order independent, so the result is
//                          bit-reproducible without a partials pass
//   ancka_disc_proto_pass  acc_i += |q~_i . r|  (prototype start, engine.py:209-218)
#include "common.cuh"

namespace ancka {

constexpr int kDT = 64;           // rows per score tile
constexpr int kDTS = kDT + 4;     // padded stride of the transposed tile

__global__ void disc_normalize_kernel(const float* __restrict__ Q, int64_t ldq, int64_t col0,
                                      int64_t n, int k, float* __restrict__ qt, int64_t ldt,
                                      int* __restrict__ zero_rows) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w0; i < n; i += nw) {
    const float* q = Q + i * ldq + col0;
    double nrm = 0.0;
    if (lane == 0)   // np.linalg.norm(q, axis=1): pairwise sum of q*q in f64
      nrm = sqrt(np_pairwise_sum_g([q](int64_t c) {
        const double v = (double)q[c];
        return __dmul_rn(v, v);
      }, k));
    nrm = __shfl_sync(0xffffffffu, nrm, 0);
    if (lane == 0 && nrm == 0.0) atomicAdd(zero_rows, 1);
    for (int c = lane; c < (int)ldt; c += 32)
      qt[i * ldt + c] = (c < k && nrm > 0.0) ? (float)((double)q[c] / nrm) : 0.f;
  }
}

__global__ void __launch_bounds__(256)
disc_score_kernel(const float* __restrict__ qt, int64_t ldt, int64_t n, int k,
                  const float* __restrict__ R, int64_t ldr, int32_t* __restrict__ labels,
                  float* __restrict__ margin) {
  extern __shared__ __align__(16) float dsm[];
  const int kp = (k + 3) & ~3, nch = kp / 4;
  float* sR = dsm;                                  // k x kp
  float* zt = sR + (size_t)k * kp;                  // kp x kDTS (transposed tile)
  float* cb = zt + (size_t)kp * kDTS;               // kDT x nch best
  float* cs = cb + kDT * nch;                       // kDT x nch second
  int* ci = reinterpret_cast<int*>(cs + kDT * nch); // kDT x nch argmax
  for (int e = threadIdx.x; e < k * kp; e += blockDim.x) {
    const int l = e / kp, j = e - l * kp;
    sR[e] = j < k ? R[(int64_t)l * ldr + j] : 0.f;
  }
  for (int64_t t0 = (int64_t)blockIdx.x * kDT; t0 < n; t0 += (int64_t)gridDim.x * kDT) {
    const int tr = (int)lmin(kDT, n - t0);
    __syncthreads();
    for (int e = threadIdx.x; e < kDT * kp; e += blockDim.x) {
      const int r = e / kp, l = e - r * kp;
      zt[l * kDTS + r] = (r < tr && l < k) ? qt[(t0 + r) * ldt + l] : 0.f;
    }
    __syncthreads();
    for (int pp = threadIdx.x; pp < (kDT / 4) * nch; pp += blockDim.x) {
      const int rg = pp / nch, ch = pp - rg * nch;
      const int r0 = rg * 4, j0 = ch * 4;
      float o[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) o[u][v] = 0.f;
      for (int l = 0; l < k; ++l) {   // same per-entry FMA order as a row dot product
        const float4 z = *reinterpret_cast<const float4*>(zt + l * kDTS + r0);
        const float4 w = *reinterpret_cast<const float4*>(sR + l * kp + j0);
        const float zv[4] = {z.x, z.y, z.z, z.w}, wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) o[u][v] = fmaf(zv[u], wv[v], o[u][v]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float best = -INFINITY, second = -INFINITY;
        int lab = -1;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const float sv = o[u][v];
          if (j0 + v < k) {
            if (sv > best) { second = best; best = sv; lab = j0 + v; }
            else if (sv > second) second = sv;
          }
        }
        cb[(r0 + u) * nch + ch] = best;
        cs[(r0 + u) * nch + ch] = second;
        ci[(r0 + u) * nch + ch] = lab;
      }
    }
    __syncthreads();
    if (threadIdx.x < tr) {     // merge chunks in ascending column order (first max)
      const int r = threadIdx.x;
      float best = cb[r * nch], second = cs[r * nch];
      int lab = ci[r * nch];
      for (int ch = 1; ch < nch; ++ch) {
        const float b2 = cb[r * nch + ch], s2 = cs[r * nch + ch];
        if (b2 > best) { second = fmaxf(best, s2); best = b2; lab = ci[r * nch + ch]; }
        else second = fmaxf(second, b2);
      }
      labels[t0 + r] = lab;
      margin[t0 + r] = k >= 2 ? second : best;
    }
  }
}

// grid (row blocks, column blocks of 32); fixed point value * 2^shift
__global__ void __launch_bounds__(256)
disc_accum_kernel(const float* __restrict__ qt, int64_t ldt, int64_t n, int k,
                  const int32_t* __restrict__ labels, double scale,
                  unsigned long long* __restrict__ S, unsigned long long* __restrict__ counts) {
  extern __shared__ __align__(16) unsigned long long acc[];   // k x 32 (+ k counts)
  unsigned long long* cnt = acc + (size_t)k * 32;
  const int j0 = blockIdx.y * 32;
  const bool do_cnt = blockIdx.y == 0;
  for (int e = threadIdx.x; e < k * 32 + k; e += blockDim.x) acc[e] = 0ull;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int j = j0 + lane;
  const int64_t rpb = ceil_div(n, gridDim.x);
  const int64_t r0 = (int64_t)blockIdx.x * rpb, r1 = lmin(n, r0 + rpb);
  for (int64_t i = r0 + w; i < r1; i += nw) {   // warp per row, lane per column
    const int l = labels[i];
    if (j < k) {
      const long long fx = llrint((double)qt[i * ldt + j] * scale);
      atomicAdd(&acc[l * 32 + lane], (unsigned long long)fx);
    }
    if (do_cnt && lane == 0) atomicAdd(&cnt[l], 1ull);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < k * 32; e += blockDim.x) {
    const int l = e / 32, jj = j0 + (e % 32);
    if (jj < k && acc[e]) atomicAdd(&S[(int64_t)l * k + jj], acc[e]);
  }
  if (do_cnt)
    for (int e = threadIdx.x; e < k; e += blockDim.x)
      if (cnt[e]) atomicAdd(&counts[e], cnt[e]);
}

__global__ void disc_proto_kernel(const float* __restrict__ qt, int64_t ldt, int64_t n, int k,
                                  const double* __restrict__ rcol, double* __restrict__ acc) {
  extern __shared__ double rs[];
  for (int l = threadIdx.x; l < k; l += blockDim.x) rs[l] = rcol[l];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double d = 0.0;
    for (int l = 0; l < k; ++l) d += (double)qt[i * ldt + l] * rs[l];
    acc[i] += fabs(d);
  }
}

}  // namespace ancka

using namespace ancka;

static int disc_grid(int64_t items, int per) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(items, per), 8 * kNumSMs));
}

extern "C" int ancka_disc_normalize(const float* Q, int64_t ldq, int64_t col0, int64_t n,
                                    int32_t k, float* qt, int64_t ldt, int32_t* zero_rows,
                                    ancka_stream_t stream) {
  ANCKA_REQUIRE(Q && qt && zero_rows && k >= 1 && ldt >= k, ANCKA_ERR_ARG, "disc_normalize: bad arguments");
  auto st = as_stream(stream);
  ANCKA_CUDA(cudaMemsetAsync(zero_rows, 0, sizeof(int32_t), st));
  disc_normalize_kernel<<<disc_grid(n * 32, 256), 256, 0, st>>>(Q, ldq, col0, n, k, qt, ldt, zero_rows);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

extern "C" int ancka_disc_score(const float* qt, int64_t ldt, int64_t n, int32_t k, const float* R,
                                int64_t ldr, int32_t* labels, float* margin, ancka_stream_t stream) {
  const int kp = (k + 3) & ~3, nch = kp / 4;
  const size_t smem = sizeof(float) * ((size_t)k * kp + (size_t)kp * kDTS + 3 * (size_t)kDT * nch);
  ANCKA_REQUIRE(k >= 1 && smem <= 227 * 1024, ANCKA_ERR_UNSUPPORTED, "disc_score: k=%d too large", k);
  auto st = as_stream(stream);
  ANCKA_CUDA(cudaFuncSetAttribute(disc_score_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 1;
  ANCKA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, disc_score_kernel, 256, smem));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kDT),
                                                                (int64_t)std::max(per_sm, 1) * kNumSMs));
  disc_score_kernel<<<grid, 256, smem, st>>>(qt, ldt, n, k, R, ldr, labels, margin);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

extern "C" int ancka_disc_accumulate(const float* qt, int64_t ldt, int64_t n, int32_t k,
                                     const int32_t* labels, double scale, int64_t* S,
                                     int64_t* counts, ancka_stream_t stream) {
  const size_t smem = sizeof(unsigned long long) * ((size_t)k * 32 + k);
  ANCKA_REQUIRE(k >= 1 && smem <= 227 * 1024, ANCKA_ERR_UNSUPPORTED, "disc_accumulate: k=%d too large", k);
  auto st = as_stream(stream);
  ANCKA_CUDA(cudaMemsetAsync(S, 0, sizeof(int64_t) * (size_t)k * k, st));
  ANCKA_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * k, st));
  if (smem > 48 * 1024)
    ANCKA_CUDA(cudaFuncSetAttribute(disc_accum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int ny = (k + 31) / 32;
  const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 2048), 2 * kNumSMs));
  disc_accum_kernel<<<dim3(gx, ny), 256, smem, st>>>(
      qt, ldt, n, k, labels, scale, reinterpret_cast<unsigned long long*>(S),
      reinterpret_cast<unsigned long long*>(counts));
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

extern "C" int ancka_disc_proto_pass(const float* qt, int64_t ldt, int64_t n, int32_t k,
                                     const double* rcol, double* acc, ancka_stream_t stream) {
  ANCKA_REQUIRE(qt && rcol && acc && k >= 1, ANCKA_ERR_ARG, "disc_proto_pass: bad arguments");
  auto st = as_stream(stream);
  disc_proto_kernel<<<disc_grid(n, 256), 256, sizeof(double) * k, st>>>(qt, ldt, n, k, rcol, acc);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}
