// Subsystem 4: SVD-based discretisation and argmax label assignment
// (engine.py:162-263) plus the post-pass repair check (engine.py:266-288).
//
// One cooperative persistent kernel runs both alternating-rounding starts
// (identity, prototype; engine.py:247-253) for up to max_iter rounds without
// returning to the host.  Per round:
//   A  every CTA: row-normalise its rows of Q[:, col0:col0+k], score them
//      against R (k x k, shared-memory broadcast), first-max argmax and
//      second-best margin, and add per-cluster column sums of Q~ into a
//      rotating global total in 64-bit fixed point (integer atomics: the sum
//      is independent of order, hence bit-reproducible).  k <= 8: thread per
//      row with direct loads, per-group f64 sums, one atomic per entry and
//      CTA; k > 8: q~ normalised once per call, 3xFP16 warp-MMA scores with
//      a certified margin (uncertified rows rescored exactly in f64), a
//      stable per-tile bucket sort by label and f64 cluster sums per CTA
//      (see phase_accumulate_tc).
//   -- one grid barrier --
//   B  every CTA, redundantly and identically: read M (k x k) and the
//      cluster sizes from the totals; Y~ = Y/size (the reference's 1/size,
//      engine.py:194-198); polar factor R = V U^T of (Y~^T Q~)^T by
//      Newton-Schulz (the SVD's V U^T, engine.py:199-205) and
//      sum(sigma) = tr(R Y~^T Q~); obj = n - 2 sum(sigma); |d obj| < tol.
// Empty clusters (rare) take a slower path with the reference's margin rule
// (engine.py:162-180).  No float atomics: results are bit-reproducible.
#include <cooperative_groups.h>
#include <cstdlib>

#include <cuda_fp16.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace ancka {

constexpr int kDiscThreads = 256;
constexpr int kDiscWideMaxK = 192;
// disc_wide_dev.cu: 64 < k <= 192
size_t discretize_wide_workspace(int64_t n, int k);
int discretize_wide(const float* Q, int64_t ldq, int64_t col0, int64_t n, int k, int max_iter,
                    double tol, int32_t* labels_out, double* info, void* ws, size_t wsb,
                    cudaStream_t st);
// blocks wider than this take the wide path (ANCKA_DISC_WIDE_MIN, >= 8, lets
// tests run it on narrower blocks)
static int disc_wide_min() {
  const char* e = getenv("ANCKA_DISC_WIDE_MIN");
  return e ? std::max(8, atoi(e)) : 64;
}

struct DiscParams {
  const float* Q;
  int64_t ldq, col0, n;
  int k, max_iter;
  double tol;
  int32_t* labels;      // working labels (output of the current run)
  int32_t* labels_run0; // saved labels of run 0
  float* margin;        // n, second-best score
  double* proto_acc;    // n, prototype accumulator
  int64_t* part_cnt;    // 2 x grid x k
  double* part_arg;     // 2 x grid x 3  (value, index, label)
  double* Rg;           // k x k f64 rotation (row l, col j), written by CTA 0
  unsigned long long* gfx;  // 3 x (k x k + k) fixed-point totals, rotating
  double fx_scale;          // 2^s with n * 2^s < 2^62
  double* info;         // output info
  unsigned long long* tdbg;  // optional phase timing (ANCKA_DISC_TIMING)
  int groups;           // accumulator groups per CTA
  int run_lo, run_hi;   // alternating-rounding starts handled by this launch
  double* fin;          // split launches: per-run (obj, rounds, conv, empties)
  float* qn;            // k > 8: normalised block q~ (n x kq, f32, zero padded)
  double* qinv;         // k > 8: 1 / ||q_i|| (0 for all-zero rows)
  int dbuf;             // k > 8: double-buffered row tiles (when shared memory allows)
  double* key;          // k > 8: per row, drift level below which its label is certified
  int32_t* rid;         // k > 8: rows to score this round (per-CTA slices)
};

// Row i of Q[:, col0:col0+k], normalised in f64 (engine.py:226-232) and
// rounded to f32 for scoring / accumulation.
template <int KMAX>
__device__ __forceinline__ void load_row_f(const DiscParams& p, int64_t i, float* qf, double& nrm) {
  const float* src = p.Q + i * p.ldq + p.col0;
  double s = 0.0;
#pragma unroll
  for (int l = 0; l < KMAX; ++l) {
    const double v = l < p.k ? (double)src[l] : 0.0;
    s += v * v;
  }
  nrm = sqrt(s);
  const double inv = nrm > 0 ? 1.0 / nrm : 0.0;
#pragma unroll
  for (int l = 0; l < KMAX; ++l) qf[l] = l < p.k ? (float)((double)src[l] * inv) : 0.f;
}

template <int KMAX>
__device__ __forceinline__ void load_row(const DiscParams& p, int64_t i, double* q, double& nrm) {
  double s = 0.0;
#pragma unroll
  for (int l = 0; l < KMAX; ++l) {
    double v = 0.0;
    if (l < p.k) v = (double)p.Q[i * p.ldq + p.col0 + l];
    q[l] = v;
    s += v * v;
  }
  nrm = sqrt(s);
  const double inv = nrm > 0 ? 1.0 / nrm : 0.0;
#pragma unroll
  for (int l = 0; l < KMAX; ++l) q[l] *= inv;
}

__host__ __device__ __forceinline__ int kpad4(int k) { return (k + 3) & ~3; }

struct Rows {
  int64_t r0, r1;
};
__device__ __forceinline__ Rows my_rows(int64_t n) {
  const int64_t rpb = ceil_div(n, gridDim.x);
  const int64_t r0 = (int64_t)blockIdx.x * rpb;
  return {r0, lmin(n, r0 + rpb)};
}

// Phase A for k <= 8.  score=true: labels + margins from R; false: keep
// labels.  Thread per row (direct loads), per-group f64 column sums in fixed
// row order, then one fixed-point atomic per entry into `gdst`.
template <int KMAX>
__device__ void phase_accumulate(const DiscParams& p, const float* sR, float* tile, int* tlab,
                                 double* acc, int* cnt, bool score, int* zeros_out,
                                 unsigned long long* gdst) {
  const int k = p.k;
  const int G = p.groups;
  for (int e = threadIdx.x; e < G * k * k; e += blockDim.x) acc[e] = 0.0;
  for (int e = threadIdx.x; e < G * k; e += blockDim.x) cnt[e] = 0;
  __syncthreads();
  const Rows R = my_rows(p.n);
  int zeros = 0;
  for (int64_t t0 = R.r0; t0 < R.r1; t0 += kDiscThreads) {
    const int64_t i = t0 + threadIdx.x;
    if (i < R.r1) {
      double nrm;
      float qf[KMAX];
      load_row_f<KMAX>(p, i, qf, nrm);
      if (nrm == 0.0) ++zeros;
      int lab;
      if (score) {
        // scores = q~ R: four columns per pass from a padded float4 rotation
        const int kp = kpad4(k);
        float best = -INFINITY, second = -INFINITY;
        lab = 0;
        for (int j0 = 0; j0 < k; j0 += 4) {
          float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
          for (int l = 0; l < KMAX; ++l)
            if (l < k) {
              const float4 r = *reinterpret_cast<const float4*>(sR + l * kp + j0);
              s0 = fmaf(qf[l], r.x, s0);
              s1 = fmaf(qf[l], r.y, s1);
              s2 = fmaf(qf[l], r.z, s2);
              s3 = fmaf(qf[l], r.w, s3);
            }
          const float sc[4] = {s0, s1, s2, s3};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float s = sc[u];
            if (j0 + u < k) {
              if (s > best) { second = best; best = s; lab = j0 + u; }
              else if (s > second) second = s;
            }
          }
        }
        p.labels[i] = lab;
        p.margin[i] = k >= 2 ? second : best;
      } else {
        lab = p.labels[i];
      }
#pragma unroll
      for (int l = 0; l < KMAX; ++l)
        if (l < k) tile[threadIdx.x * k + l] = qf[l];
      tlab[threadIdx.x] = lab;
    }
    __syncthreads();
    const int tr = (int)lmin(kDiscThreads, R.r1 - t0);
    const int t = threadIdx.x;
    if (t < G * k) {
      const int j = t % k, g = t / k;
      double* a = acc + (size_t)g * k * k;
      int* cg_ = cnt + g * k;                 // column-0 owners also count members
      for (int r = g; r < tr; r += G) {
        const int l = tlab[r];
        a[l * k + j] += (double)tile[r * k + j];
        if (j == 0) cg_[l] += 1;
      }
    }
    __syncthreads();
  }
  // one fixed-point atomic per entry (integer sums: order free)
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    double s = 0.0;
    for (int g = 0; g < G; ++g) s += acc[(size_t)g * k * k + e];
    atomicAdd(gdst + e, (unsigned long long)(long long)llrint(s * p.fx_scale));
  }
  for (int e = threadIdx.x; e < k; e += blockDim.x) {
    int s = 0;
    for (int g = 0; g < G; ++g) s += cnt[g * k + e];
    atomicAdd(gdst + k * k + e, (unsigned long long)s);
  }
  if (zeros_out) {
    __shared__ int zsum;
    if (threadIdx.x == 0) zsum = 0;
    __syncthreads();
    atomicAdd(&zsum, zeros);
    __syncthreads();
    if (threadIdx.x == 0) *zeros_out = zsum;   // reduced over CTAs via part_cnt below
  }
  __syncthreads();
}

// kernel instance: k <= 8, else the column window width (>= off + k)
__host__ __device__ constexpr int disc_kmax(int k, int off) {
  return k <= 8 ? 8 : off + k <= 16 ? 16 : off + k <= 32 ? 32 : off + k <= 48 ? 48
                    : off + k <= 64 ? 64 : 68;
}
__host__ __device__ constexpr int win_kw(int kmax) { return kmax; }
__host__ __device__ constexpr int win_sw(int kmax) {
  return ((win_kw(kmax) / 4) % 2 == 1) ? win_kw(kmax) : win_kw(kmax) + 4;
}
// scoring-rotation and row-tile bytes of the k (<= 8 : > 8) layouts
__host__ __device__ inline size_t disc_rot_bytes(int k, int off) {
  (void)off;
  return k <= 8 ? (size_t)k * kpad4(k) * 4
                : align_dev((size_t)((k + 15) / 16) * (((k + 15) & ~15) / 8) * 32 * 16) + (size_t)k * k * 8;
}
// k > 8 phase-A layout: group accumulators | group counts | tile | tile labels
__host__ __device__ inline size_t disc_tc_tile_bytes(int k, int off, int dbuf = 1) {
  const size_t tc = (dbuf ? 2 : 1) * (size_t)kDiscThreads * (((k + 15) & ~15) + 4) * 4;
  const size_t win = (dbuf ? 2 : 1) * (size_t)kDiscThreads * 4 * win_sw(disc_kmax(k, off));
  return tc > win ? tc : win;
}
__host__ __device__ inline size_t disc_tc_acc_bytes(int k, int G) {
  return (size_t)G * k * ((k + 15) & ~15) * 8;
}
__host__ __device__ inline size_t disc_tile_bytes(int k, int off) {
  return (size_t)kDiscThreads * 4 * (k <= 8 ? k : win_sw(disc_kmax(k, off)));
}

// ---- k > 8 layout.  A thread owns one row and reads it from a staged tile
// as float4s: the window of KW = KMAX columns starting at the aligned column
// c0 = col0 & ~3 holds Q[i, col0:col0+k] at offset off = col0 - c0 (the
// instance is chosen with off + k <= KMAX).
// Tile rows are SW floats apart with SW / 4 odd, so the eight 16-byte reads
// of a quarter warp hit distinct bank groups.  The scoring rotation is
// stored shifted by `off` in the same window coordinates (zero outside the
// k valid rows), so no runtime column index reaches a register array.
template <int KMAX>
struct Win {
  static constexpr int KW = win_kw(KMAX);
  static constexpr int SW = win_sw(KMAX);
};

// Stage rows [t0, t0 + tr) of Q's column window into tile (async copies,
// one commit group).
__device__ __forceinline__ void stage_window_issue(const DiscParams& p, int64_t t0, int tr,
                                                   float* tile, int SW, bool vec) {
  const int k = p.k, off = (int)(p.col0 & 3);
  const int64_t c0 = p.col0 - off;
  if (vec) {   // 16-byte chunks of the aligned window
    const int w4 = (off + k + 3) >> 2, ne = tr * w4;
    const int dr = kDiscThreads / w4, dc = kDiscThreads % w4;
    int r = threadIdx.x / w4, c = threadIdx.x % w4;
    for (int e = threadIdx.x; e < ne; e += kDiscThreads) {
      const float* src = p.Q + (t0 + r) * p.ldq + c0 + 4 * c;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(tile + r * SW + 4 * c)),
                   "l"(src)
                   : "memory");
      r += dr;
      c += dc;
      if (c >= w4) { c -= w4; ++r; }
    }
  } else {     // unaligned rows: 4-byte copies of the k valid columns
    const int ne = tr * k, dr = kDiscThreads / k, dl = kDiscThreads % k;
    int r = threadIdx.x / k, l = threadIdx.x % k;
    for (int e = threadIdx.x; e < ne; e += kDiscThreads) {
      const float* src = p.Q + (t0 + r) * p.ldq + p.col0 + l;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(tile + r * SW + off + l)),
                   "l"(src)
                   : "memory");
      r += dr;
      l += dl;
      if (l >= k) { l -= k; ++r; }
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// This thread's row from the staged tile: raw[m] = Q[i, c0 + m] inside the
// valid window [off, off + k), zero elsewhere.
template <int KMAX>
__device__ __forceinline__ void load_window(const float* rowp, int off, int k,
                                            float (&raw)[Win<KMAX>::KW]) {
  constexpr int KW = Win<KMAX>::KW;
#pragma unroll
  for (int m4 = 0; m4 < KW / 4; ++m4) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (4 * m4 < off + k) v = *reinterpret_cast<const float4*>(rowp + 4 * m4);
    raw[4 * m4 + 0] = v.x;
    raw[4 * m4 + 1] = v.y;
    raw[4 * m4 + 2] = v.z;
    raw[4 * m4 + 3] = v.w;
  }
#pragma unroll
  for (int m = 0; m < KW; ++m) raw[m] = (m >= off && m < off + k) ? raw[m] : 0.f;
}


// ---- k > 8: tensor-core scoring.  The block is normalised once per call
// into q~ (f32, kq = 8 ceil(k / 8) columns, zero padded); each round scores a
// staged 256-row tile against R with warp-level TF32 MMAs in three products
// (q_hi R_hi + q_hi R_lo + q_lo R_hi, hi = rna_tf32(x), lo = x - hi), which
// carries the f32 scoring error of the SIMT path (~2^-22 relative per
// product, f32 accumulation).  A quad of lanes owns a row; the first-max
// argmax and the second-best margin are merged by two shuffles.  The
// cluster sums M[label][j] go to NG group-private 64-bit fixed-point
// accumulators in shared memory (plain adds: each (label, column) cell of a
// group has one owner thread), folded into the global totals by integer
// atomics (order-free: bit-reproducible).
__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], float b0, float b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(__float_as_uint(b0)),
        "r"(__float_as_uint(b1)));
}
// q~ columns padded to the MMA K step (16); n-blocks of 8 output columns
__device__ __forceinline__ void mma_f16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__host__ __device__ constexpr int disc_kq(int k) { return (k + 15) & ~15; }
__host__ __device__ constexpr int disc_nbmax(int kmax) { return disc_kq(kmax >= 64 ? 64 : kmax) / 8; }

// R as per-lane FP16 B fragments (m16n8k16), split R = hi + lo:
// sRf[(ks * nb8 + nb) * 32 + lane] = (hi pair 0, hi pair 1, lo pair 0, lo pair 1),
// pair 0 = (R[16ks+2t][8nb+g], R[16ks+2t+1][8nb+g]), pair 1 = rows + 8,
// g = lane / 4, t = lane % 4; followed by R in f64 (row l, col j).
__host__ __device__ inline size_t disc_frag_bytes(int k) {
  return align_dev((size_t)(disc_kq(k) / 16) * (disc_kq(k) / 8) * 32 * 16);
}
__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
// x = hi + lo with hi = fp16(x), lo = fp16(x - hi) for an element pair
__device__ __forceinline__ void split_half2(float a, float b, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(a, b);
  const float2 hf = __half22float2(h);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = pack_half2(a - hf.x, b - hf.y);
}
template <typename Get>
__device__ __forceinline__ void store_rot_frag(unsigned char* base, int k, Get get) {
  const int ks16 = disc_kq(k) / 16, nb8 = disc_kq(k) / 8;
  uint4* sRf = reinterpret_cast<uint4*>(base);
  double* sR64 = reinterpret_cast<double*>(base + disc_frag_bytes(k));
  for (int e = threadIdx.x; e < ks16 * nb8 * 32; e += blockDim.x) {
    const int lane = e & 31, f = e >> 5, ks = f / nb8, nb = f % nb8;
    const int g = lane >> 2, t = lane & 3, j = nb * 8 + g;
    float r[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int l = ks * 16 + 2 * t + (q & 1) + ((q & 2) ? 8 : 0);
      r[q] = (l < k && j < k) ? (float)get(l, j) : 0.f;
    }
    uint4 v;
    split_half2(r[0], r[1], v.x, v.z);
    split_half2(r[2], r[3], v.y, v.w);
    sRf[e] = v;
  }
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) sR64[e] = get(e / k, e % k);
}

// q~ = Q[:, col0:col0+k] / ||.|| for this CTA's rows (warp per row, lanes
// over columns), 1/||q_i|| kept for the prototype start; returns zero rows.
__device__ int normalize_rows(const DiscParams& p) {
  const int k = p.k, kq = disc_kq(k);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const Rows R = my_rows(p.n);
  int zeros = 0;
  for (int64_t i = R.r0 + warp; i < R.r1; i += nw) {
    const float* src = p.Q + i * p.ldq + p.col0;
    const double v0 = lane < k ? (double)src[lane] : 0.0;
    const double v1 = lane + 32 < k ? (double)src[lane + 32] : 0.0;
    const double nrm = sqrt(warp_sum(v0 * v0 + v1 * v1));
    const double inv = nrm > 0 ? 1.0 / nrm : 0.0;
    float* dst = p.qn + i * kq;
    if (lane < kq) dst[lane] = (float)(v0 * inv);
    if (lane + 32 < kq) dst[lane + 32] = (float)(v1 * inv);
    if (lane == 0) {
      p.qinv[i] = inv;
      zeros += nrm == 0.0;
    }
  }
  return zeros;
}

// Certified argmax.  Scores are 3xTF32 products (q_hi R_hi + q_hi R_lo +
// q_lo R_hi, hi = rna_tf32(x), lo = x - hi truncated by the MMA): per
// product error <= 2^-20 |q||R|, plus f32 accumulation of 3k terms, so for a
// unit row and an orthogonal R every score is within 1e-5 of the f64 score
// of the same f32 iterate.  When the winner beats the runner-up by more than
// kCert = 2e-5 the f64 winner is the same column; rows below the margin
// (exact ties, near-ties) are rescored in f64 by one warp each: q~ = Q_i /
// ||Q_i||, R in f64, first max -- the reference's f64 argmax (engine.py:192)
// on this iterate.  Margins (second-best scores) of certified rows stay
// 3xTF32 values; the rare empty-cluster reseed rescores every row first.
constexpr float kCert = 2e-5f;

// One warp: f64 scores of row i against R, first-max argmax and the
// second-best value (all lanes return them).  qw: 64 doubles of scratch.
__device__ __forceinline__ void score_row_exact_warp(const DiscParams& p, const double* sR64,
                                                     int64_t i, double* qw, int& lab,
                                                     float& second_out, double* margin_out = nullptr) {
  const int k = p.k, lane = threadIdx.x & 31;
  const float* src = p.Q + i * p.ldq + p.col0;
  const double inv = p.qinv[i];
  if (lane < k) qw[lane] = (double)src[lane] * inv;
  if (lane + 32 < k) qw[lane + 32] = (double)src[lane + 32] * inv;
  __syncwarp();
  double s0 = 0.0, s1 = 0.0;
  for (int l = 0; l < k; ++l) {
    const double ql = qw[l];
    if (lane < k) s0 = fma(ql, sR64[l * k + lane], s0);
    if (lane + 32 < k) s1 = fma(ql, sR64[l * k + lane + 32], s1);
  }
  double best = lane < k ? s0 : -INFINITY, second = -INFINITY;
  int bi = lane;
  if (lane + 32 < k) {
    if (s1 > best) { second = best; best = s1; bi = lane + 32; }
    else second = s1;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const double os = __shfl_xor_sync(0xffffffffu, second, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    const bool take = ob > best || (ob == best && oi < bi);
    second = fmax(fmax(second, os), take ? best : ob);
    best = take ? ob : best;
    bi = take ? oi : bi;
  }
  lab = bi;
  second_out = (float)second;
  if (margin_out) *margin_out = best - second;
  __syncwarp();
}

// round(x * 2^sh) to int64 (round half to even, as __float2ll_rn of the
// exact product) with integer operations only: the 64-bit float->int
// conversion is a slow path on sm_100.  |x| <= 1 and sh <= 61.
__device__ __forceinline__ long long fx_round(float x, int sh) {
  const uint32_t b = __float_as_uint(x);
  const int e = (int)((b >> 23) & 0xffu);
  const uint32_t m = (b & 0x7fffffu) | 0x800000u;
  const int s = e - 150 + sh;                // x * 2^sh = m * 2^s (normal x)
  long long v;
  if (e == 0 || s <= -25) {
    v = 0;                                   // |x * 2^sh| < 1/2 (or zero / subnormal x)
  } else if (s >= 0) {
    v = (long long)m << s;
  } else {
    const int r = -s;
    const uint32_t q = m >> r, rem = m & ((1u << r) - 1u), half = 1u << (r - 1);
    v = (long long)(q + ((rem > half || (rem == half && (q & 1u))) ? 1u : 0u));
  }
  return (b >> 31) ? -v : v;
}

// 64-bit add to a shared-memory cell (lo, hi words) with two native 32-bit
// atomics: the low-word atomic's old value gives this add's carry, so the
// cell is exact mod 2^64 under any interleaving (the 64-bit shared atomic
// is a compare-and-swap loop on sm_100)
__device__ __forceinline__ void sadd64(unsigned* cell, long long v) {
  const unsigned lo = (unsigned)v, hi = (unsigned)((unsigned long long)v >> 32);
  const unsigned old = atomicAdd(cell, lo);
  const unsigned h = hi + ((old + lo < old) ? 1u : 0u);
  if (h) atomicAdd(cell + 1, h);
}

template <int KMAX>
__device__ void phase_accumulate_tc(const DiscParams& p, const uint4* sRf, const double* sR64,
                                    float* tile, int* tlab, long long* gacc, int* gcnt, bool score,
                                    unsigned long long* gdst, const unsigned long long* gprev,
                                    double cdrift, bool keys_valid) {
  constexpr int NBM = disc_nbmax(KMAX);
  const int k = p.k, kk = k * k, kq = disc_kq(k), ks16 = kq / 16, nb8 = kq / 8;
  const int SWQ = kq + 4;
  const size_t tile_floats = p.dbuf ? (size_t)kDiscThreads * SWQ : 0;
  int* flagged = tlab + 3 * kDiscThreads + 68 + 64;   // kDiscThreads
  double* wq = reinterpret_cast<double*>(flagged + kDiscThreads);   // 8 warps x 64, 16-B aligned
  int* wcnt = flagged + kDiscThreads + 2 * 8 * 64;    // 8 warps x 64 labels (after wq)
  int* told = wcnt + 8 * 64;                          // kDiscThreads
  int* tids = told + kDiscThreads;                    // kDiscThreads: row of each tile slot
  __shared__ int s_nflag, s_cnt;
  // Cluster sums in 64-bit fixed point, element by element (fx_round: the
  // same integer for the same q~ entry every round), so totals can be
  // carried: a round after the first adds only the rows whose label moved
  // (-fx to the old cluster, +fx to the new one) to the previous round's
  // totals, and the result is the exact integer a full recount gives.
  // gprev == nullptr: full recount (first round of a start, after a reseed).
  const bool full = gprev == nullptr;
  const int sh = ilogb(p.fx_scale);
  // tile labels, within-bucket ranks, entry permutation, bucket offsets and
  // sizes, rows to rescore exactly, rescoring scratch, per-warp counts,
  // labels before this round's scoring
  int* trank = tlab + kDiscThreads;
  int* perm = trank + kDiscThreads;
  int* boff = perm + kDiscThreads;        // k + 1 (68 slots)
  int* bcnt = boff + 68;                  // k (64 slots)
  (void)bcnt;
  __shared__ int s_nchg;
  for (int e = threadIdx.x; e < k * kq; e += blockDim.x) gacc[e] = 0;
  for (int e = threadIdx.x; e < k; e += blockDim.x) gcnt[e] = 0;
  if (!full)   // carry: this CTA's slice of the previous totals
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < kk + k;
         e += (int64_t)gridDim.x * blockDim.x) {
      const unsigned long long v = __ldcg(gprev + e);
      if (v) atomicAdd(gdst + e, v);
    }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const bool dbg = p.tdbg && blockIdx.x == 0 && threadIdx.x == 0;
  const bool dbg0 = p.tdbg && blockIdx.x == 0 && threadIdx.x == 0;
  const Rows R = my_rows(p.n);
  // Rows to score.  A row scored when the cumulative rotation drift was C0
  // with a certified margin m keeps its argmax while the drift since then
  // stays below m / 2 (|q~ (R' - R)_j| <= max_j ||R'_j - R_j|| per score,
  // unit rows): key = C0 + m / 2, and it is scored again only once the
  // drift cdrift reaches its key.  Until the keys of this start exist, or
  // when most rows are due, every row is scored.
  int64_t nrows = R.r1 - R.r0;
  bool list = false;
  if (score && keys_valid) {
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    for (int64_t i0 = R.r0; i0 < R.r1; i0 += kDiscThreads) {
      const int64_t i = i0 + threadIdx.x;
      const bool due = i < R.r1 && p.key[i] <= cdrift;
      const unsigned m = __ballot_sync(0xffffffffu, due);
      int base = 0;
      if (lane == 0 && m) base = atomicAdd(&s_cnt, __popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (due) p.rid[R.r0 + base + __popc(m & ((1u << lane) - 1u))] = (int32_t)i;
    }
    __syncthreads();
    if (2 * (int64_t)s_cnt <= nrows) {
      list = true;
      nrows = s_cnt;
    }
    if (dbg0) p.tdbg[11] += (unsigned long long)(R.r1 - R.r0 - nrows);   // rows skipped
  }
  const int ntile = (int)ceil_div(nrows, (int64_t)kDiscThreads);
  const int c4 = kq / 4;
  auto slot_id = [&](int ti) -> int64_t {    // row of this thread's slot in tile ti
    const int64_t pos = (int64_t)ti * kDiscThreads + threadIdx.x;
    if (pos >= nrows) return -1;
    return list ? (int64_t)p.rid[R.r0 + pos] : R.r0 + pos;
  };
  auto stage = [&](int ti, int64_t my_id) {   // 16-byte async copies of tile ti into buffer ti & 1
    if (list) {   // gathered rows: each thread copies its own slot's row
      float* dst = tile + (ti & 1) * tile_floats + threadIdx.x * SWQ;
      if (my_id >= 0)
        for (int c = 0; c < c4; ++c)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                           (uint32_t)__cvta_generic_to_shared(dst + 4 * c)),
                       "l"(p.qn + my_id * kq + 4 * c)
                       : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
      return;
    }
    const int64_t t0 = R.r0 + (int64_t)ti * kDiscThreads;
    const int tr = (int)lmin(kDiscThreads, R.r1 - t0);
    float* dst = tile + (ti & 1) * tile_floats;
    const int ne = tr * c4, dr = kDiscThreads / c4, dc = kDiscThreads % c4;
    int r = threadIdx.x / c4, c = threadIdx.x % c4;
    for (int e = threadIdx.x; e < ne; e += kDiscThreads) {
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(dst + r * SWQ + 4 * c)),
                   "l"(p.qn + (t0 + r) * kq + 4 * c)
                   : "memory");
      r += dr;
      c += dc;
      if (c >= c4) { c -= c4; ++r; }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  long long c_prev = dbg ? clock64() : 0;
#define SUBSTAMP(slot)                                  \
  do {                                                  \
    if (dbg) {                                          \
      const long long _c = clock64();                   \
      p.tdbg[(slot)] += (unsigned long long)(_c - c_prev); \
      c_prev = _c;                                      \
    }                                                   \
  } while (0)
  // slot rows and their labels before this round, read ahead (latency off
  // the scoring path)
  int64_t id_cur = slot_id(0), id_nxt = slot_id(1);
  int old_cur = (!full && id_cur >= 0) ? __ldcg(p.labels + id_cur) : -1;
  if (ntile > 0 && p.dbuf) stage(0, id_cur);
  for (int ti = 0; ti < ntile; ++ti) {
    const int tr = (int)lmin(kDiscThreads, nrows - (int64_t)ti * kDiscThreads);
    told[threadIdx.x] = old_cur;
    tids[threadIdx.x] = (int)id_cur;
    const int64_t id_nn = slot_id(ti + 2);
    const int old_nxt = (!full && id_nxt >= 0) ? __ldcg(p.labels + id_nxt) : -1;
    if (!p.dbuf) {
      stage(ti, id_cur);
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    } else if (ti + 1 < ntile) {
      stage(ti + 1, id_nxt);               // overlaps this tile's work
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    if (threadIdx.x == 0) s_nflag = 0;
    __syncthreads();
    SUBSTAMP(8);
    const float* tl = tile + (ti & 1) * tile_floats;
    if (score) {
      if (warp * 32 < tr) {
        float acc[2][NBM][4];
#pragma unroll
        for (int mb = 0; mb < 2; ++mb)
#pragma unroll
          for (int nb = 0; nb < NBM; ++nb)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[mb][nb][c] = 0.f;
        const float* wt = tl + warp * 32 * SWQ;
#pragma unroll 1
        for (int ks = 0; ks < ks16; ++ks) {
          uint32_t ah[2][4], al[2][4];
#pragma unroll
          for (int mb = 0; mb < 2; ++mb)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float2 x = *reinterpret_cast<const float2*>(
                  wt + (mb * 16 + g + ((q & 1) ? 8 : 0)) * SWQ + ks * 16 + 2 * t + ((q & 2) ? 8 : 0));
              split_half2(x.x, x.y, ah[mb][q], al[mb][q]);
            }
#pragma unroll
          for (int nb = 0; nb < NBM; ++nb) {
            if (nb < nb8) {
              const uint4 b = sRf[(ks * nb8 + nb) * 32 + lane];
#pragma unroll
              for (int mb = 0; mb < 2; ++mb) {
                mma_f16(acc[mb][nb], ah[mb], b.x, b.y);
                mma_f16(acc[mb][nb], ah[mb], b.z, b.w);
                mma_f16(acc[mb][nb], al[mb], b.x, b.y);
              }
            }
          }
        }
#pragma unroll
        for (int mb = 0; mb < 2; ++mb)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float best = -INFINITY, second = -INFINITY;
            int bi = 0x7fffffff;
#pragma unroll
            for (int nb = 0; nb < NBM; ++nb)
#pragma unroll
              for (int c = 0; c < 2; ++c) {
                const int j = nb * 8 + 2 * t + c;
                const float v = (nb < nb8 && j < k) ? acc[mb][nb][h * 2 + c] : -INFINITY;
                second = fmaxf(second, fminf(best, v));
                bi = v > best ? j : bi;
                best = fmaxf(best, v);
              }
#pragma unroll
            for (int o = 1; o <= 2; o <<= 1) {
              const float ob = __shfl_xor_sync(0xffffffffu, best, o);
              const float os = __shfl_xor_sync(0xffffffffu, second, o);
              const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
              const bool take = ob > best || (ob == best && oi < bi);
              second = fmaxf(fmaxf(second, os), take ? best : ob);
              best = take ? ob : best;
              bi = take ? oi : bi;
            }
            const int row = warp * 32 + mb * 16 + g + h * 8;
            if (t == 0 && row < tr) {
              const int64_t id = tids[row];
              if (!(best - second > kCert)) flagged[atomicAdd(&s_nflag, 1)] = row;
              else p.key[id] = cdrift + 0.5 * ((double)best - (double)second - (double)kCert);
              p.labels[id] = bi;
              tlab[row] = bi;
            }
          }
      }
      __syncthreads();
      SUBSTAMP(9);
      if (dbg) p.tdbg[14] += s_nflag;
      // exact f64 rescoring (a warp per row) of the rows the margin does not certify
      for (int f = warp; f < s_nflag; f += kDiscThreads / 32) {
        const int row = flagged[f];
        const int64_t id = tids[row];
        int lab;
        float second;
        double marg;
        score_row_exact_warp(p, sR64, id, wq + warp * 64, lab, second, &marg);
        if (lane == 0) {
          p.labels[id] = lab;
          p.key[id] = cdrift + 0.5 * marg;
          tlab[row] = lab;
        }
      }
    } else {
      for (int r = threadIdx.x; r < tr; r += blockDim.x) tlab[r] = p.labels[tids[r]];
    }
    __syncthreads();
    SUBSTAMP(10);
    // rows whose cluster changed (every row in a full recount)
    if (threadIdx.x == 0) s_nchg = 0;
    __syncthreads();
    {   // one shared atomic per warp: ballot, then ranks within the warp
      const bool mv = threadIdx.x < tr && tlab[threadIdx.x] != told[threadIdx.x];
      const unsigned m = __ballot_sync(0xffffffffu, mv);
      int base = 0;
      if (lane == 0 && m) base = atomicAdd(&s_nchg, __popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (mv) perm[base + __popc(m & ((1u << lane) - 1u))] = threadIdx.x;
    }
    __syncthreads();
    if (dbg) p.tdbg[13] += s_nchg;
    // a warp per changed row, lanes over columns: +fx to the new cluster,
    // -fx to the old one (shared 64-bit atomics; integers: order free)
    for (int c = warp; c < s_nchg; c += kDiscThreads / 32) {
      const int r = perm[c], l = tlab[r], o = told[r];
      const float* row = tl + r * SWQ;
      unsigned* acc = reinterpret_cast<unsigned*>(gacc);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        if (j < k) {
          const long long fx = fx_round(row[j], sh);
          if (fx != 0) {
            sadd64(acc + 2 * (l * kq + j), fx);
            if (o >= 0) sadd64(acc + 2 * (o * kq + j), -fx);
          }
        }
      }
      if (lane == 0) {
        atomicAdd(&gcnt[l], 1);
        if (o >= 0) atomicAdd(&gcnt[o], -1);
      }
    }
    __syncthreads();
    SUBSTAMP(12);
    id_cur = id_nxt;
    old_cur = old_nxt;
    id_nxt = id_nn;
  }
#undef SUBSTAMP
  // CTA deltas -> global totals (integer atomics: order free)
  for (int e = threadIdx.x; e < kk; e += blockDim.x) {
    const int l = e / k, j = e - l * k;
    const long long v = gacc[l * kq + j];
    if (v != 0) atomicAdd(gdst + e, (unsigned long long)v);
  }
  for (int e = threadIdx.x; e < k; e += blockDim.x)
    if (gcnt[e] != 0) atomicAdd(gdst + kk + e, (unsigned long long)(long long)gcnt[e]);
  __syncthreads();
}

// Exact (f64) second-best scores of every row of this CTA, before the rare
// empty-cluster reseed picks the largest margin (engine.py:170-179).  A
// thread per row: q~_i in registers, R in shared memory (broadcast reads),
// two score columns per pass; each score sums l = 0..k-1 in order, the same
// f64 values as score_row_exact_warp.
template <int KMAX>
__device__ void exact_margins(const DiscParams& p, const double* sR64) {
  const Rows R = my_rows(p.n);
  const int k = p.k;
  for (int64_t i = R.r0 + threadIdx.x; i < R.r1; i += blockDim.x) {
    const float* src = p.Q + i * p.ldq + p.col0;
    const double inv = p.qinv[i];
    double q[KMAX];
#pragma unroll
    for (int l = 0; l < KMAX; ++l) q[l] = l < k ? (double)src[l] * inv : 0.0;
    double best = -INFINITY, second = -INFINITY;
    for (int j = 0; j < k; j += 2) {
      const bool two = j + 1 < k;
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int l = 0; l < KMAX; ++l)
        if (l < k) {
          s0 = fma(q[l], sR64[l * k + j], s0);
          if (two) s1 = fma(q[l], sR64[l * k + j + 1], s1);
        }
      if (s0 > best) { second = best; best = s0; } else if (s0 > second) second = s0;
      if (two) {
        if (s1 > best) { second = best; best = s1; } else if (s1 > second) second = s1;
      }
    }
    p.margin[i] = (float)second;
  }
  __syncthreads();
}

__device__ void reduce_arg(const double* part, int nb, bool want_max, double& v_out,
                           long long& i_out, int& lab_out, double* sv, long long* si, int* sl) {
  double v = 0.0;
  long long id = -1;
  int lb = 0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    const long long i2 = (long long)part[b * 3 + 1];
    const double v2 = part[b * 3];
    const bool take = i2 >= 0 && (id < 0 || (want_max ? v2 > v : v2 < v) || (v2 == v && i2 < id));
    if (take) { v = v2; id = i2; lb = (int)part[b * 3 + 2]; }
  }
  sv[threadIdx.x] = v;
  si[threadIdx.x] = id;
  sl[threadIdx.x] = lb;
  __syncthreads();
  for (int s = kDiscThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double v2 = sv[threadIdx.x + s];
      const long long i2 = si[threadIdx.x + s];
      const double v1 = sv[threadIdx.x];
      const long long i1 = si[threadIdx.x];
      const bool take = i2 >= 0 && (i1 < 0 || (want_max ? v2 > v1 : v2 < v1) || (v2 == v1 && i2 < i1));
      if (take) { sv[threadIdx.x] = v2; si[threadIdx.x] = i2; sl[threadIdx.x] = sl[threadIdx.x + s]; }
    }
    __syncthreads();
  }
  v_out = sv[0];
  i_out = si[0];
  lab_out = sl[0];
  __syncthreads();
}

// CTA-local first-max/first-min (value, index, label) -> part[blockIdx]
__device__ void block_arg(double v, long long id, int lab, bool want_max, double* part,
                          double* sv, long long* si, int* sl) {
  sv[threadIdx.x] = v;
  si[threadIdx.x] = id;
  sl[threadIdx.x] = lab;
  __syncthreads();
  for (int s = kDiscThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double v2 = sv[threadIdx.x + s];
      const long long i2 = si[threadIdx.x + s];
      const double v1 = sv[threadIdx.x];
      const long long i1 = si[threadIdx.x];
      const bool take = i2 >= 0 && (i1 < 0 || (want_max ? v2 > v1 : v2 < v1) || (v2 == v1 && i2 < i1));
      if (take) { sv[threadIdx.x] = v2; si[threadIdx.x] = i2; sl[threadIdx.x] = sl[threadIdx.x + s]; }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[blockIdx.x * 3] = sv[0];
    part[blockIdx.x * 3 + 1] = (double)si[0];
    part[blockIdx.x * 3 + 2] = (double)sl[0];
  }
  __syncthreads();
}

// Polar factor of A^T (A = M~ = U S V^T):  X -> V U^T by Newton-Schulz
// X <- 1.5 X - 0.5 X X^T X from X0 = A^T / s with s >= sigma_max(A) (all
// singular values in (0, 1]).  Returns sum(sigma) = tr(X A).  Identical
// arithmetic in every CTA.  k <= 8 first runs quintic sweeps
// X <- X (a I + b Y + c Y^2) (small singular values grow ~3.4x per sweep and
// all stay in (0, 1.13], the basin of the cubic iteration).
constexpr int kQuinticSweeps = 5;

// Upper bound on sigma_max(A) (k x k, shared memory), called by one full
// warp: min(||A||_F, sqrt(||A||_1 ||A||_inf)).  Scaling the Newton-Schulz
// start by it instead of ||A||_F alone puts the singular values of a
// well-conditioned A near 1 (||A||_F overestimates sigma_max by up to
// sqrt(k)), so the linear phase of the iteration is short.
__device__ __forceinline__ double sigma_bound_warp(const double* A, int k, bool tight) {
  const int lane = threadIdx.x & 31;
  double f = 0.0, rmax = 0.0, cmax = 0.0;
  for (int e = lane; e < k * k; e += 32) f += A[e] * A[e];
  f = warp_sum(f);
  if (!tight) return sqrt(f);
  for (int r = lane; r < k; r += 32) {
    double rs = 0.0, cs = 0.0;
    for (int c = 0; c < k; ++c) {
      rs += fabs(A[r * k + c]);
      cs += fabs(A[c * k + r]);
    }
    rmax = fmax(rmax, rs);
    cmax = fmax(cmax, cs);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
    cmax = fmax(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
  }
  return fmin(sqrt(f), sqrt(rmax * cmax));
}

// Polar factor for k <= 8 with the whole CTA: the k x k blocks are padded
// to 8 x 8 in shared memory (zeros outside k, so padded terms vanish) and
// each product C = op(A) B is 64 entries x 8 terms = 512 products on 256
// threads, summed over aligned 8-lane groups by three shuffles -- one
// barrier per product instead of a k-long dependent shuffle chain per entry
// in one warp (4x shorter per sweep).  Same recipe as the warp version:
// quintic f32 sweeps, cubic f32 sweeps to 1e-4, cubic f64 to the fixed point.
template <typename T>
__device__ __forceinline__ T seg8_sum(T v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  return v;
}

// C[r][c] = sum_l op(A)[r][l] B[l][c] on 8 x 8 blocks; TA: op(A) = A^T
template <typename T, bool TA>
__device__ __forceinline__ void mm8(const T* A, const T* B, T* C) {
  const int t = threadIdx.x, l = t & 7;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int e = (t >> 3) + 32 * h, r = e >> 3, c = e & 7;
    T v = (TA ? A[l * 8 + r] : A[r * 8 + l]) * B[l * 8 + c];
    v = seg8_sum(v);
    if (l == 0) C[e] = v;
  }
  __syncthreads();
}

// cubic sweeps X <- 1.5 X - 0.5 X (X^T X) until no entry moves more than tol
template <typename T>
__device__ int ns_sweeps_cta(T* X, T* Y, T* Tm, T tol, int max_it) {
  int it = 0;
  for (; it < max_it; ++it) {
    mm8<T, true>(X, X, Y);
    mm8<T, false>(X, Y, Tm);
    bool moved = false;
    if (threadIdx.x < 64) {
      const T xo = X[threadIdx.x];
      const T xn = T(1.5) * xo - T(0.5) * Tm[threadIdx.x];
      moved = fabs(xn - xo) > tol;
      X[threadIdx.x] = xn;
    }
    if (!__syncthreads_or(moved)) { ++it; break; }
  }
  return it;
}

__device__ double polar_ns_small_cta(const double* A, double* X, int k, int* iters, double* red) {
  __shared__ float xf[64], yf[64], zf[64], tf[64];
  __shared__ double xd[64], yd[64], td[64];
  __shared__ double s_inv;
  const int t = threadIdx.x;
  // Frobenius start (measured faster here than the tight bound, which leaves
  // the quintic sweeps overshooting on the ill-conditioned small-k blocks)
  if (t < 32) {
    const double sb = sigma_bound_warp(A, k, false);
    if (t == 0) s_inv = sb > 0 ? 1.0 / sb : 0.0;
  }
  __syncthreads();
  if (t < 64) {   // X = A^T / sb, padded
    const int r = t >> 3, c = t & 7;
    xf[t] = (r < k && c < k) ? (float)(A[c * k + r] * s_inv) : 0.f;
  }
  __syncthreads();
  constexpr float qa = 3.4445f, qb = -4.7750f, qc = 2.0315f;
  for (int q = 0; q < kQuinticSweeps; ++q) {   // X <- X (a I + b Y + c Y^2)
    mm8<float, true>(xf, xf, yf);
    mm8<float, false>(yf, yf, zf);
    if (t < 64) zf[t] = qb * yf[t] + qc * zf[t];
    __syncthreads();
    mm8<float, false>(xf, zf, tf);
    if (t < 64) xf[t] = qa * xf[t] + tf[t];
    __syncthreads();
  }
  int it = kQuinticSweeps;
  it += ns_sweeps_cta<float>(xf, yf, tf, 1e-4f, 60);
  if (t < 64) xd[t] = (double)xf[t];
  __syncthreads();
  it += ns_sweeps_cta<double>(xd, yd, td, 1e-14 * k, 100);
  double tr = 0.0;   // tr(X A) = sum_{a,b} X[a][b] A[b][a]
  if (t < 64) {
    const int r = t >> 3, c = t & 7;
    if (r < k && c < k) {
      X[r * k + c] = xd[t];
      tr = xd[t] * A[c * k + r];
    }
  }
  tr = block_sum(tr, red);
  if (t == 0) *iters = it;
  __syncthreads();
  return tr;
}

// C = op(A) B for k x k row-major blocks (op(A) = A^T when TA): 16 x 16
// threads, each a TB x TB register block (TB = ceil(k / 16), compile time)
template <int TB, bool TA>
__device__ __forceinline__ void mm_blk(const double* A, const double* B, double (&acc)[TB][TB], int k) {
  const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
#pragma unroll
  for (int u = 0; u < TB; ++u)
#pragma unroll
    for (int v = 0; v < TB; ++v) acc[u][v] = 0.0;
  for (int l = 0; l < k; ++l) {
    double xa[TB], xb[TB];
#pragma unroll
    for (int u = 0; u < TB; ++u) {
      const int a = ty * TB + u, b = tx * TB + u;
      xa[u] = a < k ? (TA ? A[l * k + a] : A[a * k + l]) : 0.0;
      xb[u] = b < k ? B[l * k + b] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < TB; ++u)
#pragma unroll
      for (int v = 0; v < TB; ++v) acc[u][v] = fma(xa[u], xb[v], acc[u][v]);
  }
}
template <int TB, typename F>
__device__ __forceinline__ void blk_each(int k, F f) {
  const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
#pragma unroll
  for (int u = 0; u < TB; ++u)
#pragma unroll
    for (int v = 0; v < TB; ++v) {
      const int a = ty * TB + u, b = tx * TB + v;
      if (a < k && b < k) f(u, v, a * k + b);
    }
}

// k > 8: X -> polar factor by Newton-Schulz in f64.  `qs` quintic sweeps
// X <- X (a I + b Y + c Y^2), Y = X^T X, first (small singular values grow
// 3.44x per sweep for 3 products, against 1.5x per cubic step for 2; all
// stay in (0, 1.13], inside the cubic basin), then cubic steps to the
// fixed point.  The caller sizes qs from the previous round's count (the
// rounds of one call have similar conditioning); the limit is the polar
// factor either way.
template <int TB>
__device__ double polar_ns_tb(const double* A, double* X, double* Y, double* T, int k, int qs,
                              int* flag, double* red, int* iters) {
  __shared__ double s_tr;
  const int kk = k * k, t = threadIdx.x;
  if (t < 32) {
    const double sb = sigma_bound_warp(A, k, true);
    if (t == 0) s_tr = sb;
  }
  __syncthreads();
  const double inv = s_tr > 0 ? 1.0 / s_tr : 0.0;
  __syncthreads();
  for (int e = t; e < kk; e += blockDim.x) X[(e % k) * k + e / k] = A[e] * inv;  // A^T
  __syncthreads();
  double acc[TB][TB];
  int it = 0;
  for (int q = 0; q < qs; ++q, ++it) {
    constexpr double qa = 3.4445, qb = -4.7750, qc = 2.0315;
    mm_blk<TB, true>(X, X, acc, k);                      // Y = X^T X
    blk_each<TB>(k, [&](int u, int v, int e) { Y[e] = acc[u][v]; });
    __syncthreads();
    mm_blk<TB, false>(Y, Y, acc, k);                     // T = a I + b Y + c Y^2
    blk_each<TB>(k, [&](int u, int v, int e) {
      T[e] = qb * Y[e] + qc * acc[u][v] + ((e / k == e % k) ? qa : 0.0);
    });
    __syncthreads();
    mm_blk<TB, false>(X, T, acc, k);                     // X <- X T
    __syncthreads();
    blk_each<TB>(k, [&](int u, int v, int e) { X[e] = acc[u][v]; });
    __syncthreads();
  }
  for (int c = 0; c < 100; ++c) {
    mm_blk<TB, true>(X, X, acc, k);                      // Y = X^T X
    blk_each<TB>(k, [&](int u, int v, int e) { Y[e] = acc[u][v]; });
    __syncthreads();
    if (t == 0) *flag = 0;
    mm_blk<TB, false>(X, Y, acc, k);                     // T = X Y
    __syncthreads();                                     // all reads of X done
    bool moved = false;
    blk_each<TB>(k, [&](int u, int v, int e) {
      const double xo = X[e];
      const double xn = 1.5 * xo - 0.5 * acc[u][v];
      moved |= fabs(xn - xo) > 1e-14 * k;
      X[e] = xn;
    });
    ++it;
    if (moved) *flag = 1;
    __syncthreads();
    const bool more = *flag != 0;
    __syncthreads();
    if (!more) break;
  }
  double tr = 0.0;                                        // tr(X A)
  for (int e = t; e < kk; e += blockDim.x) {
    const int a = e / k, b = e % k;
    tr += X[a * k + b] * A[b * k + a];
  }
  tr = block_sum(tr, red);
  if (t == 0) *iters = it;
  __syncthreads();
  return tr;
}

template <int KMAX>
__device__ double polar_ns(const double* A, double* X, double* Y, double* T, int k, int qs,
                           int* flag, double* red, int* iters) {
  if (k <= 8) return polar_ns_small_cta(A, X, k, iters, red);
  constexpr int TB = KMAX <= 16 ? 1 : KMAX <= 32 ? 2 : KMAX <= 48 ? 3 : 4;
  return polar_ns_tb<TB>(A, X, Y, T, k, qs, flag, red, iters);
}

// Totals accumulated by the fixed-point atomics of phase A (buffer ri % 3);
// CTA 0 clears buffer (ri + 2) % 3, whose next use is two barriers away.
__device__ void reduce_all(const DiscParams& p, double* M, long long* sizes, int ri) {
  const int k = p.k, ne = k * k + k;
  const unsigned long long* src = p.gfx + (size_t)(ri % 3) * ne;
  for (int e = threadIdx.x; e < k * k; e += blockDim.x)
    M[e] = (double)(long long)__ldcg(src + e) / p.fx_scale;
  for (int e = threadIdx.x; e < k; e += blockDim.x) sizes[e] = (long long)__ldcg(src + k * k + e);
  if (blockIdx.x == 0)
    for (int e = threadIdx.x; e < ne; e += blockDim.x) p.gfx[(size_t)((ri + 2) % 3) * ne + e] = 0ull;
  __syncthreads();
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// CTA 0 accumulates ns between stamps: slot s gets (now - previous stamp)
#define TSTAMP(s)                                                      \
  do {                                                                 \
    if (p.tdbg && blockIdx.x == 0 && threadIdx.x == 0) {               \
      const unsigned long long _n = gtimer();                          \
      if ((s) != 0) p.tdbg[(s)] += _n - t_prev;                        \
      else if (t_prev) p.tdbg[15] += _n - t_prev;                      \
      t_prev = _n;                                                     \
    }                                                                  \
  } while (0)

template <int KMAX>
__global__ void __launch_bounds__(kDiscThreads, 1)
discretize_kernel(DiscParams p) {
  unsigned long long t_prev = 0;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smraw[];
  const int k = p.k, kk = k * k, kp = kpad4(k);
  const int G = p.groups;
  const int nb = gridDim.x;
  // persistent: scoring rotation (f32, rows padded to kp; k > 8: TF32 B
  // fragments) and prototype rotation (f64)
  float* sR = reinterpret_cast<float*>(smraw);
  const uint4* sRf = reinterpret_cast<const uint4*>(smraw);
  const double* sR64 = reinterpret_cast<const double*>(smraw + (KMAX > 8 ? disc_frag_bytes(k) : 0));
  double* sRp = reinterpret_cast<double*>(smraw + align_dev(disc_rot_bytes(k, (int)(p.col0 & 3))));
  unsigned char* dyn = smraw + align_dev(disc_rot_bytes(k, (int)(p.col0 & 3))) + align_dev((size_t)kk * 8);
  // phase-A view (k <= 8: G f64 accumulator groups; k > 8: split fixed-point totals)
  double* acc = reinterpret_cast<double*>(dyn);
  long long* gacc = reinterpret_cast<long long*>(dyn);
  int* gcnt = reinterpret_cast<int*>(dyn + align_dev(disc_tc_acc_bytes(k, G)));
  float* tile = reinterpret_cast<float*>(
      KMAX > 8 ? dyn + align_dev(disc_tc_acc_bytes(k, G)) + align_dev((size_t)G * k * 4)
               : dyn + align_dev((size_t)G * kk * 8));
  int* tlab = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(tile) +
                                     align_dev(KMAX > 8 ? disc_tc_tile_bytes(k, (int)(p.col0 & 3), p.dbuf)
                                                        : disc_tile_bytes(k, (int)(p.col0 & 3))));
  int* cnt = tlab + kDiscThreads;
  // phase-B view (aliases phase A)
  double* M = reinterpret_cast<double*>(dyn);
  double* X = M + kk;
  double* Y = X + kk;
  double* T = Y + kk;
  long long* sizes = reinterpret_cast<long long*>(T + kk);
  __shared__ double sv[kDiscThreads];
  __shared__ long long si[kDiscThreads];
  __shared__ int sl[kDiscThreads];
  __shared__ double red[32];
  __shared__ int s_flag, s_zero;
  __shared__ double s_pcol[KMAX > 8 ? Win<KMAX>::KW : 1];
  __shared__ long long s_mvi[64];    // reseed moves: row, old cluster, new cluster
  __shared__ int s_mvo[64], s_mvc[64], s_nmv;
  const bool vec = (p.ldq % 4 == 0) && ((reinterpret_cast<uintptr_t>(p.Q) & 15) == 0);

  const bool cta0 = blockIdx.x == 0;
  const Rows rows = my_rows(p.n);
  int buf = 0;                 // partial-buffer parity (advances per barrier)
  int ri = 0;                  // accumulate/reduce counter (rotating fixed-point totals)
  double final_obj[2] = {0.0, 0.0};
  int final_rounds[2] = {0, 0};
  double final_conv[2] = {0.0, 0.0};
  int empties_left[2] = {0, 0};
  if (KMAX > 8) {            // q~ once per call (the rounds read the f32 copy)
    const int z = normalize_rows(p);
    if (threadIdx.x == 0) s_zero = 0;
    __syncthreads();
    if (z) atomicAdd(&s_zero, z);
    __syncthreads();
  }

  int qs_next = 0;             // quintic Newton-Schulz sweeps for the next polar factor
  for (int run = p.run_lo; run < p.run_hi; ++run) {
    // ---------------------------------------------------- initial rotation
    if (run == 0) {
      if (KMAX > 8)
        store_rot_frag(smraw, k, [](int l, int j) { return l == j ? 1.0 : 0.0; });
      else
        for (int e = threadIdx.x; e < k * kp; e += blockDim.x) sR[e] = (e / kp == e % kp) ? 1.f : 0.f;
      if (cta0) for (int e = threadIdx.x; e < kk; e += blockDim.x) p.Rg[e] = (e / k == e % k) ? 1.0 : 0.0;
    } else {
      // prototype rotation (engine.py:209-218): R[:,0] = q~[0]; greedy rows
      if (threadIdx.x == 0) {
        double q[KMAX], nrm;
        load_row<KMAX>(p, 0, q, nrm);
        for (int l = 0; l < k; ++l) sRp[l * k] = q[l];
      }
      for (int64_t i = rows.r0 + threadIdx.x; i < rows.r1; i += blockDim.x) p.proto_acc[i] = 0.0;
      __syncthreads();
      TSTAMP(0);
      for (int j = 1; j < k; ++j) {
        double best = 0.0;
        long long bi = -1;
        if (KMAX > 8) {
          // staged window tiles (coalesced reads); column j-1 of the
          // prototype rotation shifted into window coordinates
          constexpr int KW = Win<KMAX>::KW, SW = Win<KMAX>::SW;
          const int off = (int)(p.col0 & 3);
          for (int m = threadIdx.x; m < KW; m += blockDim.x) {
            const int l = m - off;
            s_pcol[m] = (l >= 0 && l < k) ? sRp[l * k + (j - 1)] : 0.0;
          }
          __syncthreads();
          // double-buffered window tiles: the copy of tile ti + 1 overlaps
          // the dot products of tile ti
          const int ntl = (int)ceil_div(rows.r1 - rows.r0, (int64_t)kDiscThreads);
          const size_t wbuf = (size_t)kDiscThreads * SW;
          auto issue = [&](int ti) {
            const int64_t s0 = rows.r0 + (int64_t)ti * kDiscThreads;
            stage_window_issue(p, s0, (int)lmin(kDiscThreads, rows.r1 - s0),
                               tile + (p.dbuf ? (ti & 1) * wbuf : 0), SW, vec);
          };
          if (ntl > 0 && p.dbuf) issue(0);
          // 1/||q_i|| and the running sum of this thread's row, one tile ahead
          double inv_next = 0.0, acc_next = 0.0;
          if (rows.r0 + threadIdx.x < rows.r1) {
            inv_next = p.qinv[rows.r0 + threadIdx.x];
            acc_next = p.proto_acc[rows.r0 + threadIdx.x];
          }
          for (int ti = 0; ti < ntl; ++ti) {
            const int64_t t0 = rows.r0 + (int64_t)ti * kDiscThreads;
            const int tr = (int)lmin(kDiscThreads, rows.r1 - t0);
            const double inv = inv_next, acc_prev = acc_next;
            if (t0 + kDiscThreads + threadIdx.x < rows.r1) {
              inv_next = p.qinv[t0 + kDiscThreads + threadIdx.x];
              acc_next = p.proto_acc[t0 + kDiscThreads + threadIdx.x];
            }
            if (!p.dbuf) {
              issue(ti);
              asm volatile("cp.async.wait_group 0;" ::: "memory");
            } else if (ti + 1 < ntl) {
              issue(ti + 1);
              asm volatile("cp.async.wait_group 1;" ::: "memory");
            } else {
              asm volatile("cp.async.wait_group 0;" ::: "memory");
            }
            __syncthreads();
            if (threadIdx.x < tr) {
              const int64_t i = t0 + threadIdx.x;
              float raw[KW];
              load_window<KMAX>(tile + (p.dbuf ? (ti & 1) * wbuf : 0) + threadIdx.x * SW, off, k, raw);
              double d = 0.0;
#pragma unroll
              for (int m = 0; m < KW; ++m) d += ((double)raw[m] * inv) * s_pcol[m];
              const double a = acc_prev + fabs(d);
              p.proto_acc[i] = a;
              if (bi < 0 || a < best) { best = a; bi = i; }
            }
            __syncthreads();
          }
        } else {
          for (int64_t i = rows.r0 + threadIdx.x; i < rows.r1; i += blockDim.x) {
            double q[KMAX], nrm;
            load_row<KMAX>(p, i, q, nrm);
            double d = 0.0;
#pragma unroll
            for (int l = 0; l < KMAX; ++l)
              if (l < k) d += q[l] * sRp[l * k + (j - 1)];
            const double a = p.proto_acc[i] + fabs(d);
            p.proto_acc[i] = a;
            if (bi < 0 || a < best) { best = a; bi = i; }
          }
        }
        double* part = p.part_arg + (size_t)buf * nb * 3;
        block_arg(best, bi, 0, false, part, sv, si, sl);
        grid.sync();
        TSTAMP(5);
        double v;
        long long idx;
        int lab;
        reduce_arg(part, nb, false, v, idx, lab, sv, si, sl);
        if (threadIdx.x == 0) {
          double q[KMAX], nrm;
          load_row<KMAX>(p, idx < 0 ? 0 : idx, q, nrm);
          for (int l = 0; l < k; ++l) sRp[l * k + j] = q[l];
        }
        buf ^= 1;
        __syncthreads();
      }
      if (KMAX > 8)
        store_rot_frag(smraw, k, [&](int l, int j) { return sRp[l * k + j]; });
      else
        for (int e = threadIdx.x; e < k * kp; e += blockDim.x)
          sR[e] = e % kp < k ? (float)sRp[(e / kp) * k + e % kp] : 0.f;
      if (cta0) for (int e = threadIdx.x; e < kk; e += blockDim.x) p.Rg[e] = sRp[e];
    }
    __syncthreads();

    // ---------------------------------------------------------- rounds
    double obj_prev = 0.0;
    double cdrift = 0.0;         // cumulative rotation drift of this start (row keys)
    bool conv = false;
    int rounds = 0;
    for (int it = 0; it < p.max_iter; ++it) {
      TSTAMP(0);
      if (KMAX > 8)
        phase_accumulate_tc<KMAX>(p, sRf, sR64, tile, tlab, gacc, gcnt, true,
                                  p.gfx + (size_t)(ri % 3) * (kk + k),
                                  (run == p.run_lo && it == 0) ? nullptr
                                                               : p.gfx + (size_t)((ri + 2) % 3) * (kk + k),
                                  cdrift, it > 0);
      else
        phase_accumulate<KMAX>(p, sR, tile, tlab, acc, cnt, true,
                               (run == 0 && it == 0) ? &s_zero : nullptr,
                               p.gfx + (size_t)(ri % 3) * (kk + k));
      if (run == 0 && it == 0 && threadIdx.x == 0)   // fold the zero-row count into the
        p.part_cnt[((size_t)(buf ^ 1) * nb + blockIdx.x) * k] = s_zero;  // idle buffer
      TSTAMP(6);
      grid.sync();
      TSTAMP(1);
      if (run == 0 && it == 0 && cta0 && threadIdx.x == 0) {   // zero rows (engine.py:239-242)
        long long z = 0;
        for (int b = 0; b < nb; ++b) z += p.part_cnt[((size_t)(buf ^ 1) * nb + b) * k];
        p.info[5] = (double)z;
      }
      reduce_all(p, M, sizes, ri);
      ++ri;
      TSTAMP(2);
      buf ^= 1;
      int nempty = 0;
      for (int c = 0; c < k; ++c) nempty += sizes[c] == 0;
      if (nempty > 0 && k >= 2) {
        if (KMAX > 8)
          exact_margins<KMAX>(p, sR64);
        // _reseed_empty_columns (engine.py:162-180): every CTA tracks sizes
        if (threadIdx.x == 0) s_nmv = 0;
        __syncthreads();
        for (int c = 0; c < k; ++c) {
          if (sizes[c] != 0) continue;
          double bestm = 0.0;
          long long bi = -1;
          int blab = 0;
          for (int64_t i = rows.r0 + threadIdx.x; i < rows.r1; i += blockDim.x) {
            const int l = p.labels[i];
            if (sizes[l] >= 2) {
              const double m = p.margin[i];
              if (bi < 0 || m > bestm) { bestm = m; bi = i; blab = l; }
            }
          }
          double* part = p.part_arg + (size_t)buf * nb * 3;
          block_arg(bestm, bi, blab, true, part, sv, si, sl);
          grid.sync();
          double v;
          long long idx;
          int old;
          reduce_arg(part, nb, true, v, idx, old, sv, si, sl);
          buf ^= 1;
          if (idx < 0) break;                          // no movable node left
          if (threadIdx.x == 0) {
            sizes[old] -= 1;
            sizes[c] += 1;
            if (idx >= rows.r0 && idx < rows.r1) {                  // owner CTA
              p.labels[idx] = c;
              if (KMAX > 8) p.key[idx] = -INFINITY;                  // score it next round
            }
            s_mvi[s_nmv] = idx;
            s_mvo[s_nmv] = old;
            s_mvc[s_nmv] = c;
            ++s_nmv;
          }
          __syncthreads();
        }
        if (KMAX > 8) {
          // new totals = previous totals (carried slice by slice) + the moved
          // rows' fixed-point deltas, applied by their owner CTAs: the exact
          // integers a recount gives (phase_accumulate_tc's invariant)
          unsigned long long* gdst = p.gfx + (size_t)(ri % 3) * (kk + k);
          const unsigned long long* gprev = p.gfx + (size_t)((ri + 2) % 3) * (kk + k);
          for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < kk + k;
               e += (int64_t)gridDim.x * blockDim.x) {
            const unsigned long long v = __ldcg(gprev + e);
            if (v) atomicAdd(gdst + e, v);
          }
          const int sh = ilogb(p.fx_scale), kq = disc_kq(k);
          for (int m = 0; m < s_nmv; ++m) {
            const long long idx = s_mvi[m];
            if (idx < rows.r0 || idx >= rows.r1) continue;
            const int old = s_mvo[m], c = s_mvc[m];
            for (int j = threadIdx.x; j < k; j += blockDim.x) {
              const long long fx = fx_round(p.qn[idx * kq + j], sh);
              if (fx != 0) {
                atomicAdd(gdst + c * k + j, (unsigned long long)fx);
                atomicAdd(gdst + old * k + j, (unsigned long long)(-fx));
              }
            }
            if (threadIdx.x == 0) {
              atomicAdd(gdst + kk + c, 1ull);
              atomicAdd(gdst + kk + old, ~0ull);
            }
          }
        } else
          phase_accumulate<KMAX>(p, sR, tile, tlab, acc, cnt, false, nullptr,
                                 p.gfx + (size_t)(ri % 3) * (kk + k));
        grid.sync();
        reduce_all(p, M, sizes, ri);
        ++ri;
        buf ^= 1;
      }
      // Y~ = Y / size, polar factor and objective
      for (int e = threadIdx.x; e < kk; e += blockDim.x) {
        const long long sz = sizes[e / k];
        M[e] = sz > 0 ? M[e] / (double)sz : 0.0;
      }
      __syncthreads();
      TSTAMP(3);
      int ns_it = 0;
      const double ssum = polar_ns<KMAX>(M, X, Y, T, k, qs_next, &s_flag, red, &s_flag);
      ns_it = s_flag;
      {   // quintic sweeps for the next round: each replaces ~3 cubic steps
        const int cubic = ns_it - qs_next;
        qs_next = cubic > 7 ? qs_next + (cubic - 5) / 3 : (cubic < 5 && qs_next > 0 ? qs_next - 1 : qs_next);
        if (qs_next > 12) qs_next = 12;
      }
      if (p.tdbg && cta0 && threadIdx.x == 0) p.tdbg[7] += ns_it;
      TSTAMP(4);
      const double obj = (double)p.n - 2.0 * ssum;
      if (cta0 && threadIdx.x == 0) p.info[8 + run * p.max_iter + it] = obj;
      conv = it >= 1 && fabs(obj - obj_prev) < p.tol;
      obj_prev = obj;
      rounds = it + 1;
      if (conv || it + 1 == p.max_iter) {
        int ne = 0;
        for (int c = 0; c < k; ++c) ne += sizes[c] == 0;
        empties_left[run] = ne;
        break;
      }
      // next rotation R = V U^T (engine.py:205)
      if (KMAX > 8) {
        // drift of the rotation: max_j ||X_j - R_j|| bounds every row's score
        // change (row keys, phase_accumulate_tc)
        double cm = 0.0;
        for (int j = threadIdx.x; j < k; j += blockDim.x) {
          double s2 = 0.0;
          for (int l = 0; l < k; ++l) {
            const double d = X[l * k + j] - sR64[l * k + j];
            s2 += d * d;
          }
          cm = fmax(cm, sqrt(s2));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, o));
        __syncthreads();
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cm;
        __syncthreads();
        double dmax = 0.0;
        for (int w = 0; w < kDiscThreads / 32; ++w) dmax = fmax(dmax, red[w]);
        cdrift += dmax * (1.0 + 1e-6) + 1e-14;    // rows of norm 1 + O(2^-24), f64 rounding
        __syncthreads();
        store_rot_frag(smraw, k, [&](int l, int j) { return X[l * k + j]; });
      }
      else
        for (int e = threadIdx.x; e < k * kp; e += blockDim.x)
          sR[e] = e % kp < k ? (float)X[(e / kp) * k + e % kp] : 0.f;
      if (cta0) for (int e = threadIdx.x; e < kk; e += blockDim.x) p.Rg[e] = X[e];
      __syncthreads();
    }
    final_obj[run] = obj_prev;
    final_rounds[run] = rounds;
    final_conv[run] = conv ? 1.0 : 0.0;
    // publish the rotation that produced this run's final scores
    if (cta0) {
      __syncthreads();
      for (int e = threadIdx.x; e < kk; e += blockDim.x)
        p.info[8 + 2 * p.max_iter + run * kk + e] = p.Rg[e];
    }
    if (run == 0 && p.run_hi == 2)
      for (int64_t i = rows.r0 + threadIdx.x; i < rows.r1; i += blockDim.x)
        p.labels_run0[i] = p.labels[i];
    __syncthreads();
  }
  if (p.run_hi - p.run_lo == 1) {   // split launch: the finish kernel picks the winner
    if (cta0 && threadIdx.x == 0) {
      const int r = p.run_lo;
      p.fin[r * 4 + 0] = final_obj[r];
      p.fin[r * 4 + 1] = final_rounds[r];
      p.fin[r * 4 + 2] = final_conv[r];
      p.fin[r * 4 + 3] = empties_left[r];
    }
    return;
  }
  // identity wins unless the prototype run is lower by more than 1e-15
  const int win = final_obj[1] < final_obj[0] - 1e-15 ? 1 : 0;
  if (cta0 && threadIdx.x == 0) {
    p.info[0] = final_obj[win];
    p.info[1] = final_rounds[win];
    p.info[2] = final_conv[win];
    p.info[3] = win;
    p.info[4] = empties_left[win];
    p.info[6] = final_rounds[0];
    p.info[7] = final_rounds[1];
  }
  if (win == 0)
    for (int64_t i = rows.r0 + threadIdx.x; i < rows.r1; i += blockDim.x)
      p.labels[i] = p.labels_run0[i];
}

// Split launches: pick the winning start (same rule as the fused tail) and
// move the identity run's labels into the output when it wins.
__global__ void discretize_finish_kernel(const double* __restrict__ fin, double* __restrict__ info,
                                         const int32_t* __restrict__ labels_run0,
                                         int32_t* __restrict__ labels, int64_t n) {
  const int win = fin[4] < fin[0] - 1e-15 ? 1 : 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    info[0] = fin[win * 4 + 0];
    info[1] = fin[win * 4 + 1];
    info[2] = fin[win * 4 + 2];
    info[3] = win;
    info[4] = fin[win * 4 + 3];
    info[6] = fin[1];
    info[7] = fin[5];
  }
  if (win == 0)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
      labels[i] = labels_run0[i];
}

}  // namespace ancka

using namespace ancka;

static size_t disc_smem(int k, int G, int off, int dbuf = 1) {
  const size_t kk = (size_t)k * k;
  const size_t fixed = align_dev(disc_rot_bytes(k, off)) + align_dev(kk * 8);
  const size_t a = k > 8 ? align_dev(disc_tc_acc_bytes(k, G)) + align_dev((size_t)G * k * 4) +
                               align_dev(disc_tc_tile_bytes(k, off, dbuf)) +
                               (6 * kDiscThreads + 68 + 64) * 4 + 8 * 64 * 8 + 8 * 64 * 4
                         : align_dev((size_t)G * kk * 8) + align_dev(disc_tile_bytes(k, off)) +
                               (kDiscThreads + (size_t)G * k) * 4;
  const size_t b = 4 * kk * 8 + (size_t)k * 8;
  return fixed + std::max(a, b) + 64;
}

// accumulator groups: k <= 8 f64 groups of k x k; k > 8 fixed-point groups
// of k x kq, as many as the threads and ~210 KB of shared memory allow
static int disc_groups(int k, int off) {
  if (k <= 8) {
    int g = kDiscThreads / k;
    const int cap = (int)((96 * 1024) / ((size_t)k * k * 8));
    if (g > cap) g = cap;
    return g < 1 ? 1 : g;
  }
  (void)off;
  return 1;          // one accumulator: buckets give each (label, column) one owner
}

static int disc_grid_cap() { return 4 * kNumSMs; }

extern "C" size_t ancka_discretize_workspace_size(int64_t n, int32_t k, int32_t max_iter) {
  (void)max_iter;
  if (k > disc_wide_min()) return discretize_wide_workspace(n, k);
  Carver cv(nullptr, 0);
  const int grid = disc_grid_cap();
  cv.take<int32_t>(n);              // labels_run0
  cv.take<double>(n);               // proto_acc
  cv.take<double>(8);               // fin
  if (k > 8) {
    cv.take<float>((size_t)n * disc_kq(k));   // qn
    cv.take<double>(n);                       // qinv
    cv.take<double>(n);                       // key
    cv.take<int32_t>(n);                      // rid
  }
  for (int r = 0; r < 2; ++r) {     // per start (split launches run concurrently)
    cv.take<float>(n);              // margin
    cv.take<int64_t>((size_t)2 * grid * k);
    cv.take<double>((size_t)2 * grid * 3);
    cv.take<double>((size_t)k * k);
    cv.take<unsigned long long>((size_t)3 * (k * k + k));
  }
  return cv.used;
}

template <int KMAX>
static int launch_disc(DiscParams& p, cudaStream_t st, int sm_share) {
  auto kern = discretize_kernel<KMAX>;
  const size_t smem = disc_smem(p.k, p.groups, (int)(p.col0 & 3), p.dbuf);
  ANCKA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  ANCKA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kDiscThreads, smem));
  ANCKA_REQUIRE(per_sm >= 1, ANCKA_ERR_UNSUPPORTED, "discretize: kernel does not fit an SM");
  int dev = 0, sms = 0;
  ANCKA_CUDA(cudaGetDevice(&dev));
  ANCKA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // rows per CTA (tunable): enough work per phase to amortise the grid barrier
  static const int64_t min_rows =
      getenv("ANCKA_DISC_ROWS") ? atoll(getenv("ANCKA_DISC_ROWS")) : kDiscThreads;
  int64_t want = ceil_div(p.n, std::max<int64_t>(kDiscThreads, min_rows));
  int64_t grid = std::min(want, std::min((int64_t)per_sm * sms / sm_share, (int64_t)disc_grid_cap()));
  if (grid < 1) grid = 1;
  void* args[] = {&p};
  note_launch();
  ANCKA_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3((unsigned)grid), dim3(kDiscThreads),
                                         args, smem, st));
  return ANCKA_OK;
}

static int launch_disc_k(DiscParams& p, int k, int64_t col0, cudaStream_t st, int sm_share) {
  switch (disc_kmax(k, (int)(col0 & 3))) {
    case 8: return launch_disc<8>(p, st, sm_share);
    case 16: return launch_disc<16>(p, st, sm_share);
    case 32: return launch_disc<32>(p, st, sm_share);
    case 48: return launch_disc<48>(p, st, sm_share);
    case 64: return launch_disc<64>(p, st, sm_share);
    default: return launch_disc<68>(p, st, sm_share);
  }
}

// Second stream + fork/join events for the split launches (one per device,
// created on first use; legal inside stream capture).
struct DiscSide {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
static int disc_side(DiscSide** out) {
  static DiscSide sides[16];
  int dev = 0;
  ANCKA_CUDA(cudaGetDevice(&dev));
  DiscSide& d = sides[dev & 15];
  if (!d.s) {
    ANCKA_CUDA(cudaStreamCreateWithFlags(&d.s, cudaStreamNonBlocking));
    ANCKA_CUDA(cudaEventCreateWithFlags(&d.fork, cudaEventDisableTiming));
    ANCKA_CUDA(cudaEventCreateWithFlags(&d.join, cudaEventDisableTiming));
  }
  *out = &d;
  return ANCKA_OK;
}

// The two alternating-rounding starts are independent until the final
// comparison (engine.py:247-253).  Small blocks (latency-bound rounds: a grid
// barrier, a tiny polar factor) run them as two concurrent cooperative
// launches on half the SMs each, the prototype start on a side stream; large
// blocks (bandwidth/issue-bound rounds) keep one launch over the whole GPU.
static bool disc_split(int64_t n, int k) {
  static const int force = getenv("ANCKA_DISC_SPLIT") ? atoi(getenv("ANCKA_DISC_SPLIT")) : -1;
  if (force >= 0) return force != 0;
  return k <= 8 && n <= (1 << 20);
}

extern "C" int ancka_discretize(const float* Q, int64_t ldq, int64_t col0, int64_t n, int32_t k,
                                int32_t max_iter, double tol, int32_t* labels_out, double* info,
                                void* workspace, size_t workspace_bytes, ancka_stream_t stream) {
  ANCKA_REQUIRE(k >= 1 && k <= kDiscWideMaxK, ANCKA_ERR_UNSUPPORTED, "discretize: k=%d outside [1, %d]",
                k, kDiscWideMaxK);
  if (k > disc_wide_min())   // wide blocks: device-driven rounds (disc_wide_dev.cu)
    return discretize_wide(Q, ldq, col0, n, k, max_iter, tol, labels_out, info, workspace,
                           workspace_bytes, as_stream(stream));
  ANCKA_REQUIRE(n >= 1 && max_iter >= 1, ANCKA_ERR_ARG, "discretize: empty input");
  Carver cv(workspace, workspace_bytes);
  DiscParams p{};
  const int grid = disc_grid_cap();
  p.Q = Q; p.ldq = ldq; p.col0 = col0; p.n = n; p.k = k; p.max_iter = max_iter; p.tol = tol;
  p.labels = labels_out;
  p.labels_run0 = cv.take<int32_t>(n);
  p.proto_acc = cv.take<double>(n);
  p.fin = cv.take<double>(8);
  if (k > 8) {
    p.qn = cv.take<float>((size_t)n * disc_kq(k));
    p.qinv = cv.take<double>(n);
    p.key = cv.take<double>(n);
    p.rid = cv.take<int32_t>(n);
  }
  DiscParams pr[2];
  for (int r = 0; r < 2; ++r) {
    pr[r] = p;
    pr[r].margin = cv.take<float>(n);
    pr[r].part_cnt = cv.take<int64_t>((size_t)2 * grid * k);
    pr[r].part_arg = cv.take<double>((size_t)2 * grid * 3);
    pr[r].Rg = cv.take<double>((size_t)k * k);
    pr[r].gfx = cv.take<unsigned long long>((size_t)3 * (k * k + k));
  }
  {
    int bits = 1;
    while ((1ll << bits) <= n) ++bits;
    p.fx_scale = std::ldexp(1.0, 61 - bits);
  }
  p.info = info;
  p.tdbg = getenv("ANCKA_DISC_TIMING") ? (unsigned long long*)(info + 8 + 2 * (size_t)max_iter + 2 * (size_t)k * k) : nullptr;
  p.groups = disc_groups(k, (int)(col0 & 3));
  p.dbuf = disc_smem(k, p.groups, (int)(col0 & 3), 1) <= 200 * 1024 ? 1 : 0;
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "discretize: workspace too small");
  auto st = as_stream(stream);
  ANCKA_CUDA(cudaMemsetAsync(info, 0, sizeof(double) * (8 + 2 * (size_t)max_iter + 2 * (size_t)k * k + (p.tdbg ? 16 : 0)), st));
  for (int r = 0; r < 2; ++r) {
    ANCKA_CUDA(cudaMemsetAsync(pr[r].gfx, 0, sizeof(unsigned long long) * 3 * ((size_t)k * k + k), st));
    pr[r].fx_scale = p.fx_scale;
    pr[r].info = p.info;
    pr[r].tdbg = p.tdbg;
    pr[r].groups = p.groups;
    pr[r].dbuf = p.dbuf;
  }
  if (!disc_split(n, k)) {
    DiscParams q = pr[0];
    q.run_lo = 0;
    q.run_hi = 2;
    return launch_disc_k(q, k, col0, st, 1);
  }
  DiscSide* side = nullptr;
  ANCKA_TRY(disc_side(&side));
  // run 0 (identity start) writes labels_run0, run 1 (prototype) the output
  DiscParams a = pr[0], b = pr[1];
  a.run_lo = 0; a.run_hi = 1; a.labels = p.labels_run0;
  b.run_lo = 1; b.run_hi = 2;
  ANCKA_CUDA(cudaEventRecord(side->fork, st));
  ANCKA_CUDA(cudaStreamWaitEvent(side->s, side->fork, 0));
  ANCKA_TRY(launch_disc_k(b, k, col0, side->s, 2));
  ANCKA_TRY(launch_disc_k(a, k, col0, st, 2));
  ANCKA_CUDA(cudaEventRecord(side->join, side->s));
  ANCKA_CUDA(cudaStreamWaitEvent(st, side->join, 0));
  const int fg = (int)std::min<int64_t>(ceil_div(n, 256), 2 * kNumSMs);
  discretize_finish_kernel<<<fg, 256, 0, st>>>(p.fin, info, p.labels_run0, labels_out, n);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}
