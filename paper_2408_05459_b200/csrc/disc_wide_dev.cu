// Discretisation for wide blocks (64 < k <= 192: Papers100M's k = 172),
// entirely on the device: engine.py:162-263 -- alternating argmax rounding /
// Procrustes rotation from the identity and the prototype start, with the
// empty-cluster reseed -- as a short chain of kernels per round.  A host loop
// launches rounds and reads one device flag every kRoundsPerSync rounds; there
// is no host SVD and no per-round read-back.  Every kernel of a round returns
// at once after its start has converged.
//
//   dw_score    q~ R on tensor cores (mma.sync m16n8k16: q_hi R_hi + q_hi R_lo
//               + q_lo R_hi, f32 accumulation), a warp per 16 rows, first-max
//               argmax; a row whose winner does not beat the runner-up by the
//               certified error bound is rescored in f64 by the warp, so every
//               label is the f64 argmax of the iterate.  Moved rows -> a list.
//   dw_carry    totals <- previous totals (zero for a full recount)
//   dw_full     full recount (first round, or many moved rows): column blocks
//               of 32, shared-memory partials, one flush per CTA
//   dw_delta    moved rows: +fx(q~_i) to the new cluster, -fx to the old one
//   dw_reseed   (cooperative) only when a cluster is empty: exact f64 margins,
//               then _reseed_empty_columns one column at a time
//   dw_polar    (cooperative, one CTA per 16 x 16 tile of the kq x kq block)
//               M = Y~^T Q~ from the totals, polar factor of M^T by
//               Newton-Schulz in f64, objective n - 2 tr(X M), convergence,
//               next rotation (f64 and split-fp16 MMA fragments)
//
// Cluster totals are 64-bit fixed point summed element by element (the same
// integer for the same q~ entry every round), so carried totals plus moved
// rows' deltas are exactly the integers of a recount, and every reduction
// has a fixed order: the result is bit-reproducible.
#include <cooperative_groups.h>
#include <cuda_fp16.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace ancka {
namespace dw {

constexpr int kT = 256;              // threads per CTA (all kernels)
constexpr int kMaxK = 192;           // kq <= 192: R fragments fit shared memory
constexpr int kRoundsPerSync = 8;

struct Ctl {
  int done[2], rounds[2], conv[2], empties[2];
  int it;           // round within the current start
  int gr;           // global round counter: totals buffer gr % 3
  int nchg;         // moved rows this round
  int qs;           // quintic Newton-Schulz sweeps for the next polar factor
  int flags[3];     // Newton-Schulz "moved" flags (rotating)
  int zero_rows;
  int ns_total;
  int nlist;        // rows due for scoring this round (-1: all rows)
  int pad_;
  double obj_prev;
  double obj_last[2];
  double cdrift;    // cumulative rotation drift of the current start (row keys)
  int pause;        // row-partitioned mode: an empty cluster awaits the host reseed
  int pad2_;
};

struct Params {
  const float* Q;
  int64_t ldq, col0, n;
  int k, kq, nb8, max_iter;
  double tol;
  float cert;                  // certified score error bound x 2
  float* qn;                   // n x kq, q~ in f32 (zero padded)
  double* qinv;                // 1 / ||q_i|| (0 for zero rows)
  int32_t* labels;             // labels of the current start
  int32_t* chg_row;            // moved rows (capacity n)
  int32_t* chg_old;
  unsigned long long* tot;     // 3 x (k k + k) fixed-point totals
  double fx_scale;
  int fx_shift;
  double* R64;                 // k x k rotation used by the next scoring (row l, col j)
  uint4* Rfrag;                // (kq / 16) x nb8 x 32 split-fp16 B fragments
  double* W;                   // 5 x kq x kq polar workspace: M, X, Y, T, Xn
  double* part;                // per-CTA partials
  double* margin;              // n, exact second-best scores (reseed)
  double* proto_acc;           // n
  double* key;                 // n: drift level below which the row's label is certified
  int32_t* rid;                // n: rows due for scoring this round
  Ctl* ctl;
  double* info;
  // row-partitioned mode (dist.py): this rank holds global rows
  // [row0, row0 + n) of n_glob; `tots` receives the rank's current totals
  // and, after the caller's sum all-reduce, holds the global totals the
  // polar factor reads.  Single GPU: tots == nullptr, n_glob == n.
  int64_t n_glob, row0;
  unsigned long long* tots;
  double* rvec;                // k: a prototype row, summed over ranks by the caller
  double* locbest;             // 2: this rank's (value, global row) of a prototype pass
};

__device__ __forceinline__ int ld_vol(const int* p) { return *reinterpret_cast<const volatile int*>(p); }

__device__ __forceinline__ bool stopped(const Params& p, int run) {
  return ld_vol(&p.ctl->done[run]) || ld_vol(&p.ctl->pause);
}
// totals the rotation step reads: the global ones in the row-partitioned mode
__device__ __forceinline__ const unsigned long long* tot_glob(const Params& p, int gr) {
  return p.tots ? p.tots : p.tot + (size_t)(gr % 3) * (p.k * p.k + p.k);
}


__device__ __forceinline__ void mma_f16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
// x = hi + lo with hi = fp16(x), lo = fp16(x - hi), for an element pair
__device__ __forceinline__ void split_half2(float a, float b, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(a, b);
  const float2 hf = __half22float2(h);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = pack_half2(a - hf.x, b - hf.y);
}

// round(x * 2^sh) to int64 with integer operations (|x| <= 1, sh <= 61);
// the same integer for the same x every time
__device__ __forceinline__ long long fx_round(float x, int sh) {
  const uint32_t b = __float_as_uint(x);
  const int e = (int)((b >> 23) & 0xffu);
  const uint32_t m = (b & 0x7fffffu) | 0x800000u;
  const int s = e - 150 + sh;
  long long v;
  if (e == 0 || s <= -25) {
    v = 0;
  } else if (s >= 0) {
    v = (long long)m << s;
  } else {
    const int r = -s;
    const uint32_t q = m >> r, rem = m & ((1u << r) - 1u), half = 1u << (r - 1);
    v = (long long)(q + ((rem > half || (rem == half && (q & 1u))) ? 1u : 0u));
  }
  return (b >> 31) ? -v : v;
}
// 64-bit add to a shared cell (lo, hi words) with two native 32-bit atomics
__device__ __forceinline__ void sadd64(unsigned* cell, long long v) {
  const unsigned lo = (unsigned)v, hi = (unsigned)((unsigned long long)v >> 32);
  const unsigned old = atomicAdd(cell, lo);
  const unsigned h = hi + ((old + lo < old) ? 1u : 0u);
  if (h) atomicAdd(cell + 1, h);
}

// Fragment entry e of the rotation R (f64, k x k) as split fp16 pairs:
// Rfrag[(ks * nb8 + nb) * 32 + lane] = (hi pair 0, hi pair 1, lo pair 0,
// lo pair 1), pair 0 = (R[16ks+2t][8nb+g], R[16ks+2t+1][8nb+g]), pair 1 the
// rows + 8 (g = lane / 4, t = lane % 4): the m16n8k16 B-operand layout.
template <typename Get>
__device__ __forceinline__ uint4 frag_entry(int e, int k, int nb8, Get get) {
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
  return v;
}

// f64 scores of row i against R64 (lanes over columns j = lane + 32 m, l
// summed in ascending order), first-max argmax and the second-best score
__device__ void exact_row(const Params& p, int64_t i, int& lab, double& second_out,
                          double* margin_out = nullptr) {
  const int k = p.k, lane = threadIdx.x & 31;
  const float* src = p.Q + i * p.ldq + p.col0;
  const double inv = p.qinv[i];
  double ql[kMaxK / 32], s[kMaxK / 32];
#pragma unroll
  for (int m = 0; m < kMaxK / 32; ++m) {
    const int l = lane + 32 * m;
    ql[m] = l < k ? (double)src[l] * inv : 0.0;
    s[m] = 0.0;
  }
#pragma unroll
  for (int mm = 0; mm < kMaxK / 32; ++mm) {
    if (32 * mm >= k) break;
    const int lend = min(32, k - 32 * mm);
    for (int ll = 0; ll < lend; ++ll) {
      const double qv = __shfl_sync(0xffffffffu, ql[mm], ll);
      const double* Rl = p.R64 + (size_t)(32 * mm + ll) * k;
#pragma unroll
      for (int m = 0; m < kMaxK / 32; ++m) {
        const int j = lane + 32 * m;
        if (j < k) s[m] = fma(qv, __ldg(Rl + j), s[m]);
      }
    }
  }
  double best = -INFINITY, second = -INFINITY;
  int bi = 0x7fffffff;
#pragma unroll
  for (int m = 0; m < kMaxK / 32; ++m) {
    const int j = lane + 32 * m;
    if (j < k) {
      const double v = s[m];
      if (v > best) { second = best; best = v; bi = j; } else if (v > second) second = v;
    }
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
  second_out = second;
  if (margin_out) *margin_out = best - second;
}

// ----------------------------------------------------------- normalise ---
__global__ void dw_normalize(Params p) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int k = p.k, kq = p.kq;
  int zeros = 0;
  for (int64_t i = w0; i < p.n; i += nw) {
    const float* q = p.Q + i * p.ldq + p.col0;
    double s2 = 0.0;
    for (int c = lane; c < k; c += 32) {
      const double v = (double)q[c];
      s2 += v * v;
    }
    const double nrm = sqrt(warp_sum(s2));
    const double inv = nrm > 0 ? 1.0 / nrm : 0.0;
    for (int c = lane; c < kq; c += 32) p.qn[i * kq + c] = c < k ? (float)((double)q[c] * inv) : 0.f;
    if (lane == 0) {
      p.qinv[i] = inv;
      zeros += nrm == 0.0;
    }
  }
  if (lane == 0 && zeros) atomicAdd(&p.ctl->zero_rows, zeros);
}

// rotation = identity
__global__ void dw_identity(Params p) {
  const int k = p.k, ne = (p.kq / 16) * p.nb8 * 32;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k * k + ne; e += gridDim.x * blockDim.x) {
    if (e < k * k) p.R64[e] = (e / k == e % k) ? 1.0 : 0.0;
    else p.Rfrag[e - k * k] = frag_entry(e - k * k, k, p.nb8, [](int l, int j) { return l == j ? 1.0 : 0.0; });
  }
}

// ------------------------------------------------------------- scoring ---
// Rows due this round.  A row scored at cumulative rotation drift C0 with a
// certified margin m keeps its argmax while the drift since then stays
// below m / 2 (each score moves by at most max_j ||R'_j - R_j|| for a unit
// row): key = C0 + m / 2.  The first round of a start scores every row, and
// so does a round where most rows are due.
__global__ void dw_list(Params p, int run) {
  if (stopped(p, run)) return;
  if (ld_vol(&p.ctl->it) == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) p.ctl->nlist = -1;
    return;
  }
  const double c = *reinterpret_cast<volatile double*>(&p.ctl->cdrift);
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < p.n; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    const bool due = i < p.n && p.key[i] <= c;
    const unsigned m = __ballot_sync(0xffffffffu, due);
    int base = 0;
    if (lane == 0 && m) base = atomicAdd(&p.ctl->nlist, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (due) p.rid[base + __popc(m & ((1u << lane) - 1u))] = (int32_t)i;
  }
}

template <int NBMAX>
__global__ void __launch_bounds__(kT, 1) dw_score(Params p, int run, int first) {
  if (stopped(p, run)) return;
  extern __shared__ uint4 sRf[];
  const int k = p.k, kq = p.kq, ks16 = kq / 16, nb8 = p.nb8;
  for (int e = threadIdx.x; e < ks16 * nb8 * 32; e += kT) sRf[e] = p.Rfrag[e];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int64_t n = p.n;
  const int nl = ld_vol(&p.ctl->nlist);
  const bool list = nl >= 0 && 2 * (int64_t)nl <= n;
  const int64_t nrows = list ? nl : n;
  const int64_t nmb = ceil_div(nrows, 16);
  const double cdrift = *reinterpret_cast<volatile double*>(&p.ctl->cdrift);
  for (int64_t mb = (int64_t)blockIdx.x * (kT / 32) + warp; mb < nmb; mb += (int64_t)gridDim.x * (kT / 32)) {
    // the warp's 16 rows: slots mb * 16 + g and + 8 (rows of the list, or
    // consecutive rows); slots past the end read a valid row, write nothing
    const int64_t s0 = mb * 16 + g, s1 = s0 + 8;
    const int64_t r0 = s0 < nrows ? (list ? (int64_t)p.rid[s0] : s0) : n;
    const int64_t r1 = s1 < nrows ? (list ? (int64_t)p.rid[s1] : s1) : n;
    const int64_t c0 = r0 < n ? r0 : n - 1, c1 = r1 < n ? r1 : n - 1;   // clamped reads
    int old0 = -1, old1 = -1;
    if (!first && t == 0) {
      if (r0 < n) old0 = p.labels[r0];
      if (r1 < n) old1 = p.labels[r1];
    }
    float acc[NBMAX][4];
#pragma unroll
    for (int nb = 0; nb < NBMAX; ++nb)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[nb][c] = 0.f;
    const float* q0 = p.qn + c0 * kq + 2 * t;
    const float* q1 = p.qn + c1 * kq + 2 * t;
    float2 x[4];
    x[0] = *reinterpret_cast<const float2*>(q0);
    x[1] = *reinterpret_cast<const float2*>(q1);
    x[2] = *reinterpret_cast<const float2*>(q0 + 8);
    x[3] = *reinterpret_cast<const float2*>(q1 + 8);
#pragma unroll 1
    for (int ks = 0; ks < ks16; ++ks) {
      uint32_t ah[4], al[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) split_half2(x[q].x, x[q].y, ah[q], al[q]);
      if (ks + 1 < ks16) {            // next k-step's A elements (latency under the MMAs)
        const int o = (ks + 1) * 16;
        x[0] = *reinterpret_cast<const float2*>(q0 + o);
        x[1] = *reinterpret_cast<const float2*>(q1 + o);
        x[2] = *reinterpret_cast<const float2*>(q0 + o + 8);
        x[3] = *reinterpret_cast<const float2*>(q1 + o + 8);
      }
#pragma unroll
      for (int nb = 0; nb < NBMAX; ++nb) {
        if (nb < nb8) {
          const uint4 b = sRf[(ks * nb8 + nb) * 32 + lane];
          mma_f16(acc[nb], ah, b.x, b.y);
          mma_f16(acc[nb], ah, b.z, b.w);
          mma_f16(acc[nb], al, b.x, b.y);
        }
      }
    }
    int lab[2];
    bool flag[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float best = -INFINITY, second = -INFINITY;
      int bi = 0x7fffffff;
#pragma unroll
      for (int nb = 0; nb < NBMAX; ++nb)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int j = nb * 8 + 2 * t + c;
          const float v = (nb < nb8 && j < k) ? acc[nb][h * 2 + c] : -INFINITY;
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
      lab[h] = bi;
      flag[h] = !(best - second > p.cert);
      const int64_t rr = h == 0 ? r0 : r1;
      if (t == 0 && !flag[h] && rr < n) p.key[rr] = cdrift + 0.5 * ((double)best - (double)second - (double)p.cert);
    }
    // rows the margin does not certify: exact f64 rescoring by the warp
    const unsigned fm = __ballot_sync(0xffffffffu, t == 0 && ((flag[0] && r0 < n) || (flag[1] && r1 < n)));
    unsigned todo = fm;
    while (todo) {
      const int src = __ffs(todo) - 1;
      todo &= todo - 1;
      const int f0 = __shfl_sync(0xffffffffu, (int)flag[0], src);
      const int f1 = __shfl_sync(0xffffffffu, (int)flag[1], src);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t row = __shfl_sync(0xffffffffu, h == 0 ? r0 : r1, src);
        if (!(h == 0 ? f0 : f1) || row >= n) continue;
        int el;
        double sec, marg;
        exact_row(p, row, el, sec, &marg);
        if (lane == src) {
          lab[h] = el;
          p.key[row] = cdrift + 0.5 * marg;
        }
      }
    }
    // labels, moved rows
    bool mv[2] = {false, false};
    if (t == 0) {
      if (r0 < n) { p.labels[r0] = lab[0]; mv[0] = !first && lab[0] != old0; }
      if (r1 < n) { p.labels[r1] = lab[1]; mv[1] = !first && lab[1] != old1; }
    }
    if (!first) {
      const unsigned m0 = __ballot_sync(0xffffffffu, mv[0]), m1 = __ballot_sync(0xffffffffu, mv[1]);
      const int tot = __popc(m0) + __popc(m1);
      if (tot) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&p.ctl->nchg, tot);
        base = __shfl_sync(0xffffffffu, base, 0);
        const unsigned lt = (1u << lane) - 1u;
        if (mv[0]) {
          const int pos = base + __popc(m0 & lt);
          p.chg_row[pos] = (int32_t)r0;
          p.chg_old[pos] = old0;
        }
        if (mv[1]) {
          const int pos = base + __popc(m0) + __popc(m1 & lt);
          p.chg_row[pos] = (int32_t)r1;
          p.chg_old[pos] = old1;
        }
      }
    }
  }
}

// ------------------------------------------------------- cluster totals ---
__device__ __forceinline__ bool full_recount(const Params& p, int first) {
  return first || ld_vol(&p.ctl->nchg) > p.n / 16;
}

__global__ void dw_carry(Params p, int run, int first) {
  if (stopped(p, run)) return;
  const int ne = p.k * p.k + p.k, gr = ld_vol(&p.ctl->gr);
  unsigned long long* dst = p.tot + (size_t)(gr % 3) * ne;
  const unsigned long long* prev = p.tot + (size_t)((gr + 2) % 3) * ne;
  const bool full = full_recount(p, first);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += gridDim.x * blockDim.x)
    dst[e] = full ? 0ull : prev[e];
}

// grid (row blocks, ceil(k / 32)): warp per row, lane per column
__global__ void __launch_bounds__(kT) dw_full(Params p, int run, int first) {
  if (stopped(p, run) || !full_recount(p, first)) return;
  extern __shared__ unsigned sacc[];          // k x 32 cells (lo, hi) + k counts
  const int k = p.k, kq = p.kq, ne = k * k + k;
  unsigned* cnt = sacc + (size_t)k * 64;
  for (int e = threadIdx.x; e < k * 64 + k; e += kT) sacc[e] = 0u;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int j = blockIdx.y * 32 + lane;
  const bool do_cnt = blockIdx.y == 0;
  const int64_t rpb = ceil_div(p.n, gridDim.x);
  const int64_t a0 = (int64_t)blockIdx.x * rpb, a1 = lmin(p.n, a0 + rpb);
  for (int64_t i = a0 + w; i < a1; i += kT / 32) {
    const int l = p.labels[i];
    if (j < k) {
      const long long fx = fx_round(p.qn[i * kq + j], p.fx_shift);
      if (fx) sadd64(sacc + 2 * (l * 32 + lane), fx);
    }
    if (do_cnt && lane == 0) atomicAdd(&cnt[l], 1u);
  }
  __syncthreads();
  unsigned long long* dst = p.tot + (size_t)(ld_vol(&p.ctl->gr) % 3) * ne;
  for (int e = threadIdx.x; e < k * 32; e += kT) {
    const int l = e / 32, jj = blockIdx.y * 32 + (e % 32);
    const unsigned long long v = (unsigned long long)sacc[2 * e] | ((unsigned long long)sacc[2 * e + 1] << 32);
    if (jj < k && v) atomicAdd(dst + (size_t)l * k + jj, v);
  }
  if (do_cnt)
    for (int e = threadIdx.x; e < k; e += kT)
      if (cnt[e]) atomicAdd(dst + (size_t)k * k + e, (unsigned long long)cnt[e]);
}

// warp per moved row
__global__ void __launch_bounds__(kT) dw_delta(Params p, int run, int first) {
  if (stopped(p, run) || full_recount(p, first)) return;
  const int k = p.k, kq = p.kq, ne = k * k + k, nchg = ld_vol(&p.ctl->nchg);
  unsigned long long* dst = p.tot + (size_t)(ld_vol(&p.ctl->gr) % 3) * ne;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * kT + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * kT) >> 5;
  for (int64_t c = w0; c < nchg; c += nw) {
    const int64_t i = p.chg_row[c];
    const int o = p.chg_old[c], l = p.labels[i];
    for (int j = lane; j < k; j += 32) {
      const long long fx = fx_round(p.qn[i * kq + j], p.fx_shift);
      if (fx) {
        atomicAdd(dst + (size_t)l * k + j, (unsigned long long)fx);
        atomicAdd(dst + (size_t)o * k + j, (unsigned long long)(-fx));
      }
    }
    if (lane == 0) {
      atomicAdd(dst + (size_t)k * k + l, 1ull);
      atomicAdd(dst + (size_t)k * k + o, ~0ull);
    }
  }
}

__device__ double block_max(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmax(r, red[w]);
  __syncthreads();
  return r;
}

// --------------------------------------------------- block argmax helpers ---
// (value, index) arg-best of a CTA, ties to the smaller index; want_max or min
template <int NT = kT>
__device__ void block_best(double v, long long id, bool want_max, double* sv, long long* si,
                           double& v_out, long long& i_out) {
  sv[threadIdx.x] = v;
  si[threadIdx.x] = id;
  __syncthreads();
  for (int s = NT / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double v2 = sv[threadIdx.x + s], v1 = sv[threadIdx.x];
      const long long i2 = si[threadIdx.x + s], i1 = si[threadIdx.x];
      const bool take = i2 >= 0 && (i1 < 0 || (want_max ? v2 > v1 : v2 < v1) || (v2 == v1 && i2 < i1));
      if (take) { sv[threadIdx.x] = v2; si[threadIdx.x] = i2; }
    }
    __syncthreads();
  }
  v_out = sv[0];
  i_out = si[0];
  __syncthreads();
}
// global arg-best from per-CTA (value, index) partials, same order in every CTA
template <int NT = kT>
__device__ void grid_best(const double* part, int nb, bool want_max, double* sv, long long* si,
                          double& v_out, long long& i_out) {
  double v = 0.0;
  long long id = -1;
  for (int b = threadIdx.x; b < nb; b += NT) {
    const double v2 = __ldcg(part + 2 * b);
    const long long i2 = (long long)__ldcg(part + 2 * b + 1);
    const bool take = i2 >= 0 && (id < 0 || (want_max ? v2 > v : v2 < v) || (v2 == v && i2 < id));
    if (take) { v = v2; id = i2; }
  }
  block_best<NT>(v, id, want_max, sv, si, v_out, i_out);
}

// --------------------------------------------------------------- reseed ---
// _reseed_empty_columns (engine.py:162-180) when the totals show an empty
// cluster: exact second-best scores, then per empty column the movable row
// (cluster size >= 2) with the largest margin moves there; its fixed-point
// delta goes to the totals (owner CTA).
__global__ void __launch_bounds__(kT, 1) dw_reseed(Params p, int run) {
  if (stopped(p, run)) return;
  const int k = p.k, kq = p.kq, ne = k * k + k;
  if (k < 2) return;
  cg::grid_group grid = cg::this_grid();
  __shared__ long long sizes[kMaxK];
  __shared__ double sv[kT];
  __shared__ long long si[kT];
  __shared__ int s_empty;
  unsigned long long* tot = p.tot + (size_t)(ld_vol(&p.ctl->gr) % 3) * ne;
  if (threadIdx.x == 0) s_empty = 0;
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += kT) {
    sizes[c] = (long long)__ldcg(tot + (size_t)k * k + c);
    if (sizes[c] == 0) atomicAdd(&s_empty, 1);
  }
  __syncthreads();
  if (s_empty == 0) return;                       // the same decision in every CTA
  const int64_t rpb = ceil_div(p.n, gridDim.x);
  const int64_t a0 = (int64_t)blockIdx.x * rpb, a1 = lmin(p.n, a0 + rpb);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t i = a0 + warp; i < a1; i += kT / 32) {   // exact margins (np.partition [-2])
    int lab;
    double sec;
    exact_row(p, i, lab, sec);
    if (lane == 0) p.margin[i] = sec;
  }
  __syncthreads();
  int buf = 0;
  for (int c = 0; c < k; ++c) {
    if (sizes[c] != 0) continue;
    double best = 0.0;
    long long bi = -1;
    for (int64_t i = a0 + threadIdx.x; i < a1; i += kT) {
      const int l = p.labels[i];
      if (sizes[l] >= 2) {
        const double m = p.margin[i];
        if (bi < 0 || m > best) { best = m; bi = i; }
      }
    }
    double v;
    long long idx;
    block_best(best, bi, true, sv, si, v, idx);
    double* part = p.part + (size_t)buf * gridDim.x * 2;
    if (threadIdx.x == 0) {
      part[2 * blockIdx.x] = v;
      part[2 * blockIdx.x + 1] = (double)idx;
    }
    grid.sync();
    grid_best(part, gridDim.x, true, sv, si, v, idx);
    buf ^= 1;
    if (idx < 0) break;                               // no movable node left
    const bool owner = idx >= a0 && idx < a1;
    const int old = owner ? p.labels[idx] : 0;
    __syncthreads();
    if (owner) {
      for (int j = threadIdx.x; j < k; j += kT) {
        const long long fx = fx_round(p.qn[idx * kq + j], p.fx_shift);
        if (fx) {
          atomicAdd(tot + (size_t)c * k + j, (unsigned long long)fx);
          atomicAdd(tot + (size_t)old * k + j, (unsigned long long)(-fx));
        }
      }
      if (threadIdx.x == 0) {
        atomicAdd(tot + (size_t)k * k + c, 1ull);
        atomicAdd(tot + (size_t)k * k + old, ~0ull);
        p.labels[idx] = c;
        p.key[idx] = -INFINITY;                       // scored again next round
        p.part[4 * gridDim.x] = (double)old;          // the other CTAs learn the donor
      }
    }
    grid.sync();
    const int donor = (int)__ldcg(p.part + 4 * gridDim.x);
    if (threadIdx.x == 0) {
      sizes[donor] -= 1;
      sizes[c] += 1;
    }
    __syncthreads();
    grid.sync();                                      // donor slot read before its next write
  }
}

// ---------------------------------------------------------------- polar ---
// C tile (16 x 16 at (by, bx)) of op(A) B over kq (zero padded), K in chunks
// of 16 staged in shared memory; global operands read through L2 (other CTAs
// write them between grid barriers)
template <bool TA>
__device__ __forceinline__ double tile_mm(const double* A, const double* B, int kq, int by, int bx,
                                          double (*sA)[17], double (*sB)[17]) {
  const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
  double acc = 0.0;
  for (int c = 0; c < kq; c += 16) {
    sA[ty][tx] = TA ? __ldcg(A + (size_t)(c + tx) * kq + 16 * by + ty) : __ldcg(A + (size_t)(16 * by + ty) * kq + c + tx);
    sB[ty][tx] = __ldcg(B + (size_t)(c + ty) * kq + 16 * bx + tx);
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; ++u) acc = fma(sA[ty][u], sB[u][tx], acc);
    __syncthreads();
  }
  return acc;
}

__global__ void __launch_bounds__(kT, 1) dw_polar(Params p, int run) {
  if (stopped(p, run)) return;
  cg::grid_group grid = cg::this_grid();
  const int k = p.k, kq = p.kq, kk = k * k, ne = kk + k, tpr = kq / 16;
  const int by = blockIdx.x / tpr, bx = blockIdx.x % tpr, G = gridDim.x;
  const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
  const int a = 16 * by + ty, b = 16 * bx + tx;          // this thread's element
  const size_t KQ = (size_t)kq * kq;
  double* M = p.W;
  double* X = p.W + KQ;
  double* Y = p.W + 2 * KQ;
  double* T = p.W + 3 * KQ;
  double* Xn = p.W + 4 * KQ;
  __shared__ double sA[16][17], sB[16][17];
  __shared__ double red[32];
  __shared__ long long ssz[kMaxK];
  const int it = ld_vol(&p.ctl->it), gr = ld_vol(&p.ctl->gr), qs = ld_vol(&p.ctl->qs);
  const double obj_prev = *reinterpret_cast<volatile double*>(&p.ctl->obj_prev);
  const unsigned long long* tot = tot_glob(p, gr);
  for (int c = threadIdx.x; c < k; c += kT) ssz[c] = (long long)__ldcg(tot + kk + c);
  __syncthreads();
  // M = Y~^T Q~: cluster sums / sizes (engine.py:196-200), kq x kq zero padded
  double m = 0.0;
  if (a < k && b < k && ssz[a] > 0)
    m = ((double)(long long)__ldcg(tot + (size_t)a * k + b) / p.fx_scale) / (double)ssz[a];
  M[(size_t)a * kq + b] = m;
  // sigma_max bound min(||M||_F, sqrt(||M||_1 ||M||_inf)) from per-CTA partials
  {
    double* pf = p.part;                      // G
    double* prow = p.part + G;                // tpr x kq  (per column-tile row sums)
    double* pcol = prow + (size_t)tpr * kq;   // tpr x kq  (per row-tile column sums)
    const double f = block_sum(m * m, red);
    if (threadIdx.x == 0) pf[blockIdx.x] = f;
    // row a: |m| summed over this tile's 16 columns; column b likewise
    sA[ty][tx] = fabs(m);
    __syncthreads();
    if (threadIdx.x < 16) {
      double rs = 0.0, cs = 0.0;
      for (int u = 0; u < 16; ++u) { rs += sA[threadIdx.x][u]; cs += sA[u][threadIdx.x]; }
      prow[(size_t)bx * kq + 16 * by + threadIdx.x] = rs;
      pcol[(size_t)by * kq + 16 * bx + threadIdx.x] = cs;
    }
    grid.sync();
    double fr = 0.0, rmax = 0.0, cmax = 0.0;
    for (int c2 = 0; c2 < G; ++c2) fr += __ldcg(pf + c2);
    for (int r = threadIdx.x; r < kq; r += kT) {
      double rs = 0.0, cs = 0.0;
      for (int t2 = 0; t2 < tpr; ++t2) {
        rs += __ldcg(prow + (size_t)t2 * kq + r);
        cs += __ldcg(pcol + (size_t)t2 * kq + r);
      }
      rmax = fmax(rmax, rs);
      cmax = fmax(cmax, cs);
    }
    // block max
    __shared__ double smx[2][kT];
    smx[0][threadIdx.x] = rmax;
    smx[1][threadIdx.x] = cmax;
    __syncthreads();
    for (int s = kT / 2; s > 0; s >>= 1) {
      if (threadIdx.x < s) {
        smx[0][threadIdx.x] = fmax(smx[0][threadIdx.x], smx[0][threadIdx.x + s]);
        smx[1][threadIdx.x] = fmax(smx[1][threadIdx.x], smx[1][threadIdx.x + s]);
      }
      __syncthreads();
    }
    const double sb = fmin(sqrt(fr), sqrt(smx[0][0] * smx[1][0]));
    const double inv = sb > 0 ? 1.0 / sb : 0.0;
    __syncthreads();
    X[(size_t)b * kq + a] = m * inv;           // X0 = M^T / sb (this CTA writes the transposed tile)
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) p.ctl->flags[0] = p.ctl->flags[1] = p.ctl->flags[2] = 0;
  grid.sync();
  // Newton-Schulz: quintic sweeps X <- X (a I + b Y + c Y^2), then cubic
  // X <- 1.5 X - 0.5 X (X^T X) until no entry moves more than 1e-14 k
  int nsit = 0;
  for (int q = 0; q < qs; ++q, ++nsit) {
    const double y = tile_mm<true>(X, X, kq, by, bx, sA, sB);
    Y[(size_t)a * kq + b] = y;
    grid.sync();
    const double y2 = tile_mm<false>(Y, Y, kq, by, bx, sA, sB);
    T[(size_t)a * kq + b] = -4.7750 * y + 2.0315 * y2 + (a == b ? 3.4445 : 0.0);
    grid.sync();
    const double x = tile_mm<false>(X, T, kq, by, bx, sA, sB);
    Xn[(size_t)a * kq + b] = x;
    grid.sync();
    double* sw = X; X = Xn; Xn = sw;
  }
  int cub = 0;
  for (; cub < 100; ++cub) {
    const double y = tile_mm<true>(X, X, kq, by, bx, sA, sB);
    Y[(size_t)a * kq + b] = y;
    // flags[(cub + 1) % 3] was last read after the barrier closing step cub - 2
    if (blockIdx.x == 0 && threadIdx.x == 0) p.ctl->flags[(cub + 1) % 3] = 0;
    grid.sync();
    const double xy = tile_mm<false>(X, Y, kq, by, bx, sA, sB);
    const double xo = __ldcg(X + (size_t)a * kq + b);
    const double xn = 1.5 * xo - 0.5 * xy;
    Xn[(size_t)a * kq + b] = xn;
    const int moved = __syncthreads_or(fabs(xn - xo) > 1e-14 * k);
    if (moved && threadIdx.x == 0) atomicOr(&p.ctl->flags[cub % 3], 1);
    grid.sync();
    double* sw = X; X = Xn; Xn = sw;
    if (!ld_vol(&p.ctl->flags[cub % 3])) { ++cub; break; }
  }
  nsit += cub;
  // tr(X M) = sum_{a,b} X[a][b] M[b][a]; objective n - 2 tr (engine.py:201-202)
  const double xab = __ldcg(X + (size_t)a * kq + b);
  const double tpart = block_sum(xab * __ldcg(M + (size_t)b * kq + a), red);
  double* ptr = p.part + G + 2 * (size_t)tpr * kq;     // after the norm partials
  if (threadIdx.x == 0) ptr[blockIdx.x] = tpart;
  grid.sync();
  double ssum = 0.0;
  for (int c2 = 0; c2 < G; ++c2) ssum += __ldcg(ptr + c2);
  const double obj = (double)p.n_glob - 2.0 * ssum;
  const bool conv = it >= 1 && fabs(obj - obj_prev) < p.tol;
  const bool done = conv || it + 1 == p.max_iter;
  // rotation drift max_j ||X_j - R_j|| (row keys): per-CTA column partials
  // of this tile, summed over row tiles in a fixed order
  double dmax = 0.0;
  if (!done) {
    double* pd = ptr + G;                       // tpr x kq
    const double dv = (a < k && b < k) ? xab - p.R64[(size_t)a * k + b] : 0.0;
    sA[ty][tx] = dv * dv;
    __syncthreads();
    if (threadIdx.x < 16) {
      double cs = 0.0;
      for (int u = 0; u < 16; ++u) cs += sA[u][threadIdx.x];
      pd[(size_t)by * kq + 16 * bx + threadIdx.x] = cs;
    }
    __syncthreads();
    grid.sync();
    for (int c2 = threadIdx.x; c2 < k; c2 += kT) {
      double cs = 0.0;
      for (int t2 = 0; t2 < tpr; ++t2) cs += __ldcg(pd + (size_t)t2 * kq + c2);
      dmax = fmax(dmax, sqrt(cs));
    }
    dmax = block_max(dmax, red);
  }
  if (!done) {   // next rotation R = V U^T (engine.py:205): this CTA's tile of X
    sA[ty][tx] = xab;
    __syncthreads();
    if (a < k && b < k) p.R64[(size_t)a * k + b] = xab;
    if (threadIdx.x < 64) {                 // fragments of rows ks = by, columns nb = 2 bx, 2 bx + 1
      const int nb = 2 * bx + (threadIdx.x >> 5), ln = threadIdx.x & 31;
      if (nb < p.nb8) {
        const int e = (by * p.nb8 + nb) * 32 + ln;
        p.Rfrag[e] = frag_entry(e, k, p.nb8, [&](int l, int j) { return sA[l - 16 * by][j - 16 * bx]; });
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p.info[8 + (size_t)run * p.max_iter + it] = obj;
    Ctl* c = p.ctl;
    c->obj_prev = obj;
    c->obj_last[run] = obj;
    if (!done) c->cdrift += dmax * (1.0 + 1e-6) + 1e-14;   // rows of norm 1 + O(2^-24), f64 rounding
    c->nlist = 0;
    c->it = it + 1;
    c->gr = gr + 1;
    c->nchg = 0;
    c->ns_total += nsit;
    // quintic sweeps for the next round: each replaces ~3 cubic steps
    c->qs = cub > 7 ? qs + (cub - 5) / 3 : (cub < 5 && qs > 0 ? qs - 1 : qs);
    if (c->qs > 12) c->qs = 12;
    if (done) {
      int e0 = 0;
      for (int cc = 0; cc < k; ++cc) e0 += ssz[cc] == 0;
      c->empties[run] = e0;
      c->rounds[run] = it + 1;
      c->conv[run] = conv ? 1 : 0;
      c->done[run] = 1;
    }
  }
}

// ------------------------------------------------------------ prototype ---
// _prototype_rotation (engine.py:209-218): R[:, 0] = q~_0; pass j adds
// |q~ . R[:, j-1]| to every row's running sum and R[:, j] = q~ of the first
// row with the smallest sum.  q~ in f64 (Q / ||Q||).
constexpr int kTP = 512;          // prototype kernel: more rows in flight per SM
__global__ void __launch_bounds__(kTP, 1) dw_proto(Params p) {
  cg::grid_group grid = cg::this_grid();
  const int k = p.k;
  __shared__ double r[kMaxK];
  __shared__ double sv[kTP];
  __shared__ long long si[kTP];
  const int64_t rpb = ceil_div(p.n, gridDim.x);
  const int64_t a0 = (int64_t)blockIdx.x * rpb, a1 = lmin(p.n, a0 + rpb);
  auto load_row = [&](int64_t i) {
    const float* src = p.Q + i * p.ldq + p.col0;
    const double inv = p.qinv[i];
    for (int l = threadIdx.x; l < k; l += kTP) r[l] = (double)src[l] * inv;
  };
  load_row(0);
  for (int64_t i = a0 + threadIdx.x; i < a1; i += kTP) p.proto_acc[i] = 0.0;
  __syncthreads();
  if (blockIdx.x == 0)
    for (int l = threadIdx.x; l < k; l += kTP) p.R64[(size_t)l * k] = r[l];
  int buf = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = 1; j < k; ++j) {
    // a warp per 32 consecutive rows: each row's dot product with lanes over
    // columns (coalesced reads, fixed shuffle-tree sum), lane r keeps row r's;
    // the running sums and 1/||q|| of the 32 rows load coalesced up front
    double best = 0.0;
    long long bi = -1;
    for (int64_t base = a0 + (int64_t)warp * 32; base < a1; base += (int64_t)(kTP / 32) * 32) {
      const int64_t me = base + lane;
      const bool ok = me < a1;
      const double acc0 = ok ? p.proto_acc[me] : 0.0;
      const double inv = ok ? p.qinv[me] : 0.0;
      const int nr = (int)lmin(32, a1 - base);
      double mine = 0.0;
      for (int rr = 0; rr < nr; rr += 4) {      // four rows in flight
        double d[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float* src = p.Q + (base + min(rr + u, nr - 1)) * p.ldq + p.col0;
          d[u] = 0.0;
#pragma unroll
          for (int m = 0; m < kMaxK / 32; ++m) {
            const int l = lane + 32 * m;
            if (l < k) d[u] = fma((double)src[l], r[l], d[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          d[u] = warp_sum(d[u]);
          if (lane == rr + u) mine = d[u];
        }
      }
      if (ok) {
        const double av = acc0 + fabs(mine * inv);
        p.proto_acc[me] = av;
        if (bi < 0 || av < best) { best = av; bi = me; }
      }
    }
    double v;
    long long idx;
    block_best<kTP>(best, bi, false, sv, si, v, idx);
    double* part = p.part + (size_t)buf * gridDim.x * 2;
    if (threadIdx.x == 0) {
      part[2 * blockIdx.x] = v;
      part[2 * blockIdx.x + 1] = (double)idx;
    }
    grid.sync();
    grid_best<kTP>(part, gridDim.x, false, sv, si, v, idx);
    buf ^= 1;
    load_row(idx < 0 ? 0 : idx);
    __syncthreads();
    if (blockIdx.x == 0)
      for (int l = threadIdx.x; l < k; l += kTP) p.R64[(size_t)l * k + j] = r[l];
  }
  grid.sync();
  const int ne = (p.kq / 16) * p.nb8 * 32;
  for (int e = blockIdx.x * kTP + threadIdx.x; e < ne; e += gridDim.x * kTP)
    p.Rfrag[e] = frag_entry(e, k, p.nb8, [&](int l, int jj) { return __ldcg(p.R64 + (size_t)l * k + jj); });
}

// winner (identity unless the prototype start is lower by more than 1e-15,
// engine.py:247-253), labels and the info head
__global__ void dw_finish(Params p, const int32_t* labels_run0, int32_t* labels_out) {
  const Ctl* c = p.ctl;
  const int win = c->obj_last[1] < c->obj_last[0] - 1e-15 ? 1 : 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p.info[0] = c->obj_last[win];
    p.info[1] = c->rounds[win];
    p.info[2] = c->conv[win];
    p.info[3] = win;
    p.info[4] = c->empties[win];
    p.info[5] = c->zero_rows;
    p.info[6] = c->rounds[0];
    p.info[7] = c->rounds[1];
  }
  if (win == 0)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.n; i += (int64_t)gridDim.x * blockDim.x)
      labels_out[i] = labels_run0[i];
}

// ------------------------------------------------- row-partitioned mode ---
// (dist.py: the rank's rows are [row0, row0 + n) of n_glob; the caller sums
// `tots` and the prototype buffers over ranks between these kernels)

// this rank's current totals -> tots (the caller all-reduces them in place)
__global__ void dw_snap(Params p) {
  const int ne = p.k * p.k + p.k;
  const unsigned long long* src = p.tot + (size_t)(ld_vol(&p.ctl->gr) % 3) * ne;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += gridDim.x * blockDim.x)
    p.tots[e] = src[e];
}

// an empty cluster in the global totals pauses the rounds for the host reseed
__global__ void dw_check_empty(Params p, int run) {
  if (stopped(p, run) || p.k < 2) return;
  __shared__ int e;
  if (threadIdx.x == 0) e = 0;
  __syncthreads();
  for (int c = threadIdx.x; c < p.k; c += blockDim.x)
    if (p.tots[(size_t)p.k * p.k + c] == 0ull) atomicAdd(&e, 1);
  __syncthreads();
  if (threadIdx.x == 0 && e) p.ctl->pause = 1;
}

// exact second-best scores of the local rows (the reseed's margins)
__global__ void dw_margins(Params p) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < p.n; i += nw) {
    int lab;
    double sec;
    exact_row(p, i, lab, sec);
    if ((threadIdx.x & 31) == 0) p.margin[i] = sec;
  }
}

// move local row i to cluster c: labels and the rank's current totals
__global__ void dw_move_row(Params p, int64_t i, int c) {
  const int k = p.k, ne = k * k + k;
  unsigned long long* tot = p.tot + (size_t)(ld_vol(&p.ctl->gr) % 3) * ne;
  const int old = p.labels[i];
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    const long long fx = fx_round(p.qn[i * p.kq + j], p.fx_shift);
    if (fx) {
      atomicAdd(tot + (size_t)c * k + j, (unsigned long long)fx);
      atomicAdd(tot + (size_t)old * k + j, (unsigned long long)(-fx));
    }
  }
  if (threadIdx.x == 0) {
    atomicAdd(tot + (size_t)k * k + c, 1ull);
    atomicAdd(tot + (size_t)k * k + old, ~0ull);
    p.labels[i] = c;
    p.key[i] = -INFINITY;
  }
}

// prototype start, pass j (j >= 1): acc_i += |q~_i . R[:, j-1]| over the
// local rows with dw_proto's arithmetic, then per-CTA first minima
__global__ void __launch_bounds__(kTP) dw_ppass(Params p, int j) {
  const int k = p.k;
  __shared__ double r[kMaxK];
  __shared__ double sv[kTP];
  __shared__ long long si[kTP];
  for (int l = threadIdx.x; l < k; l += kTP) r[l] = p.R64[(size_t)l * k + j - 1];
  __syncthreads();
  const int64_t rpb = ceil_div(p.n, gridDim.x);
  const int64_t a0 = (int64_t)blockIdx.x * rpb, a1 = lmin(p.n, a0 + rpb);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double best = 0.0;
  long long bi = -1;
  for (int64_t base = a0 + (int64_t)warp * 32; base < a1; base += (int64_t)(kTP / 32) * 32) {
    const int64_t me = base + lane;
    const bool ok = me < a1;
    const double acc0 = ok ? p.proto_acc[me] : 0.0;
    const double inv = ok ? p.qinv[me] : 0.0;
    const int nr = (int)lmin(32, a1 - base);
    double mine = 0.0;
    for (int rr = 0; rr < nr; rr += 4) {
      double d[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float* src = p.Q + (base + min(rr + u, nr - 1)) * p.ldq + p.col0;
        d[u] = 0.0;
#pragma unroll
        for (int m = 0; m < kMaxK / 32; ++m) {
          const int l = lane + 32 * m;
          if (l < k) d[u] = fma((double)src[l], r[l], d[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        d[u] = warp_sum(d[u]);
        if (lane == rr + u) mine = d[u];
      }
    }
    if (ok) {
      const double av = acc0 + fabs(mine * inv);
      p.proto_acc[me] = av;
      if (bi < 0 || av < best) { best = av; bi = me; }
    }
  }
  double v;
  long long idx;
  block_best<kTP>(best, bi, false, sv, si, v, idx);
  if (threadIdx.x == 0) {
    p.part[2 * blockIdx.x] = v;
    p.part[2 * blockIdx.x + 1] = (double)idx;
  }
}

// the rank's first minimum -> locbest = (value, global row) (row -1: none)
__global__ void __launch_bounds__(kTP) dw_pbest(Params p, int nb) {
  __shared__ double sv[kTP];
  __shared__ long long si[kTP];
  double v;
  long long idx;
  grid_best<kTP>(p.part, nb, false, sv, si, v, idx);
  if (threadIdx.x == 0) {
    p.locbest[0] = idx < 0 ? INFINITY : v;
    p.locbest[1] = idx < 0 ? -1.0 : (double)(p.row0 + idx);
    p.locbest[2] = 0.0;
  }
}

// reseed candidates (_reseed_empty_columns, engine.py:162-180): per CTA the
// movable local row (cluster size >= 2 by the caller's global sizes) with
// the largest exact second-best score, ties to the smaller row
__global__ void __launch_bounds__(kT) dw_rcand(Params p, const long long* sizes) {
  __shared__ double sv[kT];
  __shared__ long long si[kT];
  const int64_t rpb = ceil_div(p.n, gridDim.x);
  const int64_t a0 = (int64_t)blockIdx.x * rpb, a1 = lmin(p.n, a0 + rpb);
  double best = 0.0;
  long long bi = -1;
  for (int64_t i = a0 + threadIdx.x; i < a1; i += kT) {
    if (sizes[p.labels[i]] >= 2) {
      const double m = p.margin[i];
      if (bi < 0 || m > best) { best = m; bi = i; }
    }
  }
  double v;
  long long idx;
  block_best(best, bi, true, sv, si, v, idx);
  if (threadIdx.x == 0) {
    p.part[2 * blockIdx.x] = v;
    p.part[2 * blockIdx.x + 1] = (double)idx;
  }
}

__global__ void __launch_bounds__(kT) dw_rbest(Params p, int nb) {
  __shared__ double sv[kT];
  __shared__ long long si[kT];
  double v;
  long long idx;
  grid_best(p.part, nb, true, sv, si, v, idx);
  if (threadIdx.x == 0) {
    p.locbest[0] = idx < 0 ? -INFINITY : v;
    p.locbest[1] = idx < 0 ? -1.0 : (double)(p.row0 + idx);
    p.locbest[2] = idx < 0 ? -1.0 : (double)p.labels[idx];
  }
}

// global first minimum over the ranks' (value, row) pairs (or the forced
// row); its owner writes q~ of that row (f64) into rvec, the others zeros
__global__ void dw_ppick(Params p, const double* gath, int world, long long force) {
  __shared__ long long g;
  if (threadIdx.x == 0) {
    long long gi = force;
    if (gi < 0) {
      double bv = 0.0;
      for (int w = 0; w < world; ++w) {
        const double v = gath[3 * w];
        const long long i = (long long)gath[3 * w + 1];
        if (i < 0) continue;
        if (gi < 0 || v < bv || (v == bv && i < gi)) { bv = v; gi = i; }
      }
      if (gi < 0) gi = 0;
    }
    g = gi;
  }
  __syncthreads();
  const long long li = g - p.row0;
  const bool own = li >= 0 && li < p.n;
  for (int l = threadIdx.x; l < p.k; l += blockDim.x)
    p.rvec[l] = own ? (double)p.Q[li * p.ldq + p.col0 + l] * p.qinv[li] : 0.0;
}

__global__ void dw_psetcol(Params p, int j) {
  for (int l = threadIdx.x; l < p.k; l += blockDim.x) p.R64[(size_t)l * p.k + j] = p.rvec[l];
}

__global__ void dw_pfrag(Params p) {
  const int ne = (p.kq / 16) * p.nb8 * 32;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += gridDim.x * blockDim.x)
    p.Rfrag[e] = frag_entry(e, p.k, p.nb8, [&](int l, int jj) { return p.R64[(size_t)l * p.k + jj]; });
}

// ctl -> flags[0..5] = done[0], done[1], pause, empties[0], empties[1], it
__global__ void dw_flags(Params p, int32_t* out) {
  if (threadIdx.x == 0) {
    out[0] = p.ctl->done[0];
    out[1] = p.ctl->done[1];
    out[2] = p.ctl->pause;
    out[3] = p.ctl->empties[0];
    out[4] = p.ctl->empties[1];
    out[5] = p.ctl->it;
  }
}

}  // namespace dw

// ------------------------------------------------------------------ host ---
namespace {
void carve_wide(Carver& cv, int64_t n, int k, dw::Params& p, int32_t** labels_run0) {
  const int kq = (k + 15) & ~15;
  *labels_run0 = cv.take<int32_t>(n);
  p.qn = cv.take<float>((size_t)n * kq);
  p.qinv = cv.take<double>(n);
  p.chg_row = cv.take<int32_t>(n);
  p.chg_old = cv.take<int32_t>(n);
  p.tot = cv.take<unsigned long long>((size_t)3 * (k * k + k));
  p.R64 = cv.take<double>((size_t)k * k);
  p.Rfrag = cv.take<uint4>((size_t)(kq / 16) * (kq / 8) * 32);
  p.W = cv.take<double>((size_t)5 * kq * kq);
  p.part = cv.take<double>((size_t)4 * 1024 + 16 + 3 * (size_t)kq * (kq / 16));
  p.margin = cv.take<double>(n);
  p.proto_acc = cv.take<double>(n);
  p.key = cv.take<double>(n);
  p.rid = cv.take<int32_t>(n);
  p.ctl = cv.take<dw::Ctl>(1);
}

template <int NB>
int launch_score(const dw::Params& p, int run, int first, cudaStream_t st) {
  const size_t smem = (size_t)(p.kq / 16) * p.nb8 * 32 * sizeof(uint4);
  ANCKA_CUDA(cudaFuncSetAttribute(dw::dw_score<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(ceil_div(p.n, 16), 8), kNumSMs));
  dw::dw_score<NB><<<grid, dw::kT, smem, st>>>(p, run, first);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

int coop(const void* fn, int grid, size_t smem, cudaStream_t st, void** args, int threads = dw::kT) {
  note_launch();
  ANCKA_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(threads), args, smem, st));
  return ANCKA_OK;
}

int launch_round(dw::Params& p, int run, int first, cudaStream_t st, int coop_grid) {
  dw::dw_list<<<2 * kNumSMs, dw::kT, 0, st>>>(p, run);
  ANCKA_LAUNCHED();
  ANCKA_TRY(p.nb8 <= 16 ? launch_score<16>(p, run, first, st) : launch_score<24>(p, run, first, st));
  const int ne = p.k * p.k + p.k;
  dw::dw_carry<<<(int)std::min<int64_t>(ceil_div(ne, dw::kT), 2 * kNumSMs), dw::kT, 0, st>>>(p, run, first);
  ANCKA_LAUNCHED();
  {
    const size_t smem = sizeof(unsigned) * ((size_t)p.k * 64 + p.k);
    ANCKA_CUDA(cudaFuncSetAttribute(dw::dw_full, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(p.n, 4096), kNumSMs));
    dw::dw_full<<<dim3(gx, (p.k + 31) / 32), dw::kT, smem, st>>>(p, run, first);
    ANCKA_LAUNCHED();
  }
  dw::dw_delta<<<2 * kNumSMs, dw::kT, 0, st>>>(p, run, first);
  ANCKA_LAUNCHED();
  {
    void* args[] = {&p, &run};
    ANCKA_TRY(coop((const void*)dw::dw_reseed, coop_grid, 0, st, args));
  }
  {
    void* args[] = {&p, &run};
    ANCKA_TRY(coop((const void*)dw::dw_polar, (p.kq / 16) * (p.kq / 16), 0, st, args));
  }
  return ANCKA_OK;
}
}  // namespace

size_t discretize_wide_workspace(int64_t n, int k) {
  Carver cv(nullptr, 0);
  dw::Params p{};
  int32_t* l0 = nullptr;
  carve_wide(cv, n, k, p, &l0);
  return cv.used;
}

int discretize_wide(const float* Q, int64_t ldq, int64_t col0, int64_t n, int k, int max_iter,
                    double tol, int32_t* labels_out, double* info, void* ws, size_t wsb,
                    cudaStream_t st) {
  ANCKA_REQUIRE(k > 8 && k <= dw::kMaxK, ANCKA_ERR_UNSUPPORTED,
                "discretize: device wide path supports 8 < k <= %d (got %d)", dw::kMaxK, k);
  ANCKA_REQUIRE(n >= 1 && n < (1ll << 31), ANCKA_ERR_UNSUPPORTED, "discretize: n=%lld", (long long)n);
  Carver cv(ws, wsb);
  dw::Params p{};
  int32_t* labels_run0 = nullptr;
  carve_wide(cv, n, k, p, &labels_run0);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "discretize: workspace too small");
  p.Q = Q; p.ldq = ldq; p.col0 = col0; p.n = n; p.k = k;
  p.n_glob = n;
  p.kq = (k + 15) & ~15;
  p.nb8 = p.kq / 8;
  p.max_iter = max_iter;
  p.tol = tol;
  // certified bound: split products 3 * 2^-22 + f32 accumulation of 3 kq
  // terms (2^-24 each, unit rows, orthogonal R) + the f32 copy of q~ (2^-24)
  p.cert = (float)(2.0 * (3.0 * p.kq * 0x1p-24 + 3.0 * 0x1p-22 + 0x1p-24));
  {
    int bits = 1;
    while ((1ll << bits) <= n) ++bits;
    p.fx_shift = 61 - bits;
    p.fx_scale = std::ldexp(1.0, p.fx_shift);
  }
  p.info = info;
  ANCKA_CUDA(cudaMemsetAsync(info, 0, sizeof(double) * (8 + 2 * (size_t)max_iter + 2 * (size_t)k * k), st));
  ANCKA_CUDA(cudaMemsetAsync(p.ctl, 0, sizeof(dw::Ctl), st));
  ANCKA_CUDA(cudaMemsetAsync(p.tot, 0, sizeof(unsigned long long) * 3 * ((size_t)k * k + k), st));
  ANCKA_CUDA(cudaMemsetAsync(p.W, 0, sizeof(double) * 5 * (size_t)p.kq * p.kq, st));
  dw::dw_normalize<<<(int)std::min<int64_t>(ceil_div(n * 32, dw::kT), 8 * kNumSMs), dw::kT, 0, st>>>(p);
  ANCKA_LAUNCHED();
  int coop_grid = 0;
  {
    int per_sm = 0;
    ANCKA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dw::dw_reseed, dw::kT, 0));
    int per_sm2 = 0;
    ANCKA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, dw::dw_proto, dw::kTP, 0));
    coop_grid = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)std::min(per_sm, per_sm2) * kNumSMs,
                                                              (int64_t)kNumSMs, ceil_div(n, dw::kT)}));
  }
  static int* done_host = nullptr;
  if (!done_host) ANCKA_CUDA(cudaMallocHost(&done_host, sizeof(int)));
  for (int run = 0; run < 2; ++run) {
    p.labels = run == 0 ? labels_run0 : labels_out;
    if (run == 0) {
      dw::dw_identity<<<8, dw::kT, 0, st>>>(p);
      ANCKA_LAUNCHED();
    } else {
      // the prototype start continues from run 0's labels and totals
      ANCKA_CUDA(cudaMemcpyAsync(labels_out, labels_run0, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
      ANCKA_CUDA(cudaMemsetAsync(&p.ctl->it, 0, sizeof(int), st));
      ANCKA_CUDA(cudaMemsetAsync(&p.ctl->cdrift, 0, sizeof(double), st));
      void* args[] = {&p};
      ANCKA_TRY(coop((const void*)dw::dw_proto, coop_grid, 0, st, args, dw::kTP));
    }
    for (int it0 = 0; it0 < max_iter; it0 += dw::kRoundsPerSync) {
      const int it1 = std::min(max_iter, it0 + dw::kRoundsPerSync);
      for (int it = it0; it < it1; ++it) ANCKA_TRY(launch_round(p, run, run == 0 && it == 0, st, coop_grid));
      ANCKA_CUDA(cudaMemcpyAsync(done_host, &p.ctl->done[run], sizeof(int), cudaMemcpyDeviceToHost, st));
      ANCKA_CUDA(cudaStreamSynchronize(st));
      if (*done_host) break;
    }
    // the rotation behind this start's final scores
    ANCKA_CUDA(cudaMemcpyAsync(info + 8 + 2 * (size_t)max_iter + (size_t)run * k * k, p.R64,
                               sizeof(double) * k * k, cudaMemcpyDeviceToDevice, st));
  }
  dw::dw_finish<<<(int)std::min<int64_t>(ceil_div(n, dw::kT), 2 * kNumSMs), dw::kT, 0, st>>>(p, labels_run0, labels_out);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

}  // namespace ancka

// --------------------------------------- row-partitioned mode: C entries ---
// One discretisation of a rank's rows, driven by the caller (dist.py) with
// collectives between the phases; the Params of a workspace are kept on the
// host, keyed by the workspace pointer, between ancka_discw_dist_init and
// the ANCKA_DW_FINISH op.
#include <mutex>
#include <unordered_map>

namespace {
struct DistDisc {
  ancka::dw::Params p;
  int32_t* labels_out;   // the caller's buffer: labels of the prototype start, then the winner
  int32_t* labels_run0;  // workspace: labels of the identity start
  int run;
};
std::mutex g_dw_mu;
std::unordered_map<const void*, DistDisc> g_dw;
}  // namespace

using namespace ancka;

extern "C" size_t ancka_discw_dist_workspace_size(int64_t n_loc, int32_t k) {
  return discretize_wide_workspace(n_loc < 1 ? 1 : n_loc, k);
}

extern "C" int ancka_discw_dist_init(const float* Q, int64_t ldq, int64_t col0, int64_t n_loc,
                                     int64_t n_glob, int64_t row0, int32_t k, int32_t max_iter,
                                     double tol, uint64_t* tots, double* rvec, double* locbest,
                                     int32_t* labels, double* info, void* ws, size_t wsb,
                                     ancka_stream_t stream) {
  ANCKA_REQUIRE(k > 8 && k <= dw::kMaxK, ANCKA_ERR_UNSUPPORTED,
                "discretize (row-partitioned): 8 < k <= %d (got %d)", dw::kMaxK, k);
  ANCKA_REQUIRE(n_loc >= 1 && n_glob >= n_loc && n_glob < (1ll << 31), ANCKA_ERR_ARG,
                "discretize (row-partitioned): n_loc=%lld n_glob=%lld", (long long)n_loc,
                (long long)n_glob);
  cudaStream_t st = as_stream(stream);
  Carver cv(ws, wsb);
  dw::Params p{};
  int32_t* labels_run0 = nullptr;
  carve_wide(cv, n_loc, k, p, &labels_run0);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "discretize (row-partitioned): workspace too small");
  p.Q = Q; p.ldq = ldq; p.col0 = col0; p.n = n_loc; p.k = k;
  p.n_glob = n_glob;
  p.row0 = row0;
  p.kq = (k + 15) & ~15;
  p.nb8 = p.kq / 8;
  p.max_iter = max_iter;
  p.tol = tol;
  p.cert = (float)(2.0 * (3.0 * p.kq * 0x1p-24 + 3.0 * 0x1p-22 + 0x1p-24));
  {
    int bits = 1;                       // sums over all n_glob rows fit 63 bits
    while ((1ll << bits) <= n_glob) ++bits;
    p.fx_shift = 61 - bits;
    p.fx_scale = std::ldexp(1.0, p.fx_shift);
  }
  p.info = info;
  p.tots = reinterpret_cast<unsigned long long*>(tots);
  p.rvec = rvec;
  p.locbest = locbest;
  p.labels = labels_run0;
  ANCKA_CUDA(cudaMemsetAsync(info, 0, sizeof(double) * (8 + 2 * (size_t)max_iter + 2 * (size_t)k * k), st));
  ANCKA_CUDA(cudaMemsetAsync(p.ctl, 0, sizeof(dw::Ctl), st));
  ANCKA_CUDA(cudaMemsetAsync(p.tot, 0, sizeof(unsigned long long) * 3 * ((size_t)k * k + k), st));
  ANCKA_CUDA(cudaMemsetAsync(p.W, 0, sizeof(double) * 5 * (size_t)p.kq * p.kq, st));
  dw::dw_normalize<<<(int)std::min<int64_t>(ceil_div(n_loc * 32, dw::kT), 8 * kNumSMs), dw::kT, 0, st>>>(p);
  ANCKA_LAUNCHED();
  std::lock_guard<std::mutex> lk(g_dw_mu);
  g_dw[ws] = DistDisc{p, labels, labels_run0, 0};
  return ANCKA_OK;
}

extern "C" int ancka_discw_dist_op(void* ws, int32_t op, int64_t a, int64_t b, const void* ptr,
                                   ancka_stream_t stream) {
  DistDisc d;
  {
    std::lock_guard<std::mutex> lk(g_dw_mu);
    auto it = g_dw.find(ws);
    ANCKA_REQUIRE(it != g_dw.end(), ANCKA_ERR_ARG, "discretize (row-partitioned): unknown workspace");
    if (op == ANCKA_DW_START) it->second.run = (int)a;
    d = it->second;
  }
  dw::Params p = d.p;
  int32_t* labels_out = d.labels_out;
  int32_t* labels_run0 = d.labels_run0;
  cudaStream_t st = as_stream(stream);
  const int run = (int)a;
  p.labels = d.run == 1 ? labels_out : labels_run0;
  switch (op) {
    case ANCKA_DW_START:             // a = run: 0 identity, 1 prototype setup
      if (run == 0) {
        dw::dw_identity<<<8, dw::kT, 0, st>>>(p);
        ANCKA_LAUNCHED();
      } else {
        ANCKA_CUDA(cudaMemcpyAsync(labels_out, labels_run0, sizeof(int32_t) * p.n, cudaMemcpyDeviceToDevice, st));
        ANCKA_CUDA(cudaMemsetAsync(&p.ctl->it, 0, sizeof(int), st));
        ANCKA_CUDA(cudaMemsetAsync(&p.ctl->cdrift, 0, sizeof(double), st));
        ANCKA_CUDA(cudaMemsetAsync(p.proto_acc, 0, sizeof(double) * p.n, st));
      }
      return ANCKA_OK;
    case ANCKA_DW_ROUND_LOCAL: {     // a = run, b = first round of the call
      dw::dw_list<<<2 * kNumSMs, dw::kT, 0, st>>>(p, run);
      ANCKA_LAUNCHED();
      ANCKA_TRY(p.nb8 <= 16 ? launch_score<16>(p, run, (int)b, st) : launch_score<24>(p, run, (int)b, st));
      const int ne = p.k * p.k + p.k;
      dw::dw_carry<<<(int)std::min<int64_t>(ceil_div(ne, dw::kT), 2 * kNumSMs), dw::kT, 0, st>>>(p, run, (int)b);
      ANCKA_LAUNCHED();
      {
        const size_t smem = sizeof(unsigned) * ((size_t)p.k * 64 + p.k);
        ANCKA_CUDA(cudaFuncSetAttribute(dw::dw_full, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(p.n, 4096), kNumSMs));
        dw::dw_full<<<dim3(gx, (p.k + 31) / 32), dw::kT, smem, st>>>(p, run, (int)b);
        ANCKA_LAUNCHED();
      }
      dw::dw_delta<<<2 * kNumSMs, dw::kT, 0, st>>>(p, run, (int)b);
      ANCKA_LAUNCHED();
      dw::dw_snap<<<(int)std::min<int64_t>(ceil_div(ne, dw::kT), 2 * kNumSMs), dw::kT, 0, st>>>(p);
      ANCKA_LAUNCHED();
      return ANCKA_OK;
    }
    case ANCKA_DW_SNAP: {
      const int ne = p.k * p.k + p.k;
      dw::dw_snap<<<(int)std::min<int64_t>(ceil_div(ne, dw::kT), 2 * kNumSMs), dw::kT, 0, st>>>(p);
      ANCKA_LAUNCHED();
      return ANCKA_OK;
    }
    case ANCKA_DW_CHECK_EMPTY:
      dw::dw_check_empty<<<1, dw::kT, 0, st>>>(p, run);
      ANCKA_LAUNCHED();
      return ANCKA_OK;
    case ANCKA_DW_POLAR: {
      void* args[] = {&p, const_cast<int*>(&run)};
      ANCKA_TRY(coop((const void*)dw::dw_polar, (p.kq / 16) * (p.kq / 16), 0, st, args));
      return ANCKA_OK;
    }
    case ANCKA_DW_CLEAR_PAUSE:
      ANCKA_CUDA(cudaMemsetAsync(&p.ctl->pause, 0, sizeof(int), st));
      return ANCKA_OK;
    case ANCKA_DW_MARGINS:
      dw::dw_margins<<<(int)std::min<int64_t>(ceil_div(p.n * 32, dw::kT), 8 * kNumSMs), dw::kT, 0, st>>>(p);
      ANCKA_LAUNCHED();
      return ANCKA_OK;
    case ANCKA_DW_MOVE_ROW:          // a = target cluster, b = local row
      dw::dw_move_row<<<1, dw::kT, 0, st>>>(p, b, (int)a);
      ANCKA_LAUNCHED();
      return ANCKA_OK;
    case ANCKA_DW_RESEED_CAND: {     // ptr = device int64[k] global cluster sizes
      const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(kNumSMs, ceil_div(p.n, dw::kT)));
      dw::dw_rcand<<<nb, dw::kT, 0, st>>>(p, static_cast<const long long*>(ptr));
      ANCKA_LAUNCHED();
      dw::dw_rbest<<<1, dw::kT, 0, st>>>(p, nb);
      ANCKA_LAUNCHED();
      return ANCKA_OK;
    }
    case ANCKA_DW_PROTO_PASS: {      // a = run (1), b = column j >= 1
      const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(kNumSMs, ceil_div(p.n, dw::kTP)));
      dw::dw_ppass<<<nb, dw::kTP, 0, st>>>(p, (int)b);
      ANCKA_LAUNCHED();
      dw::dw_pbest<<<1, dw::kTP, 0, st>>>(p, nb);
      ANCKA_LAUNCHED();
      return ANCKA_OK;
    }
    case ANCKA_DW_PROTO_PICK:        // b = forced global row (>= 0) or -1; ptr = gathered pairs, a = world
      dw::dw_ppick<<<1, 256, 0, st>>>(p, static_cast<const double*>(ptr), run, (long long)b);
      ANCKA_LAUNCHED();
      return ANCKA_OK;
    case ANCKA_DW_PROTO_SETCOL:      // b = column
      dw::dw_psetcol<<<1, 256, 0, st>>>(p, (int)b);
      ANCKA_LAUNCHED();
      if (b == p.k - 1 || p.k == 1) {
        dw::dw_pfrag<<<8, dw::kT, 0, st>>>(p);
        ANCKA_LAUNCHED();
      }
      return ANCKA_OK;
    case ANCKA_DW_FLAGS:             // ptr = int32[6] device
      dw::dw_flags<<<1, 32, 0, st>>>(p, static_cast<int32_t*>(const_cast<void*>(ptr)));
      ANCKA_LAUNCHED();
      return ANCKA_OK;
    case ANCKA_DW_FINISH: {          // labels_out <- winner; forget the workspace
      dw::dw_finish<<<(int)std::min<int64_t>(ceil_div(p.n, dw::kT), 2 * kNumSMs), dw::kT, 0, st>>>(
          p, labels_run0, labels_out);
      ANCKA_LAUNCHED();
      std::lock_guard<std::mutex> lk(g_dw_mu);
      g_dw.erase(ws);
      return ANCKA_OK;
    }
    default:
      break;
  }
  set_error("discretize (row-partitioned): unknown op %d", op);
  return ANCKA_ERR_ARG;
}
