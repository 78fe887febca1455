// Subsystem 4: SVD-based discretisation and argmax label assignment
// (engine.py:162-263) plus the post-pass repair check (engine.py:266-288).
//
// One cooperative persistent kernel runs both alternating-rounding starts
// (identity, prototype) for up to max_iter rounds without returning to the
// host.  Per round:
//   A  every CTA: row-normalise its rows of Q[:, col0:col0+k], score against R
//      (k x k, smem broadcast), first-max argmax + second-best margin, and
//      accumulate per-cluster column sums of Q~ deterministically (each
//      thread owns one column of one accumulator group; fixed row order).
//   B  CTA 0: fixed-order reduction of the CTA partials -> M, sizes; empty
//      clusters are re-seeded with the reference's margin rule (grid-wide
//      first-max argmax per empty cluster), then M is recomputed.
//   C  CTA 0: Y~ = Y/size, one-sided Jacobi SVD of Y~^T Q~ in f64,
//      obj = n - 2 sum(sigma), |d obj| < tol test, R = V U^T.
// No float atomics anywhere: results are bit-reproducible run to run.
#include <cooperative_groups.h>
#include <cstdlib>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace ancka {

constexpr int kDiscThreads = 256;

struct DiscParams {
  const float* Q;
  int64_t ldq, col0, n;
  int k, max_iter;
  double tol;
  int32_t* labels;      // working labels (output of the current run)
  int32_t* labels_run0; // saved labels of run 0
  float* margin;        // n, second-best score
  double* proto_acc;    // n, prototype accumulator
  double* part_m;       // grid x k x k
  int64_t* part_cnt;    // grid x k
  double* part_arg;     // grid x 2  (value, index) for grid argmax/argmin
  double* Rg;           // k x k f64 rotation (row l, col j)
  double* ctrl;         // control block (see below)
  int64_t* counts;      // k
  double* info;         // output info
  int groups;           // accumulator groups per CTA
};

// ctrl layout
enum { C_CONV = 0, C_OBJ_PREV, C_NEMPTY, C_ARGIDX, C_STOP, C_ZERO, C_NCTRL = 8 };

template <int KMAX>
struct Smem {
  // phase A view
  float* R;      // k*k f32 scores rotation
  float* tile;   // kDiscThreads*k
  int* tlab;     // kDiscThreads
  double* acc;   // groups*k*k
  int* cnt;      // k
  double* red;   // 64 scratch
};

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
  for (int l = 0; l < KMAX; ++l) q[l] = nrm > 0 ? q[l] / nrm : 0.0;
  (void)inv;
}

// Phase A.  score=true: compute labels + margins from R; false: use labels.
template <int KMAX>
__device__ void phase_accumulate(const DiscParams& p, float* sR, float* tile, int* tlab,
                                 double* acc, int* cnt, bool score, int* zero_rows) {
  const int k = p.k;
  const int G = p.groups;
  for (int e = threadIdx.x; e < G * k * k; e += blockDim.x) acc[e] = 0.0;
  for (int e = threadIdx.x; e < k; e += blockDim.x) cnt[e] = 0;
  __syncthreads();
  const int64_t rows_per_block = ceil_div(p.n, gridDim.x);
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = lmin(p.n, r0 + rows_per_block);
  int zeros = 0;
  for (int64_t t0 = r0; t0 < r1; t0 += kDiscThreads) {
    const int64_t i = t0 + threadIdx.x;
    if (i < r1) {
      double q[KMAX];
      double nrm;
      load_row<KMAX>(p, i, q, nrm);
      if (nrm == 0.0) ++zeros;
      int lab;
      if (score) {
        float best = -INFINITY, second = -INFINITY;
        lab = 0;
        for (int j = 0; j < k; ++j) {
          float s = 0.f;
#pragma unroll
          for (int l = 0; l < KMAX; ++l)
            if (l < k) s = fmaf((float)q[l], sR[l * k + j], s);
          if (s > best) { second = best; best = s; lab = j; }
          else if (s > second) second = s;
        }
        p.labels[i] = lab;
        p.margin[i] = k >= 2 ? second : best;
      } else {
        lab = p.labels[i];
      }
#pragma unroll
      for (int l = 0; l < KMAX; ++l)
        if (l < k) tile[threadIdx.x * k + l] = (float)q[l];
      tlab[threadIdx.x] = lab;
      atomicAdd(&cnt[lab], 1);  // integer: order independent
    }
    __syncthreads();
    const int tr = (int)lmin(kDiscThreads, r1 - t0);
    const int t = threadIdx.x;
    if (t < G * k) {
      const int j = t % k, g = t / k;
      double* a = acc + (size_t)g * k * k;
      for (int r = g; r < tr; r += G) a[tlab[r] * k + j] += (double)tile[r * k + j];
    }
    __syncthreads();
  }
  // combine groups (fixed order) and publish the CTA partial
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    double s = 0.0;
    for (int g = 0; g < G; ++g) s += acc[(size_t)g * k * k + e];
    p.part_m[(int64_t)blockIdx.x * k * k + e] = s;
  }
  for (int e = threadIdx.x; e < k; e += blockDim.x)
    p.part_cnt[(int64_t)blockIdx.x * k + e] = cnt[e];
  if (zero_rows) {
    __shared__ int zsum;
    if (threadIdx.x == 0) zsum = 0;
    __syncthreads();
    atomicAdd(&zsum, zeros);
    __syncthreads();
    // integer-valued double adds are exact, hence order independent
    if (threadIdx.x == 0 && zsum) atomicAdd(&p.ctrl[C_ZERO], (double)zsum);
  }
  __syncthreads();
}

// CTA 0: reduce M partials -> M (smem f64) and counts (global)
// All threads of CTA 0 take part: entry e is summed by G groups over
// interleaved block subsets, then the G group sums are added in fixed order.
__device__ void reduce_m(const DiscParams& p, double* M) {
  __shared__ double rsum[kDiscThreads];
  __shared__ long long rcnt[kDiscThreads];
  const int k = p.k, kk = k * k, nb = gridDim.x, t = threadIdx.x;
  if (kk >= kDiscThreads) {
    for (int e = t; e < kk; e += blockDim.x) {
      double s0 = 0.0, s1 = 0.0;
      int b = 0;
      for (; b + 1 < nb; b += 2) {
        s0 += p.part_m[(int64_t)b * kk + e];
        s1 += p.part_m[(int64_t)(b + 1) * kk + e];
      }
      if (b < nb) s0 += p.part_m[(int64_t)b * kk + e];
      M[e] = s0 + s1;
    }
  } else {
    const int G = kDiscThreads / kk, g = t / kk, e = t % kk;
    if (g < G) {
      double s = 0.0;
      for (int b = g; b < nb; b += G) s += p.part_m[(int64_t)b * kk + e];
      rsum[g * kk + e] = s;
    }
    __syncthreads();
    if (t < kk) {
      double s = 0.0;
      for (int gg = 0; gg < G; ++gg) s += rsum[gg * kk + t];
      M[t] = s;
    }
  }
  {
    const int G = kDiscThreads / k, g = t / k, e = t % k;
    if (g < G) {
      long long s = 0;
      for (int b = g; b < nb; b += G) s += p.part_cnt[(int64_t)b * k + e];
      rcnt[g * k + e] = s;
    }
    __syncthreads();
    if (t < k) {
      long long s = 0;
      for (int gg = 0; gg < G; ++gg) s += rcnt[gg * k + t];
      p.counts[t] = s;
    }
  }
  __syncthreads();
}

// CTA 0: reduce the per-CTA (value, index) partials in part_arg in parallel.
// want_max: first max (larger value, then smaller index) else first min
// (smaller value, then smaller index); entries with index < 0 are empty.
__device__ void cta_reduce_arg(const double* part, int nb, bool want_max, double& v_out,
                               long long& i_out) {
  __shared__ double sv[kDiscThreads];
  __shared__ long long si[kDiscThreads];
  double v = 0.0;
  long long id = -1;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    const long long i2 = (long long)part[b * 2 + 1];
    const double v2 = part[b * 2];
    const bool take = i2 >= 0 && (id < 0 || (want_max ? v2 > v : v2 < v) || (v2 == v && i2 < id));
    if (take) { v = v2; id = i2; }
  }
  sv[threadIdx.x] = v;
  si[threadIdx.x] = id;
  __syncthreads();
  for (int s = kDiscThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double v2 = sv[threadIdx.x + s];
      const long long i2 = si[threadIdx.x + s];
      const double v1 = sv[threadIdx.x];
      const long long i1 = si[threadIdx.x];
      const bool take = i2 >= 0 && (i1 < 0 || (want_max ? v2 > v1 : v2 < v1) || (v2 == v1 && i2 < i1));
      if (take) { sv[threadIdx.x] = v2; si[threadIdx.x] = i2; }
    }
    __syncthreads();
  }
  v_out = sv[0];
  i_out = si[0];
  __syncthreads();
}

// Grid-wide first-max of margin over movable rows (sizes[label] >= 2).
__device__ void partial_argmax_movable(const DiscParams& p, double* red) {
  const int64_t rows_per_block = ceil_div(p.n, gridDim.x);
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = lmin(p.n, r0 + rows_per_block);
  float best = -INFINITY;
  int64_t bi = -1;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    if (p.counts[p.labels[i]] >= 2) {
      const float m = p.margin[i];
      if (bi < 0 || m > best || (m == best && i < bi)) { best = m; bi = i; }
    }
  }
  // block reduce (value desc, index asc), deterministic
  __shared__ float sv[kDiscThreads];
  __shared__ long long si[kDiscThreads];
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int s = kDiscThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      float v2 = sv[threadIdx.x + s];
      long long i2 = si[threadIdx.x + s];
      float v1 = sv[threadIdx.x];
      long long i1 = si[threadIdx.x];
      bool take = (i2 >= 0) && (i1 < 0 || v2 > v1 || (v2 == v1 && i2 < i1));
      if (take) { sv[threadIdx.x] = v2; si[threadIdx.x] = i2; }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    p.part_arg[blockIdx.x * 2] = sv[0];
    p.part_arg[blockIdx.x * 2 + 1] = (double)si[0];
  }
  (void)red;
}

// one-sided Jacobi SVD of A (k x k, row-major f64, smem) by CTA 0.
// On return A holds U*Sigma (columns), V the right vectors; sigma in sig.
__device__ void jacobi_svd(double* A, double* V, double* sig, int k, int* flag) {
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) V[e] = (e / k == e % k) ? 1.0 : 0.0;
  __syncthreads();
  const int K2 = k + (k & 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int step = 0; step < K2 - 1; ++step) {
      for (int pi = warp; pi < K2 / 2; pi += nwarps) {
        int a, b;
        if (pi == 0) { a = step; b = K2 - 1; }
        else { a = (step + pi) % (K2 - 1); b = (step - pi + K2 - 1) % (K2 - 1); }
        if (a > b) { int t = a; a = b; b = t; }
        if (b >= k) continue;
        double al = 0, be = 0, ga = 0;
        for (int r = lane; r < k; r += 32) {
          double x = A[r * k + a], y = A[r * k + b];
          al += x * x; be += y * y; ga += x * y;
        }
        al = warp_sum(al); be = warp_sum(be); ga = warp_sum(ga);
        if (ga != 0.0 && fabs(ga) > 1e-15 * sqrt(al * be)) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
          for (int r = lane; r < k; r += 32) {
            double x = A[r * k + a], y = A[r * k + b];
            A[r * k + a] = cs * x - sn * y;
            A[r * k + b] = sn * x + cs * y;
            double vx = V[r * k + a], vy = V[r * k + b];
            V[r * k + a] = cs * vx - sn * vy;
            V[r * k + b] = sn * vx + cs * vy;
          }
          if (lane == 0) *flag = 1;
        }
      }
      __syncthreads();
    }
    if (*flag == 0) break;
    __syncthreads();
  }
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    double s = 0;
    for (int r = 0; r < k; ++r) s += A[r * k + j] * A[r * k + j];
    sig[j] = sqrt(s);
  }
  __syncthreads();
}

template <int KMAX>
__global__ void __launch_bounds__(kDiscThreads)
discretize_kernel(DiscParams p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smraw[];
  const int k = p.k;
  const int G = p.groups;
  // phase-A carve
  float* sR = reinterpret_cast<float*>(smraw);
  double* acc = reinterpret_cast<double*>(smraw + align_dev(k * k * 4));
  float* tile = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(acc) + align_dev((size_t)G * k * k * 8));
  int* tlab = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(tile) + align_dev((size_t)kDiscThreads * k * 4));
  int* cnt = tlab + kDiscThreads;
  // phase-B/C carve (CTA 0 only; aliases acc/tile)
  double* M = acc;
  double* Vm = M + k * k;
  double* sig = Vm + k * k;
  __shared__ int s_flag;
  __shared__ double s_red[64];

  const bool cta0 = blockIdx.x == 0;
  for (int run = 0; run < 2; ++run) {
    // ---- initial rotation
    if (run == 0) {
      if (cta0)
        for (int e = threadIdx.x; e < k * k; e += blockDim.x) p.Rg[e] = (e / k == e % k) ? 1.0 : 0.0;
    } else {
      // prototype rotation (engine.py:209-218): R[:,0] = q~[0]; greedy min-acc rows
      if (cta0 && threadIdx.x == 0) {
        double q[KMAX], nrm;
        load_row<KMAX>(p, 0, q, nrm);
        for (int l = 0; l < k; ++l) p.Rg[l * k + 0] = q[l];
      }
      const int64_t rpb = ceil_div(p.n, gridDim.x);
      const int64_t r0 = (int64_t)blockIdx.x * rpb, r1 = lmin(p.n, r0 + rpb);
      for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) p.proto_acc[i] = 0.0;
      grid.sync();
      for (int j = 1; j < k; ++j) {
        double best = INFINITY;
        int64_t bi = -1;
        for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
          double q[KMAX], nrm;
          load_row<KMAX>(p, i, q, nrm);
          double d = 0.0;
#pragma unroll
          for (int l = 0; l < KMAX; ++l)
            if (l < k) d += q[l] * p.Rg[l * k + (j - 1)];
          const double a = p.proto_acc[i] + fabs(d);
          p.proto_acc[i] = a;
          if (bi < 0 || a < best) { best = a; bi = i; }
        }
        // block first-min (value asc, index asc)
        __shared__ double bv[kDiscThreads];
        __shared__ long long bx[kDiscThreads];
        bv[threadIdx.x] = best;
        bx[threadIdx.x] = bi;
        __syncthreads();
        for (int s = kDiscThreads / 2; s > 0; s >>= 1) {
          if (threadIdx.x < s) {
            double v2 = bv[threadIdx.x + s];
            long long i2 = bx[threadIdx.x + s];
            bool take = i2 >= 0 && (bx[threadIdx.x] < 0 || v2 < bv[threadIdx.x] ||
                                    (v2 == bv[threadIdx.x] && i2 < bx[threadIdx.x]));
            if (take) { bv[threadIdx.x] = v2; bx[threadIdx.x] = i2; }
          }
          __syncthreads();
        }
        if (threadIdx.x == 0) {
          p.part_arg[blockIdx.x * 2] = bv[0];
          p.part_arg[blockIdx.x * 2 + 1] = (double)bx[0];
        }
        grid.sync();
        if (cta0) {
          double v;
          long long idx;
          cta_reduce_arg(p.part_arg, gridDim.x, false, v, idx);
          if (threadIdx.x == 0) {
            double q[KMAX], nrm;
            load_row<KMAX>(p, idx < 0 ? 0 : idx, q, nrm);
            for (int l = 0; l < k; ++l) p.Rg[l * k + j] = q[l];
          }
        }
        grid.sync();
      }
    }
    if (cta0 && threadIdx.x == 0) {
      p.ctrl[C_CONV] = 0;
      p.ctrl[C_STOP] = 0;
      if (run == 0) p.ctrl[C_ZERO] = 0;
    }
    grid.sync();

    int rounds = 0;
    for (int it = 0; it < p.max_iter; ++it) {
      for (int e = threadIdx.x; e < k * k; e += blockDim.x) sR[e] = (float)p.Rg[e];
      __syncthreads();
      phase_accumulate<KMAX>(p, sR, tile, tlab, acc, cnt, true,
                             (run == 0 && it == 0) ? &s_flag : nullptr);
      grid.sync();
      if (cta0) {
        reduce_m(p, M);
        if (threadIdx.x == 0) {
          int ne = 0;
          for (int c = 0; c < k; ++c) ne += p.counts[c] == 0;
          p.ctrl[C_NEMPTY] = ne;
        }
      }
      grid.sync();
      const int nempty = (int)p.ctrl[C_NEMPTY];
      if (nempty > 0 && k >= 2) {
        // _reseed_empty_columns (engine.py:162-180)
        for (int c = 0; c < k; ++c) {
          if (p.counts[c] != 0) continue;   // counts is uniform across CTAs here
          partial_argmax_movable(p, s_red);
          grid.sync();
          double vmax = 0.0;
          long long idx = -1;
          if (cta0) cta_reduce_arg(p.part_arg, gridDim.x, true, vmax, idx);
          if (cta0 && threadIdx.x == 0) {
            p.ctrl[C_ARGIDX] = (double)idx;
            if (idx >= 0) {
              const int old = p.labels[idx];
              p.labels[idx] = c;
              p.counts[old] -= 1;
              p.counts[c] += 1;
            }
          }
          grid.sync();
          if (p.ctrl[C_ARGIDX] < 0) break;  // no movable node left
        }
        phase_accumulate<KMAX>(p, sR, tile, tlab, acc, cnt, false, nullptr);
        grid.sync();
        if (cta0) reduce_m(p, M);
      }
      if (cta0) {
        // Y~ = Y / size ; SVD(Y~^T Q~)
        for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
          const int64_t sz = p.counts[e / k];
          M[e] = sz > 0 ? M[e] / (double)sz : 0.0;
        }
        __syncthreads();
        jacobi_svd(M, Vm, sig, k, &s_flag);
        if (threadIdx.x == 0) {
          double ssum = 0;
          for (int j = 0; j < k; ++j) ssum += sig[j];
          const double obj = (double)p.n - 2.0 * ssum;
          p.info[8 + run * p.max_iter + it] = obj;
          const bool conv = it >= 1 && fabs(obj - p.ctrl[C_OBJ_PREV]) < p.tol;
          p.ctrl[C_OBJ_PREV] = obj;
          p.ctrl[C_CONV] = conv ? 1.0 : 0.0;
        }
        __syncthreads();
        // keep R = the rotation that produced the final scores when the run
        // ends without converging (last round)
        if (p.ctrl[C_CONV] == 0.0 && it + 1 < p.max_iter) {
          // R = V U^T with U = A/sigma (columns)
          for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
            const int a = e / k, b = e % k;
            double s = 0;
            for (int j = 0; j < k; ++j)
              if (sig[j] > 0) s += Vm[a * k + j] * (M[b * k + j] / sig[j]);
            p.Rg[e] = s;
          }
        }
      }
      grid.sync();
      rounds = it + 1;
      if (p.ctrl[C_CONV] != 0.0) break;
    }
    // finish the run: publish its final rotation, then its summary
    if (cta0)
      for (int e = threadIdx.x; e < k * k; e += blockDim.x)
        p.info[8 + 2 * p.max_iter + run * k * k + e] = p.Rg[e];
    if (cta0 && threadIdx.x == 0) {
      p.info[6 + run] = rounds;
      const double obj = p.info[8 + run * p.max_iter + rounds - 1];
      if (run == 0) {
        p.info[0] = obj; p.info[1] = rounds; p.info[2] = p.ctrl[C_CONV]; p.info[3] = 0;
        int ne = 0;
        for (int c = 0; c < k; ++c) ne += p.counts[c] == 0;
        p.info[4] = ne;
      } else if (obj < p.info[0] - 1e-15) {
        p.info[0] = obj; p.info[1] = rounds; p.info[2] = p.ctrl[C_CONV]; p.info[3] = 1;
        int ne = 0;
        for (int c = 0; c < k; ++c) ne += p.counts[c] == 0;
        p.info[4] = ne;
      }
      if (run == 0) p.info[5] = p.ctrl[C_ZERO];
    }
    {
      const int64_t rpb = ceil_div(p.n, gridDim.x);
      const int64_t r0 = (int64_t)blockIdx.x * rpb, r1 = lmin(p.n, r0 + rpb);
      if (run == 0)
        for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) p.labels_run0[i] = p.labels[i];
    }
    grid.sync();
  }
  // winner: identity unless the prototype run won
  if (p.info[3] == 0.0) {
    const int64_t rpb = ceil_div(p.n, gridDim.x);
    const int64_t r0 = (int64_t)blockIdx.x * rpb, r1 = lmin(p.n, r0 + rpb);
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) p.labels[i] = p.labels_run0[i];
  }
}

}  // namespace ancka

using namespace ancka;

static int disc_groups(int k) {
  int g = kDiscThreads / k;
  const int cap = (int)((96 * 1024) / ((size_t)k * k * 8));
  if (g > cap) g = cap;
  return g < 1 ? 1 : g;
}

static size_t disc_smem(int k, int G) {
  size_t a = align_dev((size_t)k * k * 4) + align_dev((size_t)G * k * k * 8) +
             align_dev((size_t)kDiscThreads * k * 4) + (kDiscThreads + k) * 4;
  size_t b = align_dev((size_t)k * k * 4) + (2 * (size_t)k * k + k) * 8;
  return std::max(a, b) + 64;
}

static int disc_grid_cap() { return 4 * kNumSMs; }

extern "C" size_t ancka_discretize_workspace_size(int64_t n, int32_t k, int32_t max_iter) {
  (void)max_iter;
  Carver cv(nullptr, 0);
  const int grid = disc_grid_cap();
  cv.take<int32_t>(n);              // labels_run0
  cv.take<float>(n);                // margin
  cv.take<double>(n);               // proto_acc
  cv.take<double>((size_t)grid * k * k);
  cv.take<int64_t>((size_t)grid * k);
  cv.take<double>((size_t)grid * 2);
  cv.take<double>((size_t)k * k);
  cv.take<double>(C_NCTRL);
  cv.take<int64_t>(k);
  return cv.used;
}

template <int KMAX>
static int launch_disc(DiscParams& p, cudaStream_t st) {
  auto kern = discretize_kernel<KMAX>;
  const size_t smem = disc_smem(p.k, p.groups);
  ANCKA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  ANCKA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kDiscThreads, smem));
  ANCKA_REQUIRE(per_sm >= 1, ANCKA_ERR_UNSUPPORTED, "discretize: kernel does not fit an SM");
  int dev = 0, sms = 0;
  ANCKA_CUDA(cudaGetDevice(&dev));
  ANCKA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // rows per CTA: enough work per phase to amortise the grid barrier
  static const int64_t min_rows = getenv("ANCKA_DISC_ROWS") ? atoll(getenv("ANCKA_DISC_ROWS")) : 2048;
  int64_t want = ceil_div(p.n, std::max<int64_t>(kDiscThreads, min_rows));
  int64_t grid = std::min(want, std::min((int64_t)per_sm * sms, (int64_t)disc_grid_cap()));
  if (grid < 1) grid = 1;
  void* args[] = {&p};
  note_launch();
  ANCKA_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3((unsigned)grid), dim3(kDiscThreads),
                                         args, smem, st));
  return ANCKA_OK;
}

extern "C" int ancka_discretize(const float* Q, int64_t ldq, int64_t col0, int64_t n, int32_t k,
                                int32_t max_iter, double tol, int32_t* labels_out, double* info,
                                void* workspace, size_t workspace_bytes, ancka_stream_t stream) {
  ANCKA_REQUIRE(k >= 1 && k <= 64, ANCKA_ERR_UNSUPPORTED, "discretize: k=%d outside [1, 64]", k);
  ANCKA_REQUIRE(n >= 1 && max_iter >= 1, ANCKA_ERR_ARG, "discretize: empty input");
  Carver cv(workspace, workspace_bytes);
  DiscParams p{};
  const int grid = disc_grid_cap();
  p.Q = Q; p.ldq = ldq; p.col0 = col0; p.n = n; p.k = k; p.max_iter = max_iter; p.tol = tol;
  p.labels = labels_out;
  p.labels_run0 = cv.take<int32_t>(n);
  p.margin = cv.take<float>(n);
  p.proto_acc = cv.take<double>(n);
  p.part_m = cv.take<double>((size_t)grid * k * k);
  p.part_cnt = cv.take<int64_t>((size_t)grid * k);
  p.part_arg = cv.take<double>((size_t)grid * 2);
  p.Rg = cv.take<double>((size_t)k * k);
  p.ctrl = cv.take<double>(C_NCTRL);
  p.counts = cv.take<int64_t>(k);
  p.info = info;
  p.groups = disc_groups(k);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "discretize: workspace too small");
  auto st = as_stream(stream);
  ANCKA_CUDA(cudaMemsetAsync(info, 0, sizeof(double) * (8 + 2 * (size_t)max_iter + 2 * (size_t)k * k), st));
  if (k <= 8) return launch_disc<8>(p, st);
  if (k <= 16) return launch_disc<16>(p, st);
  if (k <= 32) return launch_disc<32>(p, st);
  return launch_disc<64>(p, st);
}
