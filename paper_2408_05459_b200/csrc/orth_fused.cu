// Fused orthogonal iterations for narrow blocks (c <= 8): one cooperative
// persistent kernel runs `steps` iterations of orthogonal_step
// (engine.py:130-149) -- the joint-walk SpMM (walk.py:177-190), the Gram
// matrix, the Cholesky factor R, Q = Z R^-1 and ||Q - Q_prev||_F^2 -- with
// four grid barriers per step instead of eight kernel launches.  This is the
// latency-bound regime of the small configurations (Cora, Citeseer, DBLP
// shapes), where every phase touches only a few MB that sit in L2.
//
// One thread owns one row and its 8 (padded) columns: the row's Gram
// contribution is thread-local, so Z never has to be re-read.  Long rows
// (KNN hubs) are processed as fixed-size pieces and combined in a fixed
// order, exactly as the multi-kernel path.  Every CTA reduces the Gram
// partials and factors the 8 x 8 matrix itself (identical arithmetic), so
// no extra barrier is needed to broadcast R^-1.  Deterministic throughout.
#include <cooperative_groups.h>
#include <cstdlib>

#include "common.cuh"
#include "spmm.cuh"

namespace cg = cooperative_groups;

namespace ancka {

constexpr int kOfThreads = 256;
constexpr int kGW = 4;                      // lanes per regular row / hyperedge
constexpr int kC = 8;                       // padded block width
constexpr int kNP = kC * (kC + 1) / 2;      // Gram upper-triangle entries
constexpr double kFx = 1125899906842624.0;  // 2^50 fixed-point scale of Gram sums
// Every partial sum of a Gram entry over a subset of rows is bounded by the
// Gram trace (Cauchy-Schwarz), so a trace below 2^12 keeps all 2^50-scaled
// int64 accumulators (and every CTA's llrint) in range.  Larger traces (hub
// rows inflating ||P q||^2) count as a suspect pivot: the host replays the
// tau-block with the exact f64 step.
constexpr double kGuardFx = 1048576.0;       // 2^20 scale of the trace guard
constexpr double kGuardMaxTrace = 4096.0;
constexpr double kFxInv = 1.0 / 1125899906842624.0;

struct OfParams {
  ancka_operator op;         // f32 operator (by value)
  float* Q[2];               // ping-pong blocks, n x 8
  float* Z;                  // n x 8
  float* T;                  // m x 8 (hypergraph)
  int c, steps;
  long long* gram_fx;        // 2 x kNP fixed-point Gram accumulators
  long long* gram_guard;     // 2 x fixed-point (2^20) Gram trace: overflow guard
  double* dq_part;           // grid
  double* stats;             // [0] dq^2 of the last step, [1] min pivot ratio, [2] += bad pivots
  unsigned long long* tdbg;  // optional phase timers (ANCKA_ORTH_TIMING): stats[4..11]
};

__device__ __forceinline__ unsigned long long of_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define OF_STAMP(s)                                                   \
  do {                                                                \
    if (P.tdbg && blockIdx.x == 0 && threadIdx.x == 0) {              \
      const unsigned long long _n = of_timer();                       \
      if ((s) >= 0) P.tdbg[(s)] += _n - t_prev;                       \
      t_prev = _n;                                                    \
    }                                                                 \
  } while (0)

__device__ __forceinline__ void f8_load(const float* p, float (&v)[kC]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p + 4));
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void f8_store(float* p, const float (&v)[kC]) {
  reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}

// acc += sum_{p in [b, e)} w_p * src[col_p]   (sequential order, 4-way batched loads)
__device__ __forceinline__ void seg8(const int32_t* __restrict__ ci, const float* __restrict__ val,
                                     const float* __restrict__ src, int64_t b, int64_t e,
                                     float (&acc)[kC]) {
  int64_t p = b;
  for (; p + 4 <= e; p += 4) {   // four index loads, then four row loads in flight
    int32_t j[4];
    float w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      j[q] = __ldg(ci + p + q);
      w[q] = val ? __ldg(val + p + q) : 1.f;
    }
    float x[4][kC];
#pragma unroll
    for (int q = 0; q < 4; ++q) f8_load(src + (int64_t)j[q] * kC, x[q]);
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int u = 0; u < kC; ++u) acc[u] = fmaf(w[q], x[q][u], acc[u]);
  }
  for (; p + 2 <= e; p += 2) {
    const int32_t j0 = __ldg(ci + p), j1 = __ldg(ci + p + 1);
    const float w0 = val ? __ldg(val + p) : 1.f, w1 = val ? __ldg(val + p + 1) : 1.f;
    float x0[kC], x1[kC];
    f8_load(src + (int64_t)j0 * kC, x0);
    f8_load(src + (int64_t)j1 * kC, x1);
#pragma unroll
    for (int u = 0; u < kC; ++u) acc[u] = fmaf(w0, x0[u], acc[u]);
#pragma unroll
    for (int u = 0; u < kC; ++u) acc[u] = fmaf(w1, x1[u], acc[u]);
  }
  if (p < e) {
    const int32_t j = __ldg(ci + p);
    const float w = val ? __ldg(val + p) : 1.f;
    float x[kC];
    f8_load(src + (int64_t)j * kC, x);
#pragma unroll
    for (int u = 0; u < kC; ++u) acc[u] = fmaf(w, x[u], acc[u]);
  }
}

// strided partial sum: lanes of a group of `gw` lanes take nonzeros
// b + lane, b + lane + gw, ... (the group's partial sums are reduced after)
__device__ __forceinline__ void seg8_strided(const int32_t* __restrict__ ci,
                                             const float* __restrict__ val,
                                             const float* __restrict__ src, int64_t b, int64_t e,
                                             int lane, int gw, float (&acc)[kC]) {
  int64_t p = b + lane;
  // four nonzeros per round: their index loads, then their row loads, are
  // in flight together (the rows are L2 hits; latency, not bandwidth, binds)
  for (; p + 3 * gw < e; p += 4 * gw) {
    int32_t j[4];
    float w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      j[q] = __ldg(ci + p + q * gw);
      w[q] = val ? __ldg(val + p + q * gw) : 1.f;
    }
    float x[4][kC];
#pragma unroll
    for (int q = 0; q < 4; ++q) f8_load(src + (int64_t)j[q] * kC, x[q]);
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int u = 0; u < kC; ++u) acc[u] = fmaf(w[q], x[q][u], acc[u]);
  }
  for (; p + gw < e; p += 2 * gw) {
    const int32_t j0 = __ldg(ci + p), j1 = __ldg(ci + p + gw);
    const float w0 = val ? __ldg(val + p) : 1.f, w1 = val ? __ldg(val + p + gw) : 1.f;
    float x0[kC], x1[kC];
    f8_load(src + (int64_t)j0 * kC, x0);
    f8_load(src + (int64_t)j1 * kC, x1);
#pragma unroll
    for (int u = 0; u < kC; ++u) acc[u] = fmaf(w0, x0[u], acc[u]);
#pragma unroll
    for (int u = 0; u < kC; ++u) acc[u] = fmaf(w1, x1[u], acc[u]);
  }
  if (p < e) {
    const int32_t j = __ldg(ci + p);
    const float w = val ? __ldg(val + p) : 1.f;
    float x[kC];
    f8_load(src + (int64_t)j * kC, x);
#pragma unroll
    for (int u = 0; u < kC; ++u) acc[u] = fmaf(w, x[u], acc[u]);
  }
}

// butterfly sum over groups of `gw` lanes (gw a power of two <= 32)
__device__ __forceinline__ void group_sum(float (&v)[kC], int gw) {
  for (int o = gw >> 1; o > 0; o >>= 1)
#pragma unroll
    for (int u = 0; u < kC; ++u) v[u] += __shfl_xor_sync(0xffffffffu, v[u], o);
}

__device__ __forceinline__ void gram_add(const float (&z)[kC], double (&g)[kNP]) {
  int q = 0;
#pragma unroll
  for (int a = 0; a < kC; ++a)
#pragma unroll
    for (int b = a; b < kC; ++b) g[q++] += (double)(z[a] * z[b]);
}

// z = mix(s, k) for row i, store, add to the Gram partial
__device__ __forceinline__ void finish8(const OfParams& P, int64_t i, const float* Qp,
                                        float (&s)[kC], float (&kk)[kC], float (&z)[kC]) {
  const ancka_operator& op = P.op;
  if (op.selfloop[i]) {
    float x[kC];
    f8_load(Qp + i * kC, x);
#pragma unroll
    for (int u = 0; u < kC; ++u) s[u] += x[u];
  }
  const float b = __ldg(static_cast<const float*>(op.beta) + i);
  const float omb = 1.f - b;
#pragma unroll
  for (int u = 0; u < kC; ++u) z[u] = u < P.c ? omb * s[u] + b * kk[u] : 0.f;
  f8_store(P.Z + i * kC, z);
}

// this row's 36 Gram products (f32) into shared-memory slot `slot`
__device__ __forceinline__ void gram_stage(float* gsm, int slot, const float (&z)[kC]) {
  int qq = 0;
#pragma unroll
  for (int a = 0; a < kC; ++a)
#pragma unroll
    for (int b2 = a; b2 < kC; ++b2, ++qq) gsm[slot * (kNP + 1) + qq] = z[a] * z[b2];
}

// deterministic CTA reduction of the per-thread Gram partial -> global slot
__device__ void block_gram(double (&g)[kNP], double* out, double* red /* 32*kNP */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < kNP; ++q) {
    double v = g[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp * kNP + q] = v;
  }
  __syncthreads();
  const int nw = blockDim.x >> 5;
  for (int q = threadIdx.x; q < kNP; q += blockDim.x) {
    double v = 0.0;
    for (int w = 0; w < nw; ++w) v += red[w * kNP + q];
    out[q] = v;
  }
  __syncthreads();
}

__device__ __forceinline__ int pidx(int a, int b) {  // a <= b, packed upper of 8 x 8
  return a * kC - (a * (a - 1)) / 2 + (b - a);
}

#ifndef ANCKA_ORTH_CTAS
#define ANCKA_ORTH_CTAS 2
#endif
__global__ void __launch_bounds__(kOfThreads, ANCKA_ORTH_CTAS)
orth_fused_kernel(OfParams P) {
  cg::grid_group grid = cg::this_grid();
  const ancka_operator& op = P.op;
  const bool hyper = op.kind == ANCKA_HYPERGRAPH;
  // scalar selects (a runtime-selected reference into parameter space would
  // force a local copy of the whole parameter block)
  const int64_t* S_rp = hyper ? op.p_v.rowptr : op.p_n.rowptr;
  const int32_t* S_ci = hyper ? op.p_v.colidx : op.p_n.colidx;
  const float* Sval = static_cast<const float*>(hyper ? op.p_v.values : op.p_n.values);
  const int64_t* K_rp = op.p_k.rowptr;
  const int32_t* K_ci = op.p_k.colidx;
  const float* Kval = static_cast<const float*>(op.p_k.values);
  const ancka_row_split& sp = op.split;
  const int64_t n = op.n;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gsz = (int64_t)gridDim.x * blockDim.x;
  const int nb = gridDim.x;

  __shared__ double red[(kOfThreads / 32) * kNP];
  __shared__ float gsm[kOfThreads * (kNP + 1)];
  __shared__ double G[kNP];
  __shared__ float Rinv[kC * kC];
  __shared__ double s_stat[2];

  unsigned long long t_prev = 0;
  const int lane0 = threadIdx.x & 31;
  const int sub0 = lane0 & (kGW - 1);
  const int64_t goct0 = gtid / kGW, noct0 = gsz / kGW;
  if (hyper) {     // T = P_E Q0 for the first step
    const float* Eval = static_cast<const float*>(op.p_e.values);
    const int64_t m = op.m;
    for (int64_t e = goct0; e < ((m + noct0 - 1) / noct0) * noct0; e += noct0) {
      float acc[kC] = {};
      if (e < m) seg8_strided(op.p_e.colidx, Eval, P.Q[0], op.p_e.rowptr[e], op.p_e.rowptr[e + 1],
                              sub0, kGW, acc);
      group_sum(acc, kGW);
      if (e < m && sub0 == 0) f8_store(P.T + e * kC, acc);
    }
    grid.sync();
  }
  for (int step = 0; step < P.steps; ++step) {
    OF_STAMP(-1);
    const float* Qp = P.Q[step & 1];
    float* Qn = P.Q[(step + 1) & 1];
    const int buf = step & 1;
    // row groups: 8 lanes per regular row, a whole warp per long row
    const int lane = threadIdx.x & 31;
    const int sub = lane & (kGW - 1);
    // lane groups / warps numbered CTA-fastest, so consecutive rows of the
    // cost order (and consecutive long rows) land on different CTAs: every
    // CTA gets an equal share of the heavy rows and the barrier after P2
    // waits less for the slowest CTA
    const int64_t gwarp = (int64_t)(threadIdx.x >> 5) * gridDim.x + blockIdx.x, nwarps = gsz >> 5;
    const int64_t goct = (int64_t)(threadIdx.x / kGW) * gridDim.x + blockIdx.x, noct = gsz / kGW;
    // T = P_E Q of this step was produced at the end of the previous step
    // (or before the loop), already multiplied by R^-1
    const float* Ssrc = hyper ? P.T : Qp;
    unsigned long long p2_t0 = 0;
    if (P.tdbg && threadIdx.x == 0) p2_t0 = of_timer();
    // ---- P2: rows of Z with their Gram contributions: regular rows by
    // kGW-lane groups (cost-ordered), long rows (KNN hubs) by whole warps.
    // Each produced row's 36 products are staged in shared memory (one slot
    // per lane group) and summed into per-thread f64 partials after every
    // round, so the Gram needs no second pass over Z and no extra barrier.
    constexpr int kGS = 7;                         // summing threads per entry
    const int gq = threadIdx.x % kNP, gg = threadIdx.x / kNP;
    constexpr int kSlots = kOfThreads / kGW;       // regular-row slots per round
    double gacc = 0.0;
    auto gram_round = [&](int nslots) {
      __syncthreads();
      if (gg < kGS)
        for (int r = gg; r < nslots; r += kGS) gacc += (double)gsm[r * (kNP + 1) + gq];
      __syncthreads();
    };
    const int64_t nround = ((n + noct - 1) / noct) * noct;
    for (int64_t i0 = goct; i0 < nround; i0 += noct) {
      const int64_t i = (sp.row_order && i0 < n) ? (int64_t)sp.row_order[i0] : i0;
      const bool live = i0 < n && !(sp.is_long && sp.is_long[i]);
      float s[kC] = {}, kk[kC] = {}, z[kC] = {};
      if (live) {
        seg8_strided(S_ci, Sval, Ssrc, S_rp[i], S_rp[i + 1], sub, kGW, s);
        seg8_strided(K_ci, Kval, Qp, K_rp[i], K_rp[i + 1], sub, kGW, kk);
      }
      group_sum(s, kGW);
      group_sum(kk, kGW);
      if (live && sub == 0) finish8(P, i, Qp, s, kk, z);
      if (sub == 0) gram_stage(gsm, threadIdx.x / kGW, z);   // zeros when not live
      gram_round(kSlots);
    }
    const int64_t lround = ((sp.n_long + nwarps - 1) / nwarps) * nwarps;
    for (int64_t li = gwarp; li < lround; li += nwarps) {
      const bool live = li < sp.n_long;
      const int64_t i = live ? sp.long_rows[li] : 0;
      float s[kC] = {}, kk[kC] = {}, z[kC] = {};
      if (live) {
        seg8_strided(S_ci, Sval, Ssrc, S_rp[i], S_rp[i + 1], lane, 32, s);
        seg8_strided(K_ci, Kval, Qp, K_rp[i], K_rp[i + 1], lane, 32, kk);
      }
      group_sum(s, 32);
      group_sum(kk, 32);
      if (live && lane == 0) finish8(P, i, Qp, s, kk, z);
      if (lane == 0) gram_stage(gsm, threadIdx.x >> 5, z);
      gram_round(kOfThreads / 32);
    }
    // CTA total of the Gram partials -> one fixed-point atomic per entry
    // (integer sums are order independent: bit-reproducible)
    if (gg < kGS) red[gg * kNP + gq] = gacc;
    __syncthreads();
    for (int qq = threadIdx.x; qq < kNP; qq += blockDim.x) {
      double v = 0.0;
      for (int g2 = 0; g2 < kGS; ++g2) v += red[g2 * kNP + qq];
      atomicAdd(reinterpret_cast<unsigned long long*>(P.gram_fx + buf * kNP + qq),
                (unsigned long long)(long long)llrint(fmin(fmax(v, -kGuardMaxTrace), kGuardMaxTrace) * kFx));
      bool diag = false;
#pragma unroll
      for (int a2 = 0; a2 < kC; ++a2) diag |= (a2 < P.c && qq == pidx(a2, a2));
      if (diag)                                  // v >= 0: a sum of squares
        atomicAdd(reinterpret_cast<unsigned long long*>(P.gram_guard + buf),
                  (unsigned long long)(long long)llrint(fmin(v, 1e12) * kGuardFx));
    }
    OF_STAMP(2);
    if (P.tdbg) {                        // per-CTA P2 duration: max and sum over CTAs
      __syncthreads();
      if (threadIdx.x == 0) {
        const unsigned long long dt = of_timer() - p2_t0;
        atomicMax(P.tdbg + 9, dt);
        atomicAdd(P.tdbg + 10, dt);
        atomicMax(P.tdbg + 11, (dt << 20) | (unsigned long long)blockIdx.x);
      }
    }
    grid.sync();                        // Z and the Gram complete
    OF_STAMP(4);
    // ---- P4: every CTA: Gram (fixed-point sums), Cholesky, R^-1 (identical)
    if (threadIdx.x < kNP) G[threadIdx.x] = (double)P.gram_fx[buf * kNP + threadIdx.x] * kFxInv;
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x < kNP) P.gram_fx[(buf ^ 1) * kNP + threadIdx.x] = 0;
    const double gtrace = (double)P.gram_guard[buf] * (1.0 / kGuardFx);
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) P.gram_guard[buf ^ 1] = 0;
    if (threadIdx.x == 0) {
      // Cholesky of the padded 8 x 8 Gram (identity on padding), fully
      // unrolled so the factor lives in registers
      double R[kC][kC], X[kC][kC], Rd[kC];
#pragma unroll
      for (int a2 = 0; a2 < kC; ++a2)
#pragma unroll
        for (int b3 = 0; b3 < kC; ++b3)
          R[a2][b3] = (a2 < P.c && b3 < P.c) ? (a2 <= b3 ? G[pidx(a2, b3)] : 0.0)
                                             : (a2 == b3 ? 1.0 : 0.0);
      double minratio = 1.0;
      int bad = gtrace >= kGuardMaxTrace / 2 ? 1 : 0;   // fixed-point range guard
#pragma unroll
      for (int j = 0; j < kC; ++j) {
        const double gjj = R[j][j];
        double piv = gjj;
#pragma unroll
        for (int l = 0; l < j; ++l) piv -= R[l][j] * R[l][j];
        const double ratio = gjj > 0 ? piv / gjj : 0.0;
        if (j < P.c) {
          minratio = fmin(minratio, ratio);
          if (!(ratio > 1e-9)) { ++bad; piv = fmax(piv, 1e-30 + 1e-9 * fmax(gjj, 0.0)); }
        }
        const double rjj = sqrt(piv);
        const double irjj = 1.0 / rjj;          // one division per column
        R[j][j] = rjj;
        Rd[j] = irjj;
#pragma unroll
        for (int q = j + 1; q < kC; ++q) {
          double v = R[j][q];
#pragma unroll
          for (int l = 0; l < j; ++l) v -= R[l][j] * R[l][q];
          R[j][q] = v * irjj;
        }
      }
#pragma unroll
      for (int bcol = 0; bcol < kC; ++bcol) {
#pragma unroll
        for (int a2 = 0; a2 < kC; ++a2) X[a2][bcol] = 0.0;
        X[bcol][bcol] = Rd[bcol];
#pragma unroll
        for (int a2 = bcol - 1; a2 >= 0; --a2) {
          double v = 0.0;
#pragma unroll
          for (int l = a2 + 1; l <= bcol; ++l) v += R[a2][l] * X[l][bcol];
          X[a2][bcol] = -v * Rd[a2];
        }
      }
#pragma unroll
      for (int a2 = 0; a2 < kC; ++a2)
#pragma unroll
        for (int b3 = 0; b3 < kC; ++b3)
          Rinv[a2 * kC + b3] = (a2 <= b3 && b3 < P.c) ? (float)X[a2][b3] : 0.f;
      s_stat[0] = minratio;
      s_stat[1] = bad;
    }
    __syncthreads();
    OF_STAMP(5);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      P.stats[1] = fmin(P.stats[1], s_stat[0]);
      P.stats[2] += s_stat[1];
    }
    // ---- next step's T = P_E Q_{t+1} = (P_E Z) R^-1: Z is complete (barrier
    // above) and R^-1 is known, so the hyperedge stage needs no barrier of
    // its own; every group applies R^-1 to the hyperedges it produced
    if (hyper) {
      const float* Eval = static_cast<const float*>(op.p_e.values);
      const int64_t m = op.m;
      for (int64_t e = goct; e < ((m + noct - 1) / noct) * noct; e += noct) {
        float acc[kC] = {};
        if (e < m) seg8_strided(op.p_e.colidx, Eval, P.Z, op.p_e.rowptr[e], op.p_e.rowptr[e + 1],
                                sub, kGW, acc);
        group_sum(acc, kGW);
        if (e < m && sub == 0) {
          float tv[kC];
#pragma unroll
          for (int b2 = 0; b2 < kC; ++b2) {
            float v = 0.f;
#pragma unroll
            for (int a = 0; a <= b2; ++a) v = fmaf(acc[a], Rinv[a * kC + b2], v);
            tv[b2] = v;
          }
          f8_store(P.T + e * kC, tv);
        }
      }
    }
    // ---- P5: Q = Z R^-1 and ||Q - Q_prev||^2
    double dq = 0.0;
    for (int64_t i = gtid; i < n; i += gsz) {
      float z[kC], qo[kC], qv[kC];
      f8_load(P.Z + i * kC, z);
      f8_load(Qp + i * kC, qo);
#pragma unroll
      for (int b2 = 0; b2 < kC; ++b2) {
        float v = 0.f;
#pragma unroll
        for (int a = 0; a <= b2; ++a) v = fmaf(z[a], Rinv[a * kC + b2], v);
        qv[b2] = v;
        const double d = (double)v - (double)qo[b2];
        dq += d * d;
      }
      f8_store(Qn + i * kC, qv);
    }
    dq = block_sum(dq, red);
    if (threadIdx.x == 0) P.dq_part[blockIdx.x] = dq;
    OF_STAMP(6);
    grid.sync();
    OF_STAMP(7);
  }
  if (blockIdx.x == 0) {
    double s = 0.0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) s += P.dq_part[b];
    s = block_sum(s, red);
    if (threadIdx.x == 0) P.stats[0] = s;
  }
}


// ---------------------------------------------------------------------------
// Fused multi-hop conductance (engine.py:291-299) for k <= 8: one cooperative
// kernel replaces the cluster-size histogram, the tag fill, gamma x (P_E pass
// + row pass) SpMM launches and the two trace kernels.  Rows are walked in the
// same cost order and lane layout as the orthogonal block above.
//   F0 = alpha Yhat;  F <- (1 - alpha) apply(F) + F0  (gamma times);
//   phi = 1 - <Yhat, F> / k   (NaN when a cluster is empty)
struct MhcParams {
  ancka_operator op;
  const int32_t* labels;
  int k, gamma;
  double alpha;
  float scale;                 // 1 - alpha
  float* F[2];                 // n x 8 ping-pong
  float* T;                    // m x 8 (hypergraph)
  unsigned long long* hist;    // k, zeroed by the host
  int64_t* sizes;              // k (output)
  double* part;                // grid trace partials
  double* phi;
  unsigned long long* tdbg;    // optional (ANCKA_MHC_TIMING): per phase CTA-0 work, max CTA work
};

#ifndef ANCKA_MHC_CTAS
#define ANCKA_MHC_CTAS 3
#endif
__global__ void __launch_bounds__(kOfThreads, ANCKA_MHC_CTAS)
mhc_fused_kernel(MhcParams P) {
  cg::grid_group grid = cg::this_grid();
  const ancka_operator& op = P.op;
  const bool hyper = op.kind == ANCKA_HYPERGRAPH;
  const int64_t* S_rp = hyper ? op.p_v.rowptr : op.p_n.rowptr;
  const int32_t* S_ci = hyper ? op.p_v.colidx : op.p_n.colidx;
  const float* Sval = static_cast<const float*>(hyper ? op.p_v.values : op.p_n.values);
  const int64_t* K_rp = op.p_k.rowptr;
  const int32_t* K_ci = op.p_k.colidx;
  const float* Kval = static_cast<const float*>(op.p_k.values);
  const ancka_row_split& sp = op.split;
  const int64_t n = op.n;
  const int k = P.k;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gsz = (int64_t)gridDim.x * blockDim.x;
  __shared__ unsigned int h[kC];
  __shared__ float tv[kC];
  __shared__ double yh[kC];
  __shared__ double red[32];
  __shared__ int s_empty;
  int ph = 0;
  unsigned long long t_ph = of_timer();
  // phase work time before a grid barrier: CTA 0's and the max over CTAs
  auto stamp = [&]() {
    if (P.tdbg) {
      __syncthreads();
      if (threadIdx.x == 0) {
        const unsigned long long now = of_timer(), dt = now - t_ph;
        if (blockIdx.x == 0) P.tdbg[2 * ph] += dt;
        atomicMax(P.tdbg + 2 * ph + 1, dt);
        if (ph < 8) P.tdbg[64 + ph * 1024 + blockIdx.x] = dt;   // last call, per CTA
      }
    }
  };
  auto after = [&]() { ++ph; if (P.tdbg && threadIdx.x == 0) t_ph = of_timer(); };

  // ---- cluster sizes (integer atomics: order-free)
  if (threadIdx.x < kC) h[threadIdx.x] = 0u;
  __syncthreads();
  for (int64_t i = gtid; i < n; i += gsz) {
    const int l = P.labels[i];
    if (l >= 0 && l < k) atomicAdd(&h[l], 1u);
  }
  __syncthreads();
  if (threadIdx.x < k && h[threadIdx.x]) atomicAdd(P.hist + threadIdx.x, (unsigned long long)h[threadIdx.x]);
  stamp();
  grid.sync();
  after();
  if (threadIdx.x == 0) s_empty = 0;
  __syncthreads();
  if (threadIdx.x < kC) {
    const int c = threadIdx.x;
    const unsigned long long sz = c < k ? __ldcg(P.hist + c) : 0ull;
    const double y = sz > 0 ? 1.0 / sqrt((double)sz) : 0.0;   // mhc_tagval_kernel
    yh[c] = y;
    tv[c] = c < k ? (float)(P.alpha * y) : 0.f;
    if (c < k && sz == 0) s_empty = 1;
    if (blockIdx.x == 0 && c < k) P.sizes[c] = (int64_t)sz;
  }
  __syncthreads();
  // ---- F0 = alpha Yhat (fill_tag_kernel)
  for (int64_t i = gtid; i < n; i += gsz) {
    const int l = P.labels[i];
    float f[kC];
#pragma unroll
    for (int u = 0; u < kC; ++u) f[u] = (u == l && u < k) ? tv[u] : 0.f;
    f8_store(P.F[0] + i * kC, f);
  }
  stamp();
  grid.sync();
  after();

  const int lane = threadIdx.x & 31;
  const int sub = lane & (kGW - 1);
  const int64_t gwarp = (int64_t)(threadIdx.x >> 5) * gridDim.x + blockIdx.x, nwarps = gsz >> 5;
  const int64_t goct = (int64_t)(threadIdx.x / kGW) * gridDim.x + blockIdx.x, noct = gsz / kGW;
  double tr = 0.0;
  for (int g = 0; g < P.gamma; ++g) {
    const float* src = P.F[g & 1];
    float* dst = P.F[(g + 1) & 1];
    const bool last = g + 1 == P.gamma;
    if (hyper) {   // T = P_E F
      const float* Eval = static_cast<const float*>(op.p_e.values);
      const int64_t m = op.m;
      for (int64_t e = goct; e < ((m + noct - 1) / noct) * noct; e += noct) {
        float acc[kC] = {};
        if (e < m) seg8_strided(op.p_e.colidx, Eval, src, op.p_e.rowptr[e], op.p_e.rowptr[e + 1],
                                sub, kGW, acc);
        group_sum(acc, kGW);
        if (e < m && sub == 0) f8_store(P.T + e * kC, acc);
      }
      stamp();
  grid.sync();
  after();
    }
    const float* Ssrc = hyper ? P.T : src;
    // out = (1 - alpha) ((1 - b) (S + self) + b K) + tag   (finish_row with the tag epilogue)
    auto finish = [&](int64_t i, float (&s)[kC], float (&kk)[kC]) {
      if (op.selfloop[i]) {
        float x[kC];
        f8_load(src + i * kC, x);
#pragma unroll
        for (int u = 0; u < kC; ++u) s[u] += x[u];
      }
      const float b = __ldg(static_cast<const float*>(op.beta) + i);
      const float omb = 1.f - b;
      const int l = __ldg(P.labels + i);
      float z[kC];
#pragma unroll
      for (int u = 0; u < kC; ++u) {
        const float v = P.scale * (omb * s[u] + b * kk[u]);
        z[u] = u < k ? v + ((u == l) ? tv[u] : 0.f) : 0.f;
      }
      f8_store(dst + i * kC, z);
      if (last) {
#pragma unroll
        for (int u = 0; u < kC; ++u)
          if (u == l) tr += yh[u] * (double)z[u];
      }
    };
    const int64_t nround = ((n + noct - 1) / noct) * noct;
    for (int64_t i0 = goct; i0 < nround; i0 += noct) {
      const int64_t i = (sp.row_order && i0 < n) ? (int64_t)sp.row_order[i0] : i0;
      const bool live = i0 < n && !(sp.is_long && sp.is_long[i]);
      float s[kC] = {}, kk[kC] = {};
      if (live) {
        seg8_strided(S_ci, Sval, Ssrc, S_rp[i], S_rp[i + 1], sub, kGW, s);
        seg8_strided(K_ci, Kval, src, K_rp[i], K_rp[i + 1], sub, kGW, kk);
        if (P.tdbg && sub == 0)
          atomicAdd(P.tdbg + 64 + 8 * 1024 + blockIdx.x,
                    (unsigned long long)(S_rp[i + 1] - S_rp[i] + K_rp[i + 1] - K_rp[i]));
      }
      group_sum(s, kGW);
      group_sum(kk, kGW);
      if (live && sub == 0) finish(i, s, kk);
    }
    const int64_t lround = ((sp.n_long + nwarps - 1) / nwarps) * nwarps;
    for (int64_t li = gwarp; li < lround; li += nwarps) {
      const bool live = li < sp.n_long;
      const int64_t i = live ? sp.long_rows[li] : 0;
      float s[kC] = {}, kk[kC] = {};
      if (live) {
        seg8_strided(S_ci, Sval, Ssrc, S_rp[i], S_rp[i + 1], lane, 32, s);
        seg8_strided(K_ci, Kval, src, K_rp[i], K_rp[i + 1], lane, 32, kk);
      }
      group_sum(s, 32);
      group_sum(kk, 32);
      if (live && lane == 0) finish(i, s, kk);
    }
    if (last) {
      tr = block_sum(tr, red);
      if (threadIdx.x == 0) P.part[blockIdx.x] = tr;
    }
    stamp();
  grid.sync();
  after();
  }
  if (blockIdx.x == 0) {   // fixed-order sum of the CTA partials (mhc_finish_kernel)
    double s = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) s += P.part[b];
    s = block_sum(s, red);
    if (threadIdx.x == 0) *P.phi = s_empty ? nan("") : 1.0 - s / (double)k;
  }
}

constexpr int kMhcTimingWords = 64 + 9 * 1024;
static unsigned long long* mhc_timing_buffer() {
  static unsigned long long* buf = nullptr;
  if (!buf) {
    cudaMalloc(&buf, kMhcTimingWords * sizeof(unsigned long long));
    cudaMemset(buf, 0, kMhcTimingWords * sizeof(unsigned long long));
  }
  return buf;
}

extern "C" void ancka_mhc_timing(unsigned long long* out, int reset) {
  unsigned long long* b = mhc_timing_buffer();
  cudaDeviceSynchronize();
  if (out) cudaMemcpy(out, b, kMhcTimingWords * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  if (reset) cudaMemset(b, 0, kMhcTimingWords * sizeof(unsigned long long));
  cudaDeviceSynchronize();
}

int mhc_fused_f32(const ancka_operator* op, const int32_t* labels, int k, double alpha, int gamma,
                  double* phi, int64_t* sizes, float* F0, float* F1, float* T,
                  unsigned long long* hist, double* part, cudaStream_t st) {
  ANCKA_REQUIRE(k >= 1 && k <= kC && gamma >= 1, ANCKA_ERR_UNSUPPORTED, "fused mhc: k <= 8");
  MhcParams P{};
  P.op = *op;
  P.labels = labels;
  P.k = k;
  P.gamma = gamma;
  P.alpha = alpha;
  P.scale = (float)(1.0 - alpha);
  P.F[0] = F0;
  P.F[1] = F1;
  P.T = T;
  P.hist = hist;
  P.sizes = sizes;
  P.part = part;
  P.phi = phi;
  P.tdbg = getenv("ANCKA_MHC_TIMING") ? mhc_timing_buffer() : nullptr;
  ANCKA_CUDA(cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * k, st));
  int per_sm = 0, dev = 0, sms = 0;
  ANCKA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mhc_fused_kernel, kOfThreads, 0));
  ANCKA_CUDA(cudaGetDevice(&dev));
  ANCKA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  ANCKA_REQUIRE(per_sm >= 1, ANCKA_ERR_UNSUPPORTED, "fused mhc does not fit an SM");
  const int64_t want = ceil_div(op->n, 32);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(
      want, std::min<int64_t>((int64_t)std::min(per_sm, ANCKA_MHC_CTAS) * sms, mhc_fused_grid_cap())));
  void* args[] = {&P};
  note_launch();
  ANCKA_CUDA(cudaLaunchCooperativeKernel((void*)mhc_fused_kernel, dim3(grid), dim3(kOfThreads),
                                         args, 0, st));
  return ANCKA_OK;
}

}  // namespace ancka

using namespace ancka;

static int of_grid_cap() { return 8 * kNumSMs; }

extern "C" size_t ancka_orth_block_workspace_size(const ancka_operator* op) {
  Carver cv(nullptr, 0);
  cv.take<float>(op && op->kind == ANCKA_HYPERGRAPH ? (size_t)op->m * kC : 1);
  cv.take<long long>(2 * kNP);
  cv.take<long long>(2);
  cv.take<double>(of_grid_cap());
  return cv.used;
}

extern "C" int ancka_orth_block_f32(const ancka_operator* op32, float* Q0, float* Q1, float* Z,
                                    int64_t ld, int32_t c, int32_t steps, double* stats,
                                    void* workspace, size_t workspace_bytes, ancka_stream_t stream) {
  ANCKA_REQUIRE(op32 && op32->dtype == ANCKA_F32, ANCKA_ERR_ARG, "orth_block needs the f32 operator");
  ANCKA_REQUIRE(op32->kind != ANCKA_MULTIPLEX, ANCKA_ERR_UNSUPPORTED,
                "fused orthogonal block: graph and hypergraph operators only");
  ANCKA_REQUIRE(ld == kC && c >= 1 && c <= kC, ANCKA_ERR_UNSUPPORTED,
                "fused orthogonal block supports c <= 8 with ld == 8");
  Carver cv(workspace, workspace_bytes);
  OfParams P{};
  P.op = *op32;
  P.Q[0] = Q0;
  P.Q[1] = Q1;
  P.Z = Z;
  P.T = cv.take<float>(op32->kind == ANCKA_HYPERGRAPH ? (size_t)op32->m * kC : 1);
  P.c = c;
  P.steps = steps;
  P.gram_fx = cv.take<long long>(2 * kNP);
  P.gram_guard = cv.take<long long>(2);
  P.dq_part = cv.take<double>(of_grid_cap());
  P.stats = stats;
  P.tdbg = getenv("ANCKA_ORTH_TIMING") ? reinterpret_cast<unsigned long long*>(stats + 4) : nullptr;
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "orth_block: workspace too small");
  ANCKA_CUDA(cudaMemsetAsync(P.gram_fx, 0, sizeof(long long) * 2 * kNP, as_stream(stream)));
  ANCKA_CUDA(cudaMemsetAsync(P.gram_guard, 0, sizeof(long long) * 2, as_stream(stream)));
  int per_sm = 0, dev = 0, sms = 0;
  ANCKA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, orth_fused_kernel, kOfThreads, 0));
  ANCKA_CUDA(cudaGetDevice(&dev));
  ANCKA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  ANCKA_REQUIRE(per_sm >= 1, ANCKA_ERR_UNSUPPORTED, "orth_block does not fit an SM");
  int64_t want = ceil_div(op32->n, 32);
  if (const char* g = getenv("ANCKA_ORTH_GRID")) want = std::max(1, atoi(g));
  // two CTAs per SM: more CTAs shorten each CTA's row share but lengthen the
  // grid barriers and the tail (measured at the DBLP shape: 2/SM 861 us per
  // 20 steps, 4/SM 975 us)
  const int64_t cap = getenv("ANCKA_ORTH_GRID") ? of_grid_cap() : ANCKA_ORTH_CTAS * (int64_t)sms;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(
      want, std::min<int64_t>((int64_t)per_sm * sms, std::min<int64_t>(cap, of_grid_cap()))));
  void* args[] = {&P};
  note_launch();
  ANCKA_CUDA(cudaLaunchCooperativeKernel((void*)orth_fused_kernel, dim3(grid), dim3(kOfThreads),
                                         args, 0, as_stream(stream)));
  return ANCKA_OK;
}
