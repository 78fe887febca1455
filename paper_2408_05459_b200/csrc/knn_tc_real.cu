// Exact cosine KNN for real-valued attributes on the tensor cores, with a
// certificate: knn.py:112-140 (blocked exact scan, strictly positive sims,
// order (value desc, index asc), scores min(s, 1)).
//
// 1. prep      xn = X * (1/||X||) in f64 exactly as _normalize_rows
//              (knn.py:62-65; the norm is numpy's pairwise sum), and its
//              split into bf16 hi = rn(xn), lo = rn(xn - hi), stored [hi | lo].
// 2. contract  a_ij = <hi_i,hi_j> + <hi_i,lo_j> + <lo_i,hi_j> by tcgen05 as one
//              K = 3 d_pad contraction of [hi|hi|lo] x [hi|lo|hi] (the column
//              map reads both operands out of the one stored [hi|lo] matrix).
//              |a_ij - s_ij| <= eps with eps = 2^-16 (split) + 3 d_pad 2^-23
//              (f32 accumulation), a bound on the unit-vector dot error.
// 3. filter    each query row keeps its top-L approximate candidates (L > K)
//              in registers, admitting only a >= max(a_(K) - 2 eps, -eps);
//              every true top-K member passes: s_(K) >= a_(K) - eps and
//              s_j >= s_(K) imply a_j >= a_(K) - 2 eps, and s_j > 0 implies
//              a_j > -eps.
// 4. rerank    the merged candidates above the threshold get their exact f64
//              dot <xn_i, xn_j>; the top K by (s desc, j asc) with s > 0 are
//              emitted.  The row is certified when no candidate that was
//              dropped for lack of slots could reach the threshold; rows that
//              are not certified (dense ties, duplicates) are recomputed by
//              the f64 CUDA-core scan (knn_simt.cu) over all keys.
// The n x n similarity matrix never leaves TMEM/registers.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdlib>

#include "common.cuh"
#include "knn.cuh"
#include "knn_tc.cuh"
#include "sm100.cuh"

namespace ancka {
using namespace sm100;

namespace {
constexpr float kInf = __builtin_huge_valf();

// Register-resident top-(K+E) of approximate cosines, order (a desc, j asc).
// As in the integer kernel the list has L fixed slots: the first L-E-K hold
// +inf padding (never displaced), the K+E live entries follow, so the K-th
// live entry is always slot L-E-1 and the last live one slot L-1 -- no slot
// is addressed by a runtime index and the arrays stay in registers.
// max of 32 accumulator words (f32 bits) by three-input FMNMX3: 17
// instructions in a 3-level tree instead of 31 two-input FMNMX
__device__ __forceinline__ float fmax3_(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float max32_f32(const uint32_t (&r)[32]) {
  float a[11];
#pragma unroll
  for (int k = 0; k < 10; ++k)
    a[k] = fmax3_(__uint_as_float(r[3 * k]), __uint_as_float(r[3 * k + 1]), __uint_as_float(r[3 * k + 2]));
  a[10] = fmaxf(__uint_as_float(r[30]), __uint_as_float(r[31]));
  const float b0 = fmax3_(a[0], a[1], a[2]), b1 = fmax3_(a[3], a[4], a[5]);
  const float b2 = fmax3_(a[6], a[7], a[8]), b3 = fmaxf(a[9], a[10]);
  return fmaxf(fmax3_(b0, b1, b2), b3);
}

template <int L, int E>
struct CandList {
  static constexpr int KSLOT = L - E - 1;
  float f[L];
  int32_t j[L];
  float thr;     // admission threshold
  float floor_;  // lower bound below which no candidate can matter

  __device__ __forceinline__ void clear(int K, float base) {
#pragma unroll
    for (int t = 0; t < L; ++t) {
      f[t] = t < L - E - K ? kInf : -kInf;
      j[t] = -1;
    }
    thr = floor_ = base;
  }
  __device__ __forceinline__ float kth() const { return f[KSLOT]; }
  __device__ __forceinline__ void refresh(float band) {
    thr = fmaxf(fmaxf(f[L - 1], f[KSLOT] - band), floor_);
  }
  __device__ __forceinline__ void raise_floor(float b) {
    floor_ = fmaxf(floor_, b);
    thr = fmaxf(thr, floor_);
  }
  __device__ __forceinline__ void insert(float ff, int32_t jj, float band) {
    int pos = 0;
#pragma unroll
    for (int t = 0; t < L; ++t) pos += (f[t] > ff || (f[t] == ff && j[t] < jj)) ? 1 : 0;
#pragma unroll
    for (int t = L - 1; t > 0; --t) {
      const bool sh = t > pos, put = t == pos;
      f[t] = sh ? f[t - 1] : (put ? ff : f[t]);
      j[t] = sh ? j[t - 1] : (put ? jj : j[t]);
    }
    if (pos == 0) { f[0] = ff; j[0] = jj; }
    refresh(band);
  }
};

// Top-K list plus a band pool (single-product path).  The K best (a desc,
// j asc) sit in a sorted register array; candidates within `band` below the
// current K-th sit unsorted in a pool of P slots.  Admission is a >= K-th -
// band (not the 32nd best of a 32-slot sorted list), so a stream of n keys
// costs ~K ln(n/K) sorted inserts instead of ~(K+P) ln(n/(K+P)), and band
// candidates are appends.  A full pool evicts its minimum; `ovf` keeps the
// largest value dropped for lack of room, which the merge's certificate
// compares with the final threshold (dead entries, below a later K-th -
// band, are evicted first and never matter).
template <int KT, int P>
struct TopPool {
  float f[KT];
  int32_t j[KT];
  float pf[P];
  int32_t pj[P];
  int pcnt;
  float ovf, thr, floor_;

  __device__ __forceinline__ void clear(int K, float base) {
#pragma unroll
    for (int t = 0; t < KT; ++t) {
      f[t] = t < KT - K ? kInf : -kInf;
      j[t] = -1;
    }
#pragma unroll
    for (int t = 0; t < P; ++t) { pf[t] = -kInf; pj[t] = -1; }
    pcnt = 0;
    ovf = -kInf;
    thr = floor_ = base;
  }
  __device__ __forceinline__ float kth() const { return f[KT - 1]; }
  __device__ __forceinline__ void refresh(float band) { thr = fmaxf(f[KT - 1] - band, floor_); }
  __device__ __forceinline__ void raise_floor(float b) {
    floor_ = fmaxf(floor_, b);
    thr = fmaxf(thr, floor_);
  }
  __device__ __forceinline__ void pool_add(float v, int32_t jj) {
    if (pcnt < P) {
#pragma unroll
      for (int t = 0; t < P; ++t) {
        pf[t] = t == pcnt ? v : pf[t];
        pj[t] = t == pcnt ? jj : pj[t];
      }
      ++pcnt;
      return;
    }
    int mi = 0;
    float mv = pf[0];
    int32_t mj = pj[0];
#pragma unroll
    for (int t = 1; t < P; ++t) {
      const bool worse = pf[t] < mv || (pf[t] == mv && pj[t] > mj);
      mi = worse ? t : mi;
      mv = worse ? pf[t] : mv;
      mj = worse ? pj[t] : mj;
    }
    if (v > mv || (v == mv && jj < mj)) {
      ovf = fmaxf(ovf, mv);
#pragma unroll
      for (int t = 0; t < P; ++t) {
        pf[t] = t == mi ? v : pf[t];
        pj[t] = t == mi ? jj : pj[t];
      }
    } else {
      ovf = fmaxf(ovf, v);
    }
  }
  __device__ __forceinline__ void insert(float v, int32_t jj, float band) {
    if (v > f[KT - 1] || (v == f[KT - 1] && jj < j[KT - 1])) {
      const float dv = f[KT - 1];
      const int32_t dj = j[KT - 1];
      int pos = 0;
#pragma unroll
      for (int t = 0; t < KT; ++t) pos += (f[t] > v || (f[t] == v && j[t] < jj)) ? 1 : 0;
#pragma unroll
      for (int t = KT - 1; t > 0; --t) {
        const bool sh = t > pos, put = t == pos;
        f[t] = sh ? f[t - 1] : (put ? v : f[t]);
        j[t] = sh ? j[t - 1] : (put ? jj : j[t]);
      }
      if (pos == 0) { f[0] = v; j[0] = jj; }
      v = dv;
      jj = dj;
    }
    if (jj >= 0 && v >= f[KT - 1] - band) pool_add(v, jj);
    refresh(band);
  }
};

template <int L_, int E_>
struct SlotCfg { static constexpr int L = L_, E = E_; };
// split-bf16 path (eps ~ 2^-16): few near-K candidates per row
template <int K_MAX>
struct Slots;
template <> struct Slots<10> : SlotCfg<16, 6> {};
template <> struct Slots<24> : SlotCfg<32, 8> {};
// single-product fp16 path (eps ~ 2 ||x - fp16(x)|| ~ 6e-4): K <= 10 live
// entries plus 22 spare slots for the wider admission band
using SlotsF16 = SlotCfg<32, 22>;

struct RealParams {
  int64_t n;
  int nkb_seg;        // 128-byte k-blocks per operand segment (d_pad / 64)
  int d_pad;          // bf16 elements per segment
  int d;              // attribute columns (MMA k-steps past d are all zeros: skipped)
  int K;
  int key_tiles, tiles_per_seg, nseg;
  float eps, band;    // |a - s| bound and 2 eps (global)
  const float* row_eps;  // per-query-row bound (fp16 path) or nullptr
  int spin;              // producer / MMA threads spin on mbarriers instead of suspending
  int resume;            // lists continue from `partial` (key-segment launches > 0)
  int kt_base;           // first key tile of this launch
  int2* partial;      // nq x lists x L  (f32 bits, j)
  uint32_t* row_bound;  // nq: shared pruning floor (order-mapped f32)
  int64_t q_begin, q_end;
  int debug;
  unsigned long long* stats;   // debug 4: [chunks passing the max test, candidates buffered,
                               //           top-K inserts, pool adds]
};
}  // namespace

// Epilogue warps (2..): thread = query row (TMEM lane), streams the
// accumulator columns of every key tile into its candidate list.
template <class SL>
__device__ __forceinline__ void real_epilogue(uint64_t* tfull, uint64_t* tempty, uint32_t tmem,
                                              float* stash_base, const RealParams& p, int64_t q0,
                                              int seg, int kt0, int ntiles) {
  using namespace tc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ew = warp - 2;
  const int quarter = warp & 3;
  const int half = ew / 4;
  const int row = quarter * 32 + lane;
  const int64_t i = q0 + row;
  const bool live = i < p.q_end;
  const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
  constexpr int L = SL::L, E = SL::E;
  const float eps_i = (live && p.row_eps) ? p.row_eps[i] : p.eps;
  const float band_i = 2.f * eps_i;
  CandList<L, E> C;
  C.clear(p.K, -eps_i);
  if (p.resume && live) {
    // key-segment launches after the first continue the row's list
    const int lists = p.nseg * (EPI_WARPS / 4);
    const int live_n = p.K + E, pad = L - live_n;
    const int2* in = p.partial + ((size_t)(i - p.q_begin) * lists + seg * (EPI_WARPS / 4) + half) * live_n;
#pragma unroll
    for (int t = 0; t < L; ++t)
      if (t >= pad) {
        const int2 e = in[t - pad];
        C.f[t] = __int_as_float(e.x);
        C.j[t] = e.y;
      }
    C.refresh(band_i);
  }
  float published = -kInf;
  float* stash = stash_base + (threadIdx.x - 64) * 33;
  // the shared floor is read one tile ahead: the L2 round trip overlaps the
  // current tile instead of stalling every tile start (a staler floor is
  // still a valid lower bound)
  uint32_t floor_next = live ? __ldcg(p.row_bound + (i - p.q_begin)) : 0u;
  for (int t = 0; t < ntiles; ++t) {
    const int acc = t & 1;
    const uint32_t acc_phase = (t >> 1) & 1;
    mbar_wait_sleep(&tfull[acc], acc_phase);
    if (live) {
      C.raise_floor(ord2f(floor_next));
      floor_next = __ldcg(p.row_bound + (i - p.q_begin));
    }
    tc_fence_after();
    const int64_t j0 = (int64_t)(kt0 + t) * BN + half * EPI_COLS;
#pragma unroll 1
    for (int ch = 0; ch < EPI_COLS / 32; ++ch) {
      uint32_t r[32];
      tmem_ld32(tmem + lane_off + acc * BN + half * EPI_COLS + ch * 32, r);
      tmem_ld_wait();
      if (ch == EPI_COLS / 32 - 1) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      }
      if (p.debug == 1) continue;
      // common case first: one max tree over the 32 columns (~1 op/column);
      // the per-column mask and the stash are built only when some column
      // reaches the admission threshold
      float mx[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) mx[u] = fmaxf(__uint_as_float(r[u]), __uint_as_float(r[u + 16]));
#pragma unroll
      for (int w = 8; w > 0; w >>= 1)
#pragma unroll
        for (int u = 0; u < w; ++u) mx[u] = fmaxf(mx[u], mx[u + w]);
      if (mx[0] < C.thr) continue;
      const int64_t jb = j0 + ch * 32;
      uint32_t mask = 0;
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const float v = __uint_as_float(r[u]);
        mask |= (uint32_t)(v >= C.thr) << u;
        stash[u] = v;
      }
      if (i >= jb && i < jb + 32) mask &= ~(1u << (int)(i - jb));   // j != i
      if (jb + 32 > p.n) mask &= p.n > jb ? (1u << (int)(p.n - jb)) - 1u : 0u;
#pragma unroll 1
      while (mask) {
        const int u = __ffs(mask) - 1;
        mask &= mask - 1;
        const float v = stash[u];
        if (v < C.thr) continue;
        C.insert(v, (int32_t)(jb + u), band_i);
        const float b = C.kth() - band_i;
        if (b > published && live) {
          atomicMax(p.row_bound + (i - p.q_begin), f2ord(b));
          published = b;
        }
      }
    }
  }
  if (live) {
    const int lists = p.nseg * (EPI_WARPS / 4);
    const int live_n = p.K + E, pad = L - live_n;
    int2* out = p.partial + ((size_t)(i - p.q_begin) * lists + seg * (EPI_WARPS / 4) + half) * live_n;
#pragma unroll
    for (int t = 0; t < L; ++t)
      if (t >= pad) out[t - pad] = make_int2(__float_as_int(C.f[t]), C.j[t]);
  }
}

// Epilogue of the single-product path.  Same admission rule and outputs as
// real_epilogue, restructured for a warp of 32 independent rows:
// * two 32-column chunks per TMEM wait (64 accumulator registers in flight);
// * candidates that pass the admission threshold are appended to a small
//   per-thread buffer (register selects, ~20 instructions) instead of being
//   inserted into the sorted list at once; when any lane's buffer is half
//   full the whole warp drains its buffers in lockstep.  A sorted insert is
//   ~450 instructions, and unbatched the warp executes one per lane per event
//   (lanes hit candidates at independent times); batched, the lanes insert
//   together.  The threshold is refreshed at each drain, so between drains it
//   is a (valid, lower) stale bound.
template <class SL, bool PAIR = false, int TN = tc::BN>
__device__ __forceinline__ void real_epilogue_batched(uint64_t* tfull, uint64_t* tempty,
                                                      uint32_t tmem, float* stash_base,
                                                      const RealParams& p, int64_t q0, int seg,
                                                      int kt0, int ntiles) {
  using namespace tc;
  // TN key columns per accumulator tile, NACC tiles in TMEM (512 columns);
  // ntiles counts TN-column tiles from key tile kt0 (in BN units)
  constexpr int NACC = TMEM_COLS / TN;
  constexpr int ECOLS = TN / (EPI_WARPS / 4);     // columns per epilogue warp and tile
  constexpr int PB = 8, DRAIN = 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ew = warp - 2;
  const int quarter = warp & 3;
  const int half = ew / 4;
  const int row = quarter * 32 + lane;
  const int64_t i = q0 + row;
  const bool live = i < p.q_end;
  const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
  constexpr int L = SL::L, E = SL::E;
  constexpr int KT = L - E, P = E - 1;   // top list (K <= KT), pool, 1 overflow slot
  const float eps_i = (live && p.row_eps) ? p.row_eps[i] : p.eps;
  const float band_i = 2.f * eps_i;
  TopPool<KT, P> C;
  C.clear(p.K, -eps_i);
  const int lists = p.nseg * (EPI_WARPS / 4);
  // list layout (live_n = K + E int2): K top entries (a desc), the pool
  // (compact, unsorted), padding (-inf, -1), and in the last slot
  // (ovf, -1): the merge stops at the first id < 0 and reads the last slot
  // as the bound on dropped candidates
  const int live_n = p.K + E, padk = KT - p.K;
  int2* slot = p.partial + ((size_t)(live ? i - p.q_begin : 0) * lists + seg * (EPI_WARPS / 4) + half) * live_n;
  if (p.resume && live) {
#pragma unroll
    for (int t = 0; t < KT; ++t)
      if (t >= padk) {
        const int2 e = slot[t - padk];
        C.f[t] = __int_as_float(e.x);
        C.j[t] = e.y;
      }
#pragma unroll
    for (int t = 0; t < P; ++t) {
      const int2 e = slot[p.K + t];
      C.pf[t] = __int_as_float(e.x);
      C.pj[t] = e.y;
      C.pcnt += e.y >= 0 ? 1 : 0;
    }
    C.ovf = __int_as_float(slot[live_n - 1].x);
    C.refresh(band_i);
  }
  if (!live) C.raise_floor(kInf);          // padding rows admit nothing
  float pf[PB];
  int32_t pj[PB];
  int pc = 0;
  float published = -kInf;
  float* stash = stash_base + (threadIdx.x - 64) * 33;
  // drain(upto): insert the buffered candidates; upto bounds the loop (the
  // warp-wide maximum of pc when all lanes drain together, PB otherwise)
  unsigned long long st_chunks = 0, st_cand = 0, st_top = 0, st_pool = 0;
  auto drain = [&](int upto) {
#pragma unroll
    for (int t = 0; t < PB; ++t) {
      if (t >= upto) break;
      if (t < pc && pf[t] >= C.thr) {
        if (p.debug == 4) {
          if (pf[t] > C.f[KT - 1] || (pf[t] == C.f[KT - 1] && pj[t] < C.j[KT - 1])) ++st_top;
          else ++st_pool;
        }
        C.insert(pf[t], pj[t], band_i);
      }
    }
    pc = 0;
    const float b = C.kth() - band_i;
    if (b > published && live) {
      atomicMax(p.row_bound + (i - p.q_begin), f2ord(b));
      published = b;
    }
  };
  // The shared floor is fetched one tile ahead into this thread's spare
  // stash slot by cp.async: a register copy of it was spilled (the load's
  // latency then stalled every tile on the spill store)
  uint32_t* floor_slot = reinterpret_cast<uint32_t*>(stash) + 32;
  const uint32_t* floor_src = p.row_bound + (live ? i - p.q_begin : 0);
  auto fetch_floor = [&]() {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n\tcp.async.commit_group;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(floor_slot)),
                 "l"(floor_src)
                 : "memory");
  };
  *floor_slot = 0u;
  if (live) fetch_floor();
  for (int t = 0; t < ntiles; ++t) {
    const int acc = t % NACC;
    const uint32_t acc_phase = (t / NACC) & 1;
    mbar_wait_backoff(&tfull[acc], acc_phase);
    if (live) {
      asm volatile("cp.async.wait_all;" ::: "memory");
      C.raise_floor(ord2f(*reinterpret_cast<volatile uint32_t*>(floor_slot)));
      fetch_floor();
    }
    tc_fence_after();
    const int64_t j0 = (int64_t)kt0 * BN + (int64_t)t * TN + half * ECOLS;
#pragma unroll 1
    for (int ch = 0; ch < ECOLS / 32; ch += 2) {
      uint32_t r[2][32];
      tmem_ld32(tmem + lane_off + acc * TN + half * ECOLS + ch * 32, r[0]);
      tmem_ld32(tmem + lane_off + acc * TN + half * ECOLS + (ch + 1) * 32, r[1]);
      tmem_ld_wait();
      if (ch + 2 == ECOLS / 32) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (PAIR) mbar_arrive_remote(mapa_rank(&tempty[acc], 0));   // leader's
          else mbar_arrive(&tempty[acc]);
        }
      }
      if (p.debug == 1) continue;
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const float cmax = max32_f32(r[h2]);
        if (cmax >= C.thr && p.debug != 3) {   // debug 3: the scan without admissions
          if (p.debug == 4) ++st_chunks;
          const int64_t jb = j0 + (ch + h2) * 32;
          uint32_t mask = 0;
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            const float v = __uint_as_float(r[h2][u]);
            mask |= (uint32_t)(v >= C.thr) << u;
            stash[u] = v;
          }
          if (i >= jb && i < jb + 32) mask &= ~(1u << (int)(i - jb));   // j != i
          if (jb + 32 > p.n) mask &= p.n > jb ? (1u << (int)(p.n - jb)) - 1u : 0u;
#pragma unroll 1
          while (mask) {
            const int u = __ffs(mask) - 1;
            mask &= mask - 1;
            const float v = stash[u];
            if (pc == PB) drain(PB);               // overflow (divergent: no warp sync)
            if (v < C.thr) continue;
#pragma unroll
            for (int q = 0; q < PB; ++q) {
              pf[q] = q == pc ? v : pf[q];
              pj[q] = q == pc ? (int32_t)(jb + u) : pj[q];
            }
            ++pc;
            if (p.debug == 4) ++st_cand;
          }
        }
      }
      if (__any_sync(0xffffffffu, pc >= DRAIN)) drain(__reduce_max_sync(0xffffffffu, pc));
    }
  }
  drain(__reduce_max_sync(0xffffffffu, pc));
  if (p.debug == 4 && p.stats && live) {
    atomicAdd(p.stats + 0, st_chunks);
    atomicAdd(p.stats + 1, st_cand);
    atomicAdd(p.stats + 2, st_top);
    atomicAdd(p.stats + 3, st_pool);
  }
  if (live) {
#pragma unroll
    for (int t = 0; t < KT; ++t)
      if (t >= padk) slot[t - padk] = make_int2(__float_as_int(C.f[t]), C.j[t]);
#pragma unroll
    for (int t = 0; t < P; ++t) slot[p.K + t] = make_int2(__float_as_int(C.pf[t]), C.pj[t]);
    slot[live_n - 1] = make_int2(__float_as_int(C.ovf), -1);
  }
}

// Streaming variant (any d): A = [hi|hi|lo], B = [hi|lo|hi] k-blocks both
// streamed through the shared pipeline of knn_tc.cuh.
template <int KM>
__global__ void __launch_bounds__(tc::THREADS, 1)
knn_real_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                RealParams p) {
  using namespace tc;
  extern __shared__ __align__(1024) unsigned char smraw[];
  const Pipe P = setup(smraw, &tmA, &tmB);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t q0 = p.q_begin + (int64_t)blockIdx.x * BM;
  const int seg = blockIdx.y;
  const int kt0 = p.kt_base + seg * p.tiles_per_seg;
  const int kt1 = min(p.key_tiles, kt0 + p.tiles_per_seg);
  const int ntiles = kt1 - kt0;
  const int nkb = 3 * p.nkb_seg;

  if (warp == 0) {
    if (lane == 0) {
      const int nks = p.nkb_seg, dp = p.d_pad;
      producer(P, &tmA, &tmB, kt0, ntiles, nkb, (int)q0, [nks, dp](int kb, int& ca, int& cb) {
        const int s = kb / nks, off = (kb - s * nks) * (ROW_BYTES / 2);
        ca = (s == 2 ? dp : 0) + off;    // [hi | hi | lo]
        cb = (s == 1 ? dp : 0) + off;    // [hi | lo | hi]
      });
    }
  } else if (warp == 1) {
    if (lane == 0) mma_issuer<false>(P, ntiles, nkb, p.debug == 2);
  } else {
    real_epilogue<Slots<KM>>(P.tfull, P.tempty, P.tmem, P.stash_base, p, q0, seg, kt0, ntiles);
  }
  teardown(P);
}

// Resident-query variant (d_pad <= 192): the CTA's 128 query rows [hi|lo]
// stay in shared memory for the whole key loop; each key tile streams its
// [hi|lo] k-blocks once, and every hi block feeds two MMAs (A_hi B_hi,
// A_lo B_hi), every lo block one (A_hi B_lo).  Shared-memory fill traffic per
// key tile drops from 3 (128 + 256) d_pad to 2 * 256 d_pad elements.
namespace res {
constexpr int B_BYTES = tc::BN * tc::ROW_BYTES;   // 32 KB per k-block of 256 keys
constexpr int A_BYTES = tc::BM * tc::ROW_BYTES;   // 16 KB per k-block of 128 queries
constexpr int STASH = 32 * tc::EPI_WARPS * 33 * 4;
__host__ __device__ constexpr int stages(int nks) { return nks <= 2 ? 4 : 3; }
__host__ __device__ constexpr size_t smem(int nks) {
  return 1024 + (size_t)2 * nks * A_BYTES + (size_t)stages(nks) * B_BYTES + 256 + STASH;
}
}  // namespace res

template <int KM>
__global__ void __launch_bounds__(tc::THREADS, 1)
knn_real_res_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    RealParams p) {
  using namespace tc;
  extern __shared__ __align__(1024) unsigned char smraw[];
  const int nks = p.nkb_seg, S = res::stages(nks);
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = base;                                    // 2 nks k-blocks: hi.., lo..
  unsigned char* sB = sA + 2 * nks * res::A_BYTES;             // S stages
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + S * res::B_BYTES);
  uint64_t* empty = full + 4;
  uint64_t* tfull = empty + 4;
  uint64_t* tempty = tfull + 2;
  uint64_t* afull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(afull + 1);
  float* stash_base = reinterpret_cast<float*>(base + 2 * nks * res::A_BYTES + S * res::B_BYTES + 256);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t q0 = p.q_begin + (int64_t)blockIdx.x * BM;
  const int seg = blockIdx.y;
  const int kt0 = p.kt_base + seg * p.tiles_per_seg;
  const int kt1 = min(p.key_tiles, kt0 + p.tiles_per_seg);
  const int ntiles = kt1 - kt0;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], EPI_WARPS); }
    mbar_init(afull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int dp = p.d_pad;
  constexpr int EL = ROW_BYTES / 2;    // bf16 elements per k-block

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(afull, 2 * nks * res::A_BYTES);
      for (int kb = 0; kb < nks; ++kb) {
        tma_load_2d(sA + kb * res::A_BYTES, &tmA, afull, kb * EL, (int)q0);
        tma_load_2d(sA + (nks + kb) * res::A_BYTES, &tmA, afull, dp + kb * EL, (int)q0);
      }
      int stage = 0;
      uint32_t phase = 0;
      for (int t = 0; t < ntiles; ++t) {
        const int krow = (kt0 + t) * BN;
        for (int kb = 0; kb < nks; ++kb)
          for (int part = 0; part < 2; ++part) {          // hi, then lo
            mbar_wait_sleep(&empty[stage], phase ^ 1);
            mbar_arrive_expect_tx(&full[stage], res::B_BYTES);
            tma_load_2d(sB + stage * res::B_BYTES, &tmB, &full[stage], part * dp + kb * EL, krow);
            if (++stage == S) { stage = 0; phase ^= 1; }
          }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc(1u, BM, BN);
      const bool skip = p.debug == 2;
      mbar_wait_sleep(afull, 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int t = 0; t < ntiles; ++t) {
        const int acc = t & 1;
        const uint32_t acc_phase = (t >> 1) & 1;
        mbar_wait_sleep(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t dtm = tmem + acc * BN;
        for (int kb = 0; kb < nks; ++kb)
          for (int part = 0; part < 2; ++part) {
            mbar_wait_sleep(&full[stage], phase);
            tc_fence_after();
            const uint32_t b_addr = smem_u32(sB + stage * res::B_BYTES);
            const uint32_t ahi = smem_u32(sA + kb * res::A_BYTES);
            const uint32_t alo = smem_u32(sA + (nks + kb) * res::A_BYTES);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t bd = sw128_kmajor_desc(b_addr + k * 32);
              if (skip || kb * 64 + k * 16 >= p.d) continue;   // zero padding past d
              const bool first = kb == 0 && part == 0 && k == 0;
              mma_f16_ss(dtm, sw128_kmajor_desc(ahi + k * 32), bd, idesc, !first);  // hi x (hi|lo)
              if (part == 0) mma_f16_ss(dtm, sw128_kmajor_desc(alo + k * 32), bd, idesc, true);
            }
            mma_commit(&empty[stage]);
            if (++stage == S) { stage = 0; phase ^= 1; }
          }
        mma_commit(&tfull[acc]);
      }
    }
  } else {
    real_epilogue<Slots<KM>>(tfull, tempty, tmem, stash_base, p, q0, seg, kt0, ntiles);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<TMEM_COLS>(tmem);
}

// Single-product fp16 variant (d_pad <= 256, K <= 10): a_ij = <h_i, h_j>
// with h = fp16(xn) (subnormals flushed to 0 in the prep, so the MMA sees
// exactly the stored values).  |a_ij - s_ij| <= l_i + l_j + 3 l_i l_j +
// d_pad 2^-23 with l = ||xn - h|| (per row, measured in f64): the bound is
// ~6e-4 instead of the split path's ~2e-5, so each row keeps K + 22
// candidates, but each key tile costs one MMA per k-step instead of three.
// The CTA's 128 query rows stay resident in shared memory; key tiles stream.
namespace res16 {
constexpr int B_BYTES = tc::BN * tc::ROW_BYTES;
constexpr int A_BYTES = tc::BM * tc::ROW_BYTES;
constexpr int STASH = 32 * tc::EPI_WARPS * 33 * 4;
__host__ __device__ constexpr int stages(int nks) { return nks <= 2 ? 5 : 4; }
__host__ __device__ constexpr size_t smem(int nks) {
  return 1024 + (size_t)nks * A_BYTES + (size_t)stages(nks) * B_BYTES + 256 + STASH;
}
}  // namespace res16

template <int TN>
__global__ void __launch_bounds__(tc::THREADS, 1)
knn_real16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  RealParams p) {
  using namespace tc;
  // TN = 256: two 256-column accumulators; TN = 128: four 128-column ones
  // (the epilogue frees each after two chunk loads, and the MMA has three
  // tiles of slack instead of one); keys stream as TN-row k-blocks
  constexpr int NACC = TMEM_COLS / TN;
  constexpr int TB_BYTES = TN * ROW_BYTES;
  extern __shared__ __align__(1024) unsigned char smraw[];
  const int nks = p.nkb_seg, S = res16::stages(nks);
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = base;                                    // nks k-blocks of h
  unsigned char* sB = sA + nks * res16::A_BYTES;               // S stages
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + S * res16::B_BYTES);
  uint64_t* empty = full + 6;
  uint64_t* tfull = empty + 6;
  uint64_t* tempty = tfull + 4;
  uint64_t* afull = tempty + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(afull + 1);
  float* stash_base = reinterpret_cast<float*>(base + nks * res16::A_BYTES + S * res16::B_BYTES + 256);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t q0 = p.q_begin + (int64_t)blockIdx.x * BM;
  const int seg = blockIdx.y;
  const int kt0 = p.kt_base + seg * p.tiles_per_seg;
  const int kt1 = min(p.key_tiles, kt0 + p.tiles_per_seg);
  const int ntiles = (kt1 - kt0) * (BN / TN);   // TN-column tiles
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s2 = 0; s2 < S; ++s2) { mbar_init(&full[s2], 1); mbar_init(&empty[s2], 1); }
    for (int s2 = 0; s2 < NACC; ++s2) { mbar_init(&tfull[s2], 1); mbar_init(&tempty[s2], EPI_WARPS); }
    mbar_init(afull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr int EL = ROW_BYTES / 2;    // fp16 elements per k-block

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(afull, nks * res16::A_BYTES);
      for (int kb = 0; kb < nks; ++kb) tma_load_2d(sA + kb * res16::A_BYTES, &tmA, afull, kb * EL, (int)q0);
      int stage = 0;
      uint32_t phase = 0;
      for (int t = 0; t < ntiles; ++t) {
        const int krow = kt0 * BN + t * TN;
        for (int kb = 0; kb < nks; ++kb) {
          mbar_wait_backoff(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], TB_BYTES);
          tma_load_2d(sB + stage * res16::B_BYTES, TN == BN ? &tmB : &tmA, &full[stage], kb * EL, krow);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc(0u, BM, TN);     // kind::f16, F16 inputs
      const bool skip = p.debug == 2;
      mbar_wait_sleep(afull, 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int t = 0; t < ntiles; ++t) {
        const int acc = t % NACC;
        const uint32_t acc_phase = (t / NACC) & 1;
        mbar_wait_backoff(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t dtm = tmem + acc * TN;
        for (int kb = 0; kb < nks; ++kb) {
          mbar_wait_backoff(&full[stage], phase);
          tc_fence_after();
          const uint32_t b_addr = smem_u32(sB + stage * res16::B_BYTES);
          const uint32_t a_addr = smem_u32(sA + kb * res16::A_BYTES);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (skip || kb * 64 + k * 16 >= p.d) continue;     // zero padding past d
            mma_f16_ss(dtm, sw128_kmajor_desc(a_addr + k * 32), sw128_kmajor_desc(b_addr + k * 32),
                       idesc, (kb | k) != 0);
          }
          mma_commit(&empty[stage]);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull[acc]);
      }
    }
  } else {
    real_epilogue_batched<SlotsF16, false, TN>(tfull, tempty, tmem, stash_base, p, q0, seg, kt0, ntiles);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<TMEM_COLS>(tmem);
}

// CTA-pair variant of knn_real16_kernel: a (2,1,1) cluster covers 256
// query rows with one M=256 N=256 MMA per k-step (tcgen05 cta_group::2).
// Each CTA stages its own 128 query rows and HALF of every 256-key tile
// (keys [0,128) in rank 0, [128,256) in rank 1), so each SM pulls half the
// key bytes from L2 per tile that the 1-CTA kernel does -- the 1-CTA
// kernel streams 12 TB of keys from L2 per Amazon2M search and is bound by
// that (~9.6 TB/s), not by the tensor cores.  The accumulator layout in
// each CTA's TMEM (its 128 rows x 256 columns) and the epilogue are the
// 1-CTA ones; only the accumulator-free handshake goes to the leader.
namespace pair16 {
constexpr int HB_BYTES = (tc::BN / 2) * tc::ROW_BYTES;    // half key tile per k-block (16 KB)
constexpr int A_BYTES = tc::BM * tc::ROW_BYTES;
constexpr int STASH = 32 * tc::EPI_WARPS * 33 * 4;
constexpr int MAXS = 10;
__host__ __device__ constexpr int stages(int nks) { return nks <= 2 ? 8 : (nks <= 3 ? 7 : 6); }
__host__ __device__ constexpr size_t smem(int nks) {
  return 1024 + (size_t)nks * A_BYTES + (size_t)stages(nks) * HB_BYTES + 256 + STASH;
}
}  // namespace pair16

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(tc::THREADS, 1)
knn_real16_pair_kernel(const __grid_constant__ CUtensorMap tmA, RealParams p) {
  using namespace tc;
  extern __shared__ __align__(1024) unsigned char smraw[];
  const int nks = p.nkb_seg, S = pair16::stages(nks);
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = base;
  unsigned char* sB = sA + nks * pair16::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + S * pair16::HB_BYTES);
  uint64_t* empty = full + pair16::MAXS;
  uint64_t* tfull = empty + pair16::MAXS;
  uint64_t* tempty = tfull + 2;
  uint64_t* afull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(afull + 1);
  float* stash_base =
      reinterpret_cast<float*>(base + nks * pair16::A_BYTES + S * pair16::HB_BYTES + 256);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int64_t q0 = p.q_begin + (int64_t)blockIdx.x * BM;
  const int seg = blockIdx.y;
  const int kt0 = p.kt_base + seg * p.tiles_per_seg;
  const int kt1 = min(p.key_tiles, kt0 + p.tiles_per_seg);
  const int ntiles = kt1 - kt0;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    for (int s2 = 0; s2 < S; ++s2) { mbar_init(&full[s2], 1); mbar_init(&empty[s2], 1); }
    for (int s2 = 0; s2 < 2; ++s2) { mbar_init(&tfull[s2], 1); mbar_init(&tempty[s2], 2 * EPI_WARPS); }
    mbar_init(afull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  cluster_sync();                 // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr int EL = ROW_BYTES / 2;

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t afull_l = mapa_rank(afull, 0);
      if (rank == 0) mbar_arrive_expect_tx(afull, 2 * nks * pair16::A_BYTES);
      for (int kb = 0; kb < nks; ++kb)
        tma_load_2d_pair(sA + kb * pair16::A_BYTES, &tmA, afull_l, kb * EL, (int)q0);
      int stage = 0;
      uint32_t phase = 0;
      for (int t = 0; t < ntiles; ++t) {
        const int krow = (kt0 + t) * BN + (int)rank * (BN / 2);
        for (int kb = 0; kb < nks; ++kb) {
          mbar_wait_backoff(&empty[stage], phase ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * pair16::HB_BYTES);
          tma_load_2d_pair(sB + stage * pair16::HB_BYTES, &tmA, mapa_rank(&full[stage], 0),
                           kb * EL, krow);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = make_idesc(0u, 2 * BM, BN);   // kind::f16, F16, M=256
      const bool skip = p.debug == 2;
      mbar_wait_sleep(afull, 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int t = 0; t < ntiles; ++t) {
        const int acc = t & 1;
        const uint32_t acc_phase = (t >> 1) & 1;
        mbar_wait_backoff(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t dtm = tmem + acc * BN;
        for (int kb = 0; kb < nks; ++kb) {
          mbar_wait_backoff(&full[stage], phase);
          tc_fence_after();
          const uint32_t b_addr = smem_u32(sB + stage * pair16::HB_BYTES);
          const uint32_t a_addr = smem_u32(sA + kb * pair16::A_BYTES);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (skip || kb * 64 + k * 16 >= p.d) continue;
            mma_f16_ss_pair(dtm, sw128_kmajor_desc(a_addr + k * 32),
                            sw128_kmajor_desc(b_addr + k * 32), idesc, (kb | k) != 0);
          }
          mma_commit_pair(&empty[stage]);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        mma_commit_pair(&tfull[acc]);
      }
    }
  } else {
    real_epilogue_batched<SlotsF16, true>(tfull, tempty, tmem, stash_base, p, q0, seg, kt0, ntiles);
  }
  tc_fence_before();
  cluster_sync();                 // no remote arrivals or MMA writes still in flight
  tc_fence_after();
  if (warp == 1) tmem_dealloc_pair<TMEM_COLS>(tmem);
}

// warp per query row: merge the partial lists, certify, rerank in f64
template <class SL>
__global__ void knn_real_merge_kernel(const int2* __restrict__ partial, int64_t q_begin,
                                      int64_t nq, int lists, int K, float eps_g,
                                      const float* __restrict__ row_eps,
                                      const double* __restrict__ xn, int64_t ldn, int64_t d,
                                      const double* __restrict__ norms, int32_t* __restrict__ ids,
                                      double* __restrict__ scores, int32_t* __restrict__ flagged,
                                      int* __restrict__ nflag) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t li = w0; li < nq; li += nw) {
    const int64_t i = q_begin + li;
    int32_t* oid = ids + li * K;
    double* osc = scores + li * K;
    if (norms[i] == 0.0) {                       // zero row: empty list
      for (int t = lane; t < K; t += 32) { oid[t] = -1; osc[t] = 0.0; }
      continue;
    }
    constexpr int L = SL::L, E = SL::E, KSLOT = L - E - 1;
    static_assert(L <= 32, "one list entry per lane");
    const float eps = row_eps ? row_eps[i] : eps_g;
    const float band = 2.f * eps;
    const int live_n = K + E;
    // the merged list M (CandList order: a desc, j asc; L - E - K leading
    // +inf sentinels put the K-th real entry at KSLOT) spread over the
    // warp, lane t holding entry t: an insert is one ballot and one shift
    const bool slot = lane < L;
    float mf = slot && lane < L - E - K ? kInf : -kInf;
    int32_t mj = -1;
    const float floor_ = -eps;
    float thr = floor_;
    float over = -kInf;                          // best candidate any list dropped
    for (int s = 0; s < lists; ++s) {
      const int2* src = partial + ((size_t)li * lists + s) * live_n;
      over = fmaxf(over, __int_as_float(src[live_n - 1].x));
      for (int t0 = 0; t0 < live_n; t0 += 32) {
        const int t = t0 + lane;
        const int2 e = t < live_n ? src[t] : make_int2(0, -1);
        const unsigned stop = __ballot_sync(0xffffffffu, e.y < 0);   // lists end at the first j < 0
        const int lim = stop ? __ffs(stop) - 1 : 32;
        // the threshold only rises: entries below it now are refused later
        unsigned m = __ballot_sync(0xffffffffu, lane < lim && __int_as_float(e.x) >= thr);
        while (m) {
          const int b = __ffs(m) - 1;
          m &= m - 1;
          const float ff = __int_as_float(__shfl_sync(0xffffffffu, e.x, b));
          const int32_t jj = __shfl_sync(0xffffffffu, e.y, b);
          if (!(ff >= thr)) continue;                                // warp-uniform
          const int pos = __popc(__ballot_sync(0xffffffffu, slot && (mf > ff || (mf == ff && mj < jj))));
          const float uf = __shfl_up_sync(0xffffffffu, mf, 1);
          const int32_t uj = __shfl_up_sync(0xffffffffu, mj, 1);
          if (slot && lane > pos) { mf = uf; mj = uj; }
          if (slot && lane == pos) { mf = ff; mj = jj; }
          const float last = __shfl_sync(0xffffffffu, mf, L - 1);
          const float kth = __shfl_sync(0xffffffffu, mf, KSLOT);
          thr = fmaxf(fmaxf(last, kth - band), floor_);
        }
        if (stop) break;
      }
    }
    const float theta = fmaxf(__shfl_sync(0xffffffffu, mf, KSLOT) - band, -eps);
    over = fmaxf(over, __shfl_sync(0xffffffffu, mf, L - 1));
    if (!(over < theta)) {                       // not certified: exact rescan later
      if (lane == 0) flagged[atomicAdd(nflag, 1)] = (int32_t)i;
      continue;
    }
    const double* xi = xn + i * ldn;
    double sv = -1.0;                            // lane t: f64 score of entry t
    for (unsigned m = __ballot_sync(0xffffffffu, slot && mj >= 0 && mf >= theta); m; m &= m - 1) {
      const int b = __ffs(m) - 1;
      const double* xj = xn + (int64_t)__shfl_sync(0xffffffffu, mj, b) * ldn;
      double acc = 0.0;
      for (int64_t c = lane; c < d; c += 32) acc = fma(xi[c], xj[c], acc);
      acc = warp_sum(acc);
      if (lane == b) sv = acc;
    }
    // top K of (s desc, j asc) among s > 0: each entry's rank among them
    const bool live = sv > 0.0;
    int rank = 0;
    for (int u = 0; u < L; ++u) {
      const double su = __shfl_sync(0xffffffffu, sv, u);
      const int32_t ju = __shfl_sync(0xffffffffu, mj, u);
      rank += (su > 0.0 && (su > sv || (su == sv && ju < mj))) ? 1 : 0;
    }
    const int cnt = __popc(__ballot_sync(0xffffffffu, live));
    if (live && rank < K) {
      oid[rank] = mj;
      osc[rank] = fmin(sv, 1.0);
    }
    for (int r = cnt + lane; r < K; r += 32) {
      oid[r] = -1;
      osc[r] = 0.0;
    }
  }
}

// f64 X -> xn (f64, ldn, zero padded) + norms + [hi | lo] bf16 (n_pad x 2 d_pad)
__global__ void knn_real_prep_kernel(const double* __restrict__ X, int64_t n, int64_t d,
                                     int64_t ldx, int64_t n_pad, int64_t d_pad,
                                     double* __restrict__ xn, int64_t ldn,
                                     double* __restrict__ norms, __nv_bfloat16* __restrict__ H) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < n_pad; r += nw) {
    double inv = 0.0;
    if (r < n) {
      const double* x = X + r * ldx;
      double nrm = 0.0;
      if (lane == 0)  // np.linalg.norm(x, axis=1): sqrt of the pairwise sum of x*x
        nrm = sqrt(np_pairwise_sum_g([x](int64_t c) { return __dmul_rn(x[c], x[c]); }, d));
      nrm = __shfl_sync(0xffffffffu, nrm, 0);
      inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
      if (lane == 0) norms[r] = nrm;
    }
    __nv_bfloat16* h = H + r * 2 * d_pad;
    for (int64_t c = lane; c < d_pad; c += 32) {
      const double v = (r < n && c < d) ? __dmul_rn(X[r * ldx + c], inv) : 0.0;
      if (r < n && c < ldn) xn[r * ldn + c] = v;
      const __nv_bfloat16 hi = __double2bfloat16(v);
      const __nv_bfloat16 lo = __double2bfloat16(v - (double)__bfloat162float(hi));
      h[c] = hi;
      h[d_pad + c] = lo;
    }
    if (r < n)
      for (int64_t c = d_pad + lane; c < ldn; c += 32) xn[r * ldn + c] = 0.0;
  }
}

// f64 X -> xn (f64) + norms + h = fp16(xn) (n_pad x d_pad, subnormals
// flushed to zero) + lo[i] = ||xn_i - h_i|| (rounded up) + max_i lo[i]
__global__ void knn_real16_prep_kernel(const double* __restrict__ X, int64_t n, int64_t d,
                                       int64_t ldx, int64_t n_pad, int64_t d_pad,
                                       double* __restrict__ xn, int64_t ldn,
                                       double* __restrict__ norms, __half* __restrict__ H,
                                       float* __restrict__ lo, uint32_t* __restrict__ lo_max) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < n_pad; r += nw) {
    double inv = 0.0;
    if (r < n) {
      const double* x = X + r * ldx;
      double nrm = 0.0;
      if (lane == 0)  // np.linalg.norm(x, axis=1): sqrt of the pairwise sum of x*x
        nrm = sqrt(np_pairwise_sum_g([x](int64_t c) { return __dmul_rn(x[c], x[c]); }, d));
      nrm = __shfl_sync(0xffffffffu, nrm, 0);
      inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
      if (lane == 0) norms[r] = nrm;
    }
    __half* h = H + r * d_pad;
    double l2 = 0.0;
    for (int64_t c = lane; c < d_pad; c += 32) {
      const double v = (r < n && c < d) ? __dmul_rn(X[r * ldx + c], inv) : 0.0;
      if (r < n && c < ldn) xn[r * ldn + c] = v;
      __half hv = __double2half(v);
      if (fabs(v) < 0x1p-14) hv = __double2half(0.0);      // no fp16 subnormals
      h[c] = hv;
      const double e = v - (double)__half2float(hv);
      l2 = fma(e, e, l2);
    }
    if (r < n) {
      for (int64_t c = d_pad + lane; c < ldn; c += 32) xn[r * ldn + c] = 0.0;
      l2 = warp_sum(l2);
      if (lane == 0) {
        const float l = (float)(sqrt(l2) * (1.0 + 1e-6)) + 1e-30f;
        lo[r] = l;
        atomicMax(lo_max, __float_as_uint(l));             // l >= 0: bit order = value order
      }
    }
  }
}

// per-row certificate bound eps_i = l_i + l_max + 3 l_i l_max + d_pad 2^-23
__global__ void knn_real16_eps_kernel(const float* __restrict__ lo, const uint32_t* __restrict__ lo_max,
                                      int64_t n, float acc_eps, float* __restrict__ row_eps) {
  const float lm = __uint_as_float(*lo_max);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float l = lo[i];
    row_eps[i] = (l + lm + 3.f * l * lm + acc_eps) * (1.f + 1e-5f);
  }
}

// ----------------------------------------------------------------- host side
namespace {
struct RealLayout {
  int64_t n_pad, d_pad, ldn;
  TcGrid g;
  int lists;
  KeyRange kr;
};

RealLayout real_layout(int64_t n, int64_t d, int64_t nq, KeyRange kr = {0, -1}) {
  RealLayout R;
  R.n_pad = ceil_div(n, tc::BN) * tc::BN;
  R.d_pad = ceil_div(d, 64) * 64;
  R.ldn = ceil_div(d, 16) * 16;
  R.g = tc_grid(n, nq, kr);
  R.kr = {kr.k0, kr.k1 < 0 ? n : kr.k1};
  R.lists = R.g.nseg * (tc::EPI_WARPS / 4);
  return R;
}

// partial-list slots per list: the fp16 path (K <= 10) keeps K + 22 live
int real_slots(int K) { return K <= 10 ? SlotsF16::L : Slots<24>::L; }
bool use_f16_path(int K, int64_t d_pad) {
  static const bool split = getenv("ANCKA_KNN_SPLIT") != nullptr;
  return !split && K <= 10 && d_pad <= 256;
}

struct RealWs {
  __nv_bfloat16* H;
  double *xn, *norms;
  uint32_t* rb;
  int2* part;
  int32_t* flagged;
  int* nflag;
  void* simt_ws;
  size_t simt_wsb;
  float *lo, *row_eps;
  uint32_t* lo_max;
};

void carve_real(Carver& cv, const RealLayout& R, int64_t n, int K, RealWs& w) {
  const int L = real_slots(K);
  w.H = cv.take<__nv_bfloat16>((size_t)R.n_pad * 2 * R.d_pad);
  w.xn = cv.take<double>((size_t)n * R.ldn);
  w.norms = cv.take<double>(n);
  w.rb = cv.take<uint32_t>(n);
  // nq * lists <= (n + 8 * 148 * BM) * 2 for every query range (see tc_grid)
  w.part = cv.take<int2>(((size_t)n + 8 * kNumSMs * tc::BM) * (tc::EPI_WARPS / 4) * L);
  w.flagged = cv.take<int32_t>(n);
  w.nflag = cv.take<int>(1);
  w.simt_wsb = knn_simt_list_workspace(K);
  w.simt_ws = cv.take<unsigned char>(w.simt_wsb);
  w.lo = cv.take<float>(n);
  w.row_eps = cv.take<float>(n);
  w.lo_max = cv.take<uint32_t>(1);
}

template <int KM>
int launch_real(const CUtensorMap& ma, const CUtensorMap& mb, const RealParams& p,
                const RealLayout& R, cudaStream_t st) {
  dim3 grid(R.g.q_tiles, R.g.nseg);
  const bool resident = p.nkb_seg <= 3 && !getenv("ANCKA_KNN_STREAM_A");
  if (resident) {
    auto kern = knn_real_res_kernel<KM>;
    const size_t sm = res::smem(p.nkb_seg);
    ANCKA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<grid, tc::THREADS, sm, st>>>(ma, mb, p);
  } else {
    auto kern = knn_real_kernel<KM>;
    ANCKA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc::SMEM));
    kern<<<grid, tc::THREADS, tc::SMEM, st>>>(ma, mb, p);
  }
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}
}  // namespace

namespace {
int knn_real16(const double* X, int64_t n, int64_t d, int64_t ldx, int K, int64_t q_begin,
               int64_t q_end, int32_t* ids, double* scores, const RealLayout& R, const RealWs& w,
               cudaStream_t st) {
  const int64_t nq = q_end - q_begin;
  __half* H = reinterpret_cast<__half*>(w.H);       // n_pad x d_pad fits the [hi|lo] buffer
  ANCKA_CUDA(cudaMemsetAsync(w.lo_max, 0, sizeof(uint32_t), st));
  const int pg = (int)std::min<int64_t>(ceil_div(R.n_pad * 32, 256), 16 * kNumSMs);
  knn_real16_prep_kernel<<<pg, 256, 0, st>>>(X, n, d, ldx, R.n_pad, R.d_pad, w.xn, R.ldn, w.norms,
                                             H, w.lo, w.lo_max);
  ANCKA_LAUNCHED();
  const float acc_eps = (float)((double)R.d_pad * 0x1p-23);
  knn_real16_eps_kernel<<<(int)std::min<int64_t>(ceil_div(n, 256), 8 * kNumSMs), 256, 0, st>>>(
      w.lo, w.lo_max, n, acc_eps, w.row_eps);
  ANCKA_LAUNCHED();
  CUtensorMap ma, mb;
  ANCKA_TRY(tc_make_map(&ma, H, false, R.n_pad, R.d_pad, tc::BM));
  ANCKA_TRY(tc_make_map(&mb, H, false, R.n_pad, R.d_pad, tc::BN));
  RealParams p;
  p.n = R.kr.k1;                         // key index bound
  p.nkb_seg = (int)(R.d_pad / 64);
  p.d_pad = (int)R.d_pad;
  p.d = (int)d;
  p.K = K;
  p.key_tiles = (int)(R.kr.k0 / tc::BN) + R.g.key_tiles;
  p.tiles_per_seg = R.g.tiles_per_seg;
  p.nseg = R.g.nseg;
  p.eps = 0.f;
  p.band = 0.f;
  p.row_eps = w.row_eps;
  p.resume = 0;
  p.kt_base = (int)(R.kr.k0 / tc::BN);
  p.partial = w.part;
  p.row_bound = w.rb;
  p.q_begin = q_begin;
  p.q_end = q_end;
  p.debug = getenv("ANCKA_KNN_DEBUG") ? atoi(getenv("ANCKA_KNN_DEBUG")) : 0;
  p.spin = getenv("ANCKA_KNN_SPIN") ? atoi(getenv("ANCKA_KNN_SPIN")) : 0;
  p.stats = nullptr;
  if (p.debug == 4) {
    ANCKA_CUDA(cudaMallocAsync(&p.stats, 4 * sizeof(unsigned long long), st));
    ANCKA_CUDA(cudaMemsetAsync(p.stats, 0, 4 * sizeof(unsigned long long), st));
  }
  ANCKA_CUDA(cudaMemsetAsync(w.rb, 0, sizeof(uint32_t) * nq, st));
  ANCKA_CUDA(cudaMemsetAsync(w.nflag, 0, sizeof(int), st));
  // Key segments as successive launches over all query tiles: the CTAs in
  // flight all stream the same <= ~40 MB of keys, which stays in L2 (one
  // launch over all n keys re-reads the key matrix from HBM once CTAs drift
  // apart: 6.8 TB of DRAM reads at Amazon2M).  Row lists carry across
  // launches through `partial`.
  const int64_t key_bytes = (int64_t)tc::BN * R.d_pad * 2;
  int seg_tiles = (int)std::max<int64_t>(1, (40ll << 20) / key_bytes);
  if (const char* e = getenv("ANCKA_KNN_SEG_TILES")) seg_tiles = std::max(1, atoi(e));
  const int kt_first = (int)(R.kr.k0 / tc::BN);
  const int nlaunch = (int)ceil_div(R.g.key_tiles, seg_tiles);
  int lists = R.lists;
  // CTA pairs (cta_group::2) only with ANCKA_KNN_PAIR=1 (measured equal)
  const bool pair = getenv("ANCKA_KNN_PAIR") && atoi(getenv("ANCKA_KNN_PAIR")) != 0;
  // 128-key accumulator tiles (four TMEM buffers: more slack between the MMA
  // and the epilogue) only with ANCKA_KNN_N128=1: measured slower (Amazon2M
  // 2.48 s against 1.85 s; 2.09 s with the admission work skipped)
  const bool n128 = getenv("ANCKA_KNN_N128") && atoi(getenv("ANCKA_KNN_N128")) != 0;
  const size_t sm = pair ? pair16::smem(p.nkb_seg) : res16::smem(p.nkb_seg);
  const int qt = pair ? (int)((R.g.q_tiles + 1) & ~1) : R.g.q_tiles;
  if (pair)
    ANCKA_CUDA(cudaFuncSetAttribute(knn_real16_pair_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  else
    ANCKA_CUDA(cudaFuncSetAttribute(n128 ? knn_real16_kernel<128> : knn_real16_kernel<256>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  auto launch = [&](dim3 grid) {
    if (pair) knn_real16_pair_kernel<<<grid, tc::THREADS, sm, st>>>(ma, p);
    else if (n128) knn_real16_kernel<128><<<grid, tc::THREADS, sm, st>>>(ma, mb, p);
    else knn_real16_kernel<256><<<grid, tc::THREADS, sm, st>>>(ma, mb, p);
  };
  if (nlaunch <= 1) {
    launch(dim3(qt, R.g.nseg));
    ANCKA_LAUNCHED();
  } else {
    p.nseg = 1;
    p.tiles_per_seg = seg_tiles;
    lists = tc::EPI_WARPS / 4;
    for (int l = 0; l < nlaunch; ++l) {
      p.kt_base = kt_first + l * seg_tiles;
      p.resume = l > 0;
      launch(dim3(qt, 1));
      ANCKA_LAUNCHED();
    }
  }
  if (p.stats) {   // debug 4: admission counters
    unsigned long long h[4];
    ANCKA_CUDA(cudaMemcpyAsync(h, p.stats, sizeof(h), cudaMemcpyDeviceToHost, st));
    ANCKA_CUDA(cudaStreamSynchronize(st));
    fprintf(stderr, "knn16 admissions: rows %lld chunks>=thr %llu candidates %llu top-K inserts %llu pool adds %llu\n",
            (long long)nq, h[0], h[1], h[2], h[3]);
    ANCKA_CUDA(cudaFreeAsync(p.stats, st));
  }
  const int mg = (int)std::min<int64_t>(ceil_div(nq * 32, 256), 16 * kNumSMs);
  knn_real_merge_kernel<SlotsF16><<<mg, 256, 0, st>>>(w.part, q_begin, nq, lists, K, 0.f,
                                                      w.row_eps, w.xn, R.ldn, d, w.norms, ids,
                                                      scores, w.flagged, w.nflag);
  ANCKA_LAUNCHED();
  return knn_simt_list(w.xn, n, R.ldn, w.norms, K, q_begin, w.flagged, w.nflag, ids, scores,
                       w.simt_ws, w.simt_wsb, st);
}
}  // namespace

size_t knn_real_workspace(int64_t n, int64_t d, int K) {
  Carver cv(nullptr, 0);
  RealWs w;
  carve_real(cv, real_layout(n, d, n), n, K, w);
  return cv.used;
}

int knn_real(const double* X, int64_t n, int64_t d, int64_t ldx, int K, int64_t q_begin,
             int64_t q_end, int32_t* ids, double* scores, void* ws, size_t wsb, cudaStream_t st,
             KeyRange kr) {
  ANCKA_REQUIRE(K <= 24, ANCKA_ERR_UNSUPPORTED, "tensor-core real KNN supports K <= 24 (got %d)", K);
  ANCKA_REQUIRE(n < (1ll << 31), ANCKA_ERR_UNSUPPORTED, "tensor-core KNN: n too large");
  const int64_t nq = q_end - q_begin;
  const RealLayout R = real_layout(n, d, nq, kr);
  ANCKA_REQUIRE(R.kr.k0 % tc::BN == 0 && R.kr.k0 < R.kr.k1 && R.kr.k1 <= n, ANCKA_ERR_ARG,
                "knn: key range must start on a %d-row tile", tc::BN);
  Carver cv(ws, wsb);
  RealWs w;
  carve_real(cv, R, n, K, w);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "knn_real: workspace too small");
  const int pg = (int)std::min<int64_t>(ceil_div(R.n_pad * 32, 256), 16 * kNumSMs);
  if (use_f16_path(K, R.d_pad))
    return knn_real16(X, n, d, ldx, K, q_begin, q_end, ids, scores, R, w, st);
  knn_real_prep_kernel<<<pg, 256, 0, st>>>(X, n, d, ldx, R.n_pad, R.d_pad, w.xn, R.ldn, w.norms, w.H);
  ANCKA_LAUNCHED();

  CUtensorMap ma, mb;
  ANCKA_TRY(tc_make_map(&ma, w.H, false, R.n_pad, 2 * R.d_pad, tc::BM));
  ANCKA_TRY(tc_make_map(&mb, w.H, false, R.n_pad, 2 * R.d_pad, tc::BN));
  RealParams p;
  p.n = R.kr.k1;                         // key index bound
  p.nkb_seg = (int)(R.d_pad / 64);
  p.d_pad = (int)R.d_pad;
  p.d = (int)d;
  p.K = K;
  p.key_tiles = (int)(R.kr.k0 / tc::BN) + R.g.key_tiles;
  p.tiles_per_seg = R.g.tiles_per_seg;
  p.nseg = R.g.nseg;
  // |a - s| <= 2^-16 (bf16 hi/lo split of two unit vectors, cross terms and
  // the dropped lo*lo) + 3 d_pad * 2^-23 (f32 accumulation of the terms)
  p.eps = (float)(1.6e-5 + 3.0 * (double)R.d_pad * 0x1p-23);
  if (const char* e = getenv("ANCKA_KNN_EPS")) p.eps = (float)atof(e);
  p.band = 2.f * p.eps;
  p.row_eps = nullptr;
  p.spin = 0;
  p.resume = 0;
  p.kt_base = (int)(R.kr.k0 / tc::BN);
  p.partial = w.part;
  p.row_bound = w.rb;
  p.q_begin = q_begin;
  p.q_end = q_end;
  p.debug = getenv("ANCKA_KNN_DEBUG") ? atoi(getenv("ANCKA_KNN_DEBUG")) : 0;
  ANCKA_CUDA(cudaMemsetAsync(w.rb, 0, sizeof(uint32_t) * nq, st));
  ANCKA_CUDA(cudaMemsetAsync(w.nflag, 0, sizeof(int), st));
  if (K <= 10) { ANCKA_TRY(launch_real<10>(ma, mb, p, R, st)); }
  else { ANCKA_TRY(launch_real<24>(ma, mb, p, R, st)); }

  const int mg = (int)std::min<int64_t>(ceil_div(nq * 32, 256), 16 * kNumSMs);
  if (K <= 10)
    knn_real_merge_kernel<Slots<10>><<<mg, 256, 0, st>>>(w.part, q_begin, nq, R.lists, K, p.eps, nullptr,
                                                  w.xn, R.ldn, d, w.norms, ids, scores, w.flagged, w.nflag);
  else
    knn_real_merge_kernel<Slots<24>><<<mg, 256, 0, st>>>(w.part, q_begin, nq, R.lists, K, p.eps, nullptr,
                                                  w.xn, R.ldn, d, w.norms, ids, scores, w.flagged, w.nflag);
  ANCKA_LAUNCHED();
  // uncertified rows: exact f64 rescan over all keys (device-side count)
  return knn_simt_list(w.xn, n, R.ldn, w.norms, K, q_begin, w.flagged, w.nflag, ids, scores,
                       w.simt_ws, w.simt_wsb, st);
}

int knn_real_flag_count(void* ws, size_t wsb, int64_t n, int64_t d, int K, int64_t q_begin,
                        int64_t q_end, int* out_host) {
  const RealLayout R = real_layout(n, d, q_end - q_begin);
  Carver cv(ws, wsb);
  RealWs w;
  carve_real(cv, R, n, K, w);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "knn_real: workspace too small");
  ANCKA_CUDA(cudaMemcpy(out_host, w.nflag, sizeof(int), cudaMemcpyDeviceToHost));
  return ANCKA_OK;
}

int knn_real_flag_count_async(void* ws, size_t wsb, int64_t n, int64_t d, int K, int64_t q_begin,
                              int64_t q_end, int* out_dev, cudaStream_t st) {
  const RealLayout R = real_layout(n, d, q_end - q_begin);
  Carver cv(ws, wsb);
  RealWs w;
  carve_real(cv, R, n, K, w);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "knn_real: workspace too small");
  ANCKA_CUDA(cudaMemcpyAsync(out_dev, w.nflag, sizeof(int), cudaMemcpyDeviceToDevice, st));
  return ANCKA_OK;
}

}  // namespace ancka
