// Approximate cosine KNN through an inverted-file index (SURVEY.md §8(f)
// row f4; reference knn.py:143-280, `knn_search_approx`).
//
// The reference trains nlist centroids on a sample, assigns every row to its
// best centroid by inner product (the inverted lists), and for every query
// scans the union of its nprobe best lists, keeping the top-K positive
// similarities (score desc, index asc).  On the B200 the same index lives in
// HBM and the scan is turned inside out: queries are grouped by the lists
// they probe, so one CTA holds a tile of 64 (query, list) pairs and streams
// that list's keys once for all of them.
//
//   ivf_normalize  xn = f32(x * (1/||x||)) with numpy's norm (knn.py:54-65;
//                  the approximate path searches the f32 copy, knn.py:174)
//   ivf_gemm       S = A B^T + bias (f32 SIMT tiles, 128 x 128, 8 x 8 per
//                  thread): stored (probe scores) or reduced to a first-max
//                  argmax per row through a packed 64-bit atomicMax
//                  (list assignment, k-means assignment)
//   ivf_topsel     per row, the nprobe largest of nb scores (radix select on
//                  order-preserving keys, ties to the smaller centroid)
//   ivf_bucket     counting sort of (row, slot) entries by key: the inverted
//                  lists and the list -> (query, slot) pair lists
//   ivf_search     per (list, 64-pair tile): f32 dots of the tile's queries
//                  with every key of the list, per-pair top-K2 (K2 = K + 8)
//                  of the scores above -e, e the f32 error bound of a dot,
//                  and above the best K2-th score any finished pair of the
//                  same query has reached (a per-query global threshold)
//   ivf_merge      per query (warp): top-K2 of its nprobe partial lists by
//                  f32 score, re-ranked with f64 accumulation of the f32
//                  products (exact), top-K positive by (score desc, id asc);
//                  a row whose f64 K-th score does not clear the K2-th f32
//                  score + e is flagged
//   ivf_rows_exact flagged rows (and the recall-audit rows against all keys):
//                  every candidate scored with f64 accumulation
//   ivf_kmeans_*   device Lloyd iterations for the centroids: 64-bit
//                  fixed-point cluster sums (order-free, deterministic)
//
// Every selection is a total order (score desc, id asc), so the results do
// not depend on the order of entries inside a list or on CTA scheduling.
#include <cfloat>
#include <cuda_fp16.h>

#include "common.cuh"

namespace ancka {
namespace ivf {

constexpr int kT = 256;
constexpr int TQ = 64, TK = 64, KC = 32;

__device__ __forceinline__ uint32_t ord_key(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_ord(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// ------------------------------------------------------------ normalise ---
__global__ void ivf_normalize_dense(const double* __restrict__ X, int64_t ldx, int64_t n,
                                    int64_t d, float* __restrict__ xn, int64_t dp) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < n;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const double* x = X + r * ldx;
    double nrm = 0.0;
    if (lane == 0)  // np.linalg.norm(x, axis=1): sqrt of numpy's pairwise sum of x*x
      nrm = sqrt(np_pairwise_sum_g([x](int64_t c) { return __dmul_rn(x[c], x[c]); }, d));
    nrm = __shfl_sync(0xffffffffu, nrm, 0);
    const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
    for (int64_t c = lane; c < dp; c += 32)
      xn[r * dp + c] = c < d ? (float)__dmul_rn(x[c], inv) : 0.0f;
  }
}

__global__ void ivf_normalize_csr(const int64_t* __restrict__ indptr,
                                  const int32_t* __restrict__ indices,
                                  const double* __restrict__ data, int64_t n, float* __restrict__ xn,
                                  int64_t dp) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < n;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t b = indptr[r], e = indptr[r + 1];
    double nrm = 0.0;
    if (lane == 0 && e > b) {  // scipy csr.sum(axis=1) of x.multiply(x): a[b] + pairwise(a[b+1:e])
      const double* v = data + b;
      double s = __dmul_rn(v[0], v[0]);
      if (e - b > 1)
        s = __dadd_rn(s, np_pairwise_sum_g([v](int64_t c) { return __dmul_rn(v[1 + c], v[1 + c]); },
                                           e - b - 1));
      nrm = sqrt(s);
    }
    nrm = __shfl_sync(0xffffffffu, nrm, 0);
    const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
    for (int64_t c = lane; c < dp; c += 32) xn[r * dp + c] = 0.0f;
    __syncwarp();
    for (int64_t j = b + lane; j < e; j += 32) xn[r * dp + indices[j]] = (float)__dmul_rn(data[j], inv);
  }
}

// ----------------------------------------------------------------- gemm ---
// S[r][c] = sum_k A[arow(r)][k] * B[c][k] (+ bias[c]); f32 FMA in k order.
struct GemmP {
  const float* A;
  int64_t lda;
  const int32_t* arows;
  int64_t m;
  const float* B;
  int64_t ldb;
  int32_t nb;
  int64_t d;
  const float* bias;
  float* C;
  int64_t ldc;
  unsigned long long* amax;
};

// 128 x 128 output tile per CTA, 8 x 8 per thread (rows ty + 16 i, columns
// tx + 16 j: conflict-free broadcast reads of the k-major staged operands),
// A and B staged 32 k at a time by float4 row reads; every output is the
// same k-ordered fmaf chain (zero-padded past d) as a plain dot product
constexpr int GT = 128, GLD = GT + 1;
__global__ void __launch_bounds__(kT) ivf_gemm(GemmP p) {
  __shared__ float as[KC][GLD];
  __shared__ float bs[KC][GLD];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t r0 = (int64_t)blockIdx.x * GT;
  const int c0 = blockIdx.y * GT;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;
  const bool vec = (p.lda % 4) == 0 && (p.ldb % 4) == 0;
  for (int64_t d0 = 0; d0 < p.d; d0 += KC) {
    // thread: row r = idx / 8, k quad q = idx % 8 of this 32-k block
    for (int idx = tid; idx < GT * (KC / 4); idx += kT) {
      const int r = idx >> 3, q = idx & 7;
      const int64_t k = d0 + 4 * q;
      float4 va = make_float4(0.f, 0.f, 0.f, 0.f), vb = va;
      const int64_t gr = r0 + r;
      if (gr < p.m) {
        const float* src = p.A + (p.arows ? (int64_t)p.arows[gr] : gr) * p.lda + k;
        if (vec && k + 4 <= p.d) va = *reinterpret_cast<const float4*>(src);
        else {
          if (k < p.d) va.x = src[0];
          if (k + 1 < p.d) va.y = src[1];
          if (k + 2 < p.d) va.z = src[2];
          if (k + 3 < p.d) va.w = src[3];
        }
      }
      const int gc = c0 + r;
      if (gc < p.nb) {
        const float* src = p.B + (int64_t)gc * p.ldb + k;
        if (vec && k + 4 <= p.d) vb = *reinterpret_cast<const float4*>(src);
        else {
          if (k < p.d) vb.x = src[0];
          if (k + 1 < p.d) vb.y = src[1];
          if (k + 2 < p.d) vb.z = src[2];
          if (k + 3 < p.d) vb.w = src[3];
        }
      }
      as[4 * q][r] = va.x; as[4 * q + 1][r] = va.y; as[4 * q + 2][r] = va.z; as[4 * q + 3][r] = va.w;
      bs[4 * q][r] = vb.x; bs[4 * q + 1][r] = vb.y; bs[4 * q + 2][r] = vb.z; bs[4 * q + 3][r] = vb.w;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < KC; ++kk) {
      float a[8], b[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = as[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t gr = r0 + ty + 16 * i;
    unsigned long long best = 0ull;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int gc = c0 + tx + 16 * j;
      if (gc >= p.nb) continue;
      const float s = p.bias ? acc[i][j] + p.bias[gc] : acc[i][j];
      if (p.C && gr < p.m) p.C[gr * p.ldc + gc] = s;
      const unsigned long long key = ((unsigned long long)ord_key(s) << 32) | (0xffffffffu - (uint32_t)gc);
      best = key > best ? key : best;
    }
    if (p.amax) {
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
        best = other > best ? other : best;
      }
      if (tx == 0 && gr < p.m) atomicMax(p.amax + gr, best);
    }
  }
}

__global__ void ivf_argmax_finish(unsigned long long* __restrict__ amax, int64_t m,
                                  int32_t* __restrict__ labels, int32_t* __restrict__ changed) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t lab = (int32_t)(0xffffffffu - (uint32_t)(amax[r] & 0xffffffffull));
    if (changed && labels[r] != lab) atomicAdd(changed, 1);
    labels[r] = lab;
    amax[r] = 0ull;  // ready for the next assignment
  }
}

// --------------------------------------------------------------- top-sel ---
// One warp per row: the nprobe largest of nb scores.  Radix select (4 x 8
// bits) finds the threshold key T; then keys > T, then keys == T by
// ascending centroid index until nprobe are emitted.
__global__ void __launch_bounds__(kT) ivf_topsel(const float* __restrict__ S, int64_t lds, int64_t m,
                                                  int32_t nb, int32_t nprobe,
                                                  int32_t* __restrict__ probes) {
  __shared__ int hist[kT / 32][256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int* h = hist[w];
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < m;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const float* s = S + r * lds;
    uint32_t prefix = 0, pmask = 0;
    int need = nprobe;  // how many to take among keys matching prefix (from the top)
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int b = lane; b < 256; b += 32) h[b] = 0;
      __syncwarp();
      for (int c = lane; c < nb; c += 32) {
        const uint32_t k = ord_key(s[c]);
        if ((k & pmask) == prefix) atomicAdd(&h[(k >> shift) & 255], 1);
      }
      __syncwarp();
      // digit where the count from the top crosses `need`
      int digit = 0, above = 0;
      if (lane == 0) {
        int acc = 0;
        for (int b = 255; b >= 0; --b) {
          if (acc + h[b] >= need) { digit = b; above = acc; break; }
          acc += h[b];
        }
      }
      digit = __shfl_sync(0xffffffffu, digit, 0);
      above = __shfl_sync(0xffffffffu, above, 0);
      need -= above;
      prefix |= (uint32_t)digit << shift;
      pmask |= 255u << shift;
      __syncwarp();
    }
    // emit: keys > T (count nprobe - need), then the first `need` keys == T
    int32_t* out = probes + r * (int64_t)nprobe;
    int pos = 0, eq_taken = 0;
    for (int c0 = 0; c0 < nb; c0 += 32) {
      const int c = c0 + lane;
      uint32_t k = c < nb ? ord_key(s[c]) : 0u;
      const bool gt = c < nb && k > prefix;
      const bool eq = c < nb && k == prefix;
      const unsigned bg = __ballot_sync(0xffffffffu, gt);
      const unsigned be = __ballot_sync(0xffffffffu, eq);
      const unsigned lt_mask = (1u << lane) - 1u;
      if (gt) out[pos + __popc(bg & lt_mask)] = c;
      pos += __popc(bg);
      const int eq_rank = __popc(be & lt_mask);
      if (eq && eq_taken + eq_rank < need) out[(nprobe - need) + eq_taken + eq_rank] = c;
      eq_taken += __popc(be);
      // gt entries fill [0, nprobe - need); eq entries fill [nprobe - need, nprobe)
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------- bucket ---
__global__ void ivf_bucket_count(const int32_t* __restrict__ keys, int64_t cnt, int32_t* __restrict__ c) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x)
    if (keys[i] >= 0) atomicAdd(&c[keys[i]], 1);   // negative keys: entry not bucketed
}

// exclusive scan of nbk counts (one CTA), ptr[nbk] = total; also the tile
// offsets tiles[b] = sum ceil(count / tile) when tiles != nullptr
__global__ void __launch_bounds__(1024) ivf_bucket_scan(const int32_t* __restrict__ c, int32_t nbk,
                                                        int64_t* __restrict__ ptr,
                                                        int64_t* __restrict__ tiles, int tile) {
  __shared__ int64_t part[1024], tpart[1024];
  const int t = threadIdx.x;
  const int per = (nbk + 1023) / 1024;
  const int b0 = t * per, b1 = min(nbk, b0 + per);
  int64_t s = 0, ts = 0;
  for (int b = b0; b < b1; ++b) { s += c[b]; ts += (c[b] + tile - 1) / tile; }
  part[t] = s;
  tpart[t] = ts;
  __syncthreads();
  if (t == 0) {
    int64_t a = 0, ta = 0;
    for (int i = 0; i < 1024; ++i) {
      const int64_t v = part[i], tv = tpart[i];
      part[i] = a;
      tpart[i] = ta;
      a += v;
      ta += tv;
    }
    ptr[nbk] = a;
    if (tiles) tiles[nbk] = ta;
  }
  __syncthreads();
  s = part[t];
  ts = tpart[t];
  for (int b = b0; b < b1; ++b) {
    ptr[b] = s;
    s += c[b];
    if (tiles) {
      tiles[b] = ts;
      ts += (c[b] + tile - 1) / tile;
    }
  }
}

__global__ void ivf_bucket_fill(const int32_t* __restrict__ keys, int64_t cnt,
                                const int64_t* __restrict__ ptr, int32_t* __restrict__ cursor,
                                int32_t* __restrict__ ent) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t k = keys[i];
    if (k >= 0) ent[ptr[k] + atomicAdd(&cursor[k], 1)] = (int32_t)i;
  }
}

// ---------------------------------------------------------------- search ---
struct SearchP {
  const float* xn;
  int64_t dp;
  const int32_t* perm;      // keys in list order
  const int64_t* list_ptr;  // nlist + 1
  const int64_t* pair_ptr;  // nlist + 1
  const int32_t* pair_ent;  // q_local * nprobe + slot, grouped by list
  const int64_t* tile_ptr;  // nlist + 1: 64-pair tiles per list
  int32_t* counter;         // work-item counter (zeroed by the caller)
  int32_t nlist, nprobe;
  int64_t q0;
  int32_t K2;
  float floor_;             // -e: scores at or below cannot be positive
  float* part_s;            // (m * nprobe) x K2
  int32_t* part_i;
  uint32_t* qthr;           // per query of the chunk: best K2-th score of any
                            // finished (query, list) pair (order-preserving
                            // key, 0 = none): no later pair keeps a score
                            // below it, since the merged K2-th is >= it
};

// (s, id) ranks before (s2, id2): score desc, id asc
__device__ __forceinline__ bool before(float s, int id, float s2, int id2) {
  return s > s2 || (s == s2 && id < id2);
}

// Shared layout of ivf_search (floats unless noted).  Queries of the tile
// stay resident ([dq][QS], dq = dp when dp <= kResD) or are restaged per
// 32-dim chunk; key chunks [KC][QS]; per-tile candidate buffers (scores that
// beat the query's current K2-th entry) and the per-query top-K2 lists.
constexpr int QS = TQ + 4;  // row stride: float4-aligned, 4-way store conflicts at worst
constexpr int SKC = 16;     // dims per staged key chunk (3 CTAs per SM at d = 100)
constexpr int kResD = 256;

struct SearchSmem {
  size_t qs, ks, cbs, cbi, ts, ti, ints, total;
};

__host__ __device__ inline SearchSmem search_layout(int64_t dp, int K2) {
  SearchSmem L;
  const int64_t dq = dp <= kResD ? dp : 2 * SKC;
  size_t o = 0;
  L.qs = o; o += align_dev(sizeof(float) * (size_t)dq * QS);
  L.ks = o; o += align_dev(sizeof(float) * (size_t)2 * SKC * QS);
  L.cbs = o; o += align_dev(sizeof(float) * (size_t)TQ * TK);
  L.cbi = o; o += align_dev(sizeof(uint8_t) * (size_t)TQ * TK);
  L.ts = o; o += align_dev(sizeof(float) * (size_t)TQ * K2);
  L.ti = o; o += align_dev(sizeof(int32_t) * (size_t)TQ * K2);
  L.ints = o; o += align_dev(sizeof(int32_t) * (6 * TQ + TK));
  L.total = o;
  return L;
}

template <bool RES>
__global__ void __launch_bounds__(kT) ivf_search(SearchP p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const SearchSmem L = search_layout(p.dp, p.K2);
  float* qs = reinterpret_cast<float*>(smem_raw + L.qs);
  float* ks = reinterpret_cast<float*>(smem_raw + L.ks);
  float* cbs = reinterpret_cast<float*>(smem_raw + L.cbs);
  uint8_t* cbi = smem_raw + L.cbi;             // key slot within the tile
  float* ts = reinterpret_cast<float*>(smem_raw + L.ts);
  int32_t* ti = reinterpret_cast<int32_t*>(smem_raw + L.ti);
  int32_t* qrow = reinterpret_cast<int32_t*>(smem_raw + L.ints);
  int32_t* qent = qrow + TQ;
  int32_t* tn = qent + TQ;
  int32_t* ccnt = tn + TQ;
  float* thr = reinterpret_cast<float*>(ccnt + TQ);
  float* gt = thr + TQ;
  int32_t* kid = reinterpret_cast<int32_t*>(gt + TQ);
  __shared__ int s_work;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t total = p.tile_ptr[p.nlist];
  const int64_t dp = p.dp;
  for (;;) {
    if (tid == 0) s_work = atomicAdd(p.counter, 1);
    __syncthreads();
    const int64_t w = s_work;
    if (w >= total) break;
    int lo = 0, hi = p.nlist;  // largest c with tile_ptr[c] <= w
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (p.tile_ptr[mid] <= w) lo = mid; else hi = mid;
    }
    const int c = lo;
    const int64_t pb = p.pair_ptr[c] + (w - p.tile_ptr[c]) * TQ;
    const int nq = (int)lmin(TQ, p.pair_ptr[c + 1] - pb);
    const int64_t kb = p.list_ptr[c], ke = p.list_ptr[c + 1];
    if (tid < TQ) {
      const int32_t e = tid < nq ? p.pair_ent[pb + tid] : -1;
      qent[tid] = e;
      qrow[tid] = e >= 0 ? (int32_t)(p.q0 + e / p.nprobe) : -1;
      tn[tid] = 0;
      ccnt[tid] = 0;
      thr[tid] = p.floor_;
      gt[tid] = e >= 0 ? fmaxf(p.floor_, key_ord(p.qthr[e / p.nprobe])) : p.floor_;
    }
    __syncthreads();
    if (RES) {  // the tile's queries, transposed, once per work item
      for (int64_t idx = tid; idx < (int64_t)TQ * dp; idx += kT) {
        const int r = (int)(idx / dp);
        const int64_t cc = idx - (int64_t)r * dp;
        qs[cc * QS + r] = qrow[r] >= 0 ? p.xn[(int64_t)qrow[r] * dp + cc] : 0.0f;
      }
    }
    for (int64_t k0 = kb; k0 < ke; k0 += TK) {
      const int nk = (int)lmin(TK, ke - k0);
      if (tid < TK) kid[tid] = tid < nk ? p.perm[k0 + tid] : -1;
      float acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
      __syncthreads();
      // key chunks (and query chunks when not resident) are fetched into
      // registers one chunk ahead and stored to the other shared buffer
      constexpr int NF = TK * (SKC / 4) / kT;  // float4 per thread per chunk
      float4 pk[NF], pq[NF];
      auto fetch = [&](int64_t d0) {
        const int kc = (int)lmin(SKC, dp - d0);
#pragma unroll
        for (int u = 0; u < NF; ++u) {
          const int f = tid + u * kT;
          const int r = f / (SKC / 4), c4 = (f % (SKC / 4)) * 4;
          pk[u] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (kid[r] >= 0 && c4 < kc)
            pk[u] = *reinterpret_cast<const float4*>(p.xn + (int64_t)kid[r] * dp + d0 + c4);
          if (!RES) {
            pq[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (qrow[r] >= 0 && c4 < kc)
              pq[u] = *reinterpret_cast<const float4*>(p.xn + (int64_t)qrow[r] * dp + d0 + c4);
          }
        }
      };
      auto stash = [&](int buf) {
        float* kb_ = ks + buf * SKC * QS;
        float* qb_ = qs + buf * SKC * QS;
#pragma unroll
        for (int u = 0; u < NF; ++u) {
          const int f = tid + u * kT;
          const int r = f / (SKC / 4), c4 = (f % (SKC / 4)) * 4;
          kb_[(c4 + 0) * QS + r] = pk[u].x;
          kb_[(c4 + 1) * QS + r] = pk[u].y;
          kb_[(c4 + 2) * QS + r] = pk[u].z;
          kb_[(c4 + 3) * QS + r] = pk[u].w;
          if (!RES) {
            qb_[(c4 + 0) * QS + r] = pq[u].x;
            qb_[(c4 + 1) * QS + r] = pq[u].y;
            qb_[(c4 + 2) * QS + r] = pq[u].z;
            qb_[(c4 + 3) * QS + r] = pq[u].w;
          }
        }
      };
      fetch(0);
      stash(0);
      __syncthreads();
      int buf = 0;
      for (int64_t d0 = 0; d0 < dp; d0 += SKC) {
        const int kc = (int)lmin(SKC, dp - d0);
        const bool more = d0 + SKC < dp;
        if (more) fetch(d0 + SKC);
        const float* qb = RES ? qs + d0 * QS : qs + buf * SKC * QS;
        const float* kb_ = ks + buf * SKC * QS;
#pragma unroll 4
        for (int kk = 0; kk < kc; ++kk) {
          const float4 a = *reinterpret_cast<const float4*>(qb + kk * QS + ty * 4);
          const float4 b = *reinterpret_cast<const float4*>(kb_ + kk * QS + tx * 4);
          const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        if (more) stash(buf ^ 1);
        __syncthreads();
        buf ^= 1;
      }
      // filter in registers against each query's current K2-th entry
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int q = ty * 4 + i;
        if (q >= nq) continue;
        const bool full = tn[q] == p.K2;
        const float ts_ = thr[q], g_ = gt[q];
        const int ti_ = full ? ti[q * p.K2 + p.K2 - 1] : 0;
        const int me = qrow[q];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int id = kid[tx * 4 + j];
          const float sv = acc[i][j];
          if (id < 0 || id == me) continue;
          if (sv > g_ && (full ? before(sv, id, ts_, ti_) : sv > ts_)) {
            const int slot = atomicAdd(&ccnt[q], 1);
            cbs[q * TK + slot] = sv;
            cbi[q * TK + slot] = (uint8_t)(tx * 4 + j);
          }
        }
      }
      __syncthreads();
      if (p.K2 <= 32) {
        // warp-cooperative insertion: lane t holds entry t of the list
        const int lane = tid & 31, wp = tid >> 5;
        for (int q = wp; q < nq; q += kT / 32) {
          const int nb = ccnt[q];
          if (nb == 0) continue;
          int cnt = tn[q];
          float es = lane < cnt ? ts[q * p.K2 + lane] : -FLT_MAX;
          int ei = lane < cnt ? ti[q * p.K2 + lane] : 0x7fffffff;
          for (int u = 0; u < nb; ++u) {
            const float sv = cbs[q * TK + u];
            const int id = kid[cbi[q * TK + u]];
            const float ls_ = __shfl_sync(0xffffffffu, es, p.K2 - 1);
            const int li_ = __shfl_sync(0xffffffffu, ei, p.K2 - 1);
            if (cnt == p.K2 && !before(sv, id, ls_, li_)) continue;
            const int pos = __popc(__ballot_sync(0xffffffffu, lane < cnt && before(es, ei, sv, id)));
            const float us = __shfl_up_sync(0xffffffffu, es, 1);
            const int ui = __shfl_up_sync(0xffffffffu, ei, 1);
            if (lane > pos) { es = us; ei = ui; }
            if (lane == pos) { es = sv; ei = id; }
            cnt = min(cnt + 1, p.K2);
          }
          if (lane < cnt) {
            ts[q * p.K2 + lane] = es;
            ti[q * p.K2 + lane] = ei;
          }
          if (lane == 0) {
            tn[q] = cnt;
            ccnt[q] = 0;
          }
          const float last = __shfl_sync(0xffffffffu, es, p.K2 - 1);
          if (lane == 0) thr[q] = cnt == p.K2 ? last : p.floor_;
        }
      } else if (tid < nq) {
        const int q = tid;
        float* ls = ts + q * p.K2;
        int32_t* li = ti + q * p.K2;
        int cnt = tn[q];
        const int nb = ccnt[q];
        for (int u = 0; u < nb; ++u) {
          const float sv = cbs[q * TK + u];
          const int id = kid[cbi[q * TK + u]];
          if (cnt == p.K2 && !before(sv, id, ls[cnt - 1], li[cnt - 1])) continue;
          int pos = cnt < p.K2 ? cnt++ : p.K2 - 1;
          while (pos > 0 && before(sv, id, ls[pos - 1], li[pos - 1])) {
            ls[pos] = ls[pos - 1];
            li[pos] = li[pos - 1];
            --pos;
          }
          ls[pos] = sv;
          li[pos] = id;
        }
        tn[q] = cnt;
        ccnt[q] = 0;
        thr[q] = cnt == p.K2 ? ls[p.K2 - 1] : p.floor_;
      }
      __syncthreads();
    }
    if (tid < nq) {
      const int r = tid;
      const int64_t base = (int64_t)qent[r] * p.K2;
      const int cnt = tn[r];
      for (int t = 0; t < p.K2; ++t) {
        p.part_s[base + t] = t < cnt ? ts[r * p.K2 + t] : -FLT_MAX;
        p.part_i[base + t] = t < cnt ? ti[r * p.K2 + t] : -1;
      }
      if (cnt == p.K2) atomicMax(p.qthr + qent[r] / p.nprobe, ord_key(ts[r * p.K2 + p.K2 - 1]));
    }
    __syncthreads();
  }
}

// ------------------------------------------------ tensor-core scan (fp16) ---
// The same (list, 64-pair) tiles scored on the tensor cores: h = fp16(xn)
// (entries below 2^-14 flushed), one mma.sync.m16n8k16 product per 16 dims
// with f32 accumulation.  |h_q.h_j - xn_q.xn_j| <= l_q + l_j + l_q l_j + acc
// with l the per-row residual ||xn - h|| (ivf_half_prep), so a row's
// floor and the merge's certificate use e_q = l_q + l_max + l_q l_max + e.
__global__ void ivf_half_prep(const float* __restrict__ xn, int64_t n, int64_t dp, __half* __restrict__ h,
                              int64_t dh, float* __restrict__ lres, unsigned* __restrict__ lmax_bits) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < n;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double s2 = 0.0;
    for (int64_t c = lane; c < dh; c += 32) {
      const float v = c < dp ? xn[r * dp + c] : 0.f;
      __half hv = __float2half_rn(v);
      if (fabsf(v) < 0x1p-14f) hv = __float2half_rn(0.f);
      h[r * dh + c] = hv;
      const double d = (double)v - (double)__half2float(hv);
      s2 = fma(d, d, s2);
    }
    s2 = warp_sum(s2);
    if (lane == 0) {
      const float l = (float)(sqrt(s2) * (1.0 + 1e-6)) + 1e-30f;   // rounded up
      lres[r] = l;
      atomicMax(lmax_bits, __float_as_uint(l));                    // l >= 0: bit order = value order
    }
  }
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

struct SearchTcP {
  SearchP s;
  const __half* h;   // n x dh
  int64_t dh;
  const float* lres;
  const unsigned* lmax_bits;
  float acc_err;
};

constexpr int kMaxDh = 256;

__host__ __device__ inline size_t search_tc_smem(int64_t dh, int K2) {
  const size_t hs = (size_t)(dh + 8);                      // halves per staged row
  return align_dev(2 * hs * TQ) + 3 * align_dev(2 * hs * TK) + align_dev(4 * (size_t)TQ * TK) +
         align_dev((size_t)TQ * TK) + align_dev(4 * (size_t)TQ * K2) + align_dev(4 * (size_t)TQ * K2) +
         align_dev(4 * (7 * (size_t)TQ + TK));
}

constexpr int kTcStages = 3;      // key tiles in flight

// B fragments of two 8-key column tiles (keys n0..n0+15 of a row-major
// key tile, k-step k) with one ldmatrix.x4: {b0, b1} of tile n0, then n0 + 8
__device__ __forceinline__ void ldsm_b2(const __half* kt, int hs, int n0, int k, int lane, uint32_t (&b)[4]) {
  const __half* ptr = kt + (size_t)(n0 + ((lane >> 4) << 3) + (lane & 7)) * hs + k + ((lane >> 3) & 1) * 8;
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3])
               : "r"((uint32_t)__cvta_generic_to_shared(ptr)));
}

// KS > 0: dh == 16 KS at most, the warp's query fragments stay in registers
// for all key tiles of a pair tile; KS == 0: re-read from shared per k-step
template <int KS>
__global__ void __launch_bounds__(kT) ivf_search_tc(SearchTcP P) {
  const SearchP& p = P.s;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int hs = (int)P.dh + 8;
  unsigned char* o = smem_raw;
  __half* qh = reinterpret_cast<__half*>(o); o += align_dev(2 * (size_t)hs * TQ);
  __half* kh[kTcStages];
  for (int st = 0; st < kTcStages; ++st) {
    kh[st] = reinterpret_cast<__half*>(o);
    o += align_dev(2 * (size_t)hs * TK);
  }
  float* cbs = reinterpret_cast<float*>(o); o += align_dev(4 * (size_t)TQ * TK);
  uint8_t* cbi = o; o += align_dev((size_t)TQ * TK);
  float* ts = reinterpret_cast<float*>(o); o += align_dev(4 * (size_t)TQ * p.K2);
  int32_t* ti = reinterpret_cast<int32_t*>(o); o += align_dev(4 * (size_t)TQ * p.K2);
  int32_t* qrow = reinterpret_cast<int32_t*>(o);
  int32_t* qent = qrow + TQ;
  int32_t* tn = qent + TQ;
  int32_t* ccnt = tn + TQ;
  float* thr = reinterpret_cast<float*>(ccnt + TQ);
  float* gt = thr + TQ;
  float* eq = gt + TQ;
  __shared__ int s_work, s_nql;
  __shared__ int32_t kids[kTcStages][TK];                 // key ids of each staged tile
  __shared__ int32_t qlist[TQ];                           // queries with candidates in the tile
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int wr = (warp & 3) * 16, wc = (warp >> 2) * 32;   // warp tile: 16 queries x 32 keys
  const int64_t total = p.tile_ptr[p.nlist];
  const int nch = (int)(P.dh / 8);                          // 16-byte chunks per row
  const float lmax = __uint_as_float(*P.lmax_bits);
  uint32_t areg[KS > 0 ? KS : 1][4];
  // stage key tile [k0, k0 + TK) of the list (ids read from perm by the
  // issuing threads; thread r < TK records id r for the filter)
  auto stage_keys = [&](int64_t k0, int64_t ke, int b) {
    static_assert(kT == 4 * TK, "four threads per staged key row");
    const int r = tid >> 2;
    const int32_t id = k0 + r < ke ? p.perm[k0 + r] : -1;
    if ((tid & 3) == 0) kids[b][r] = id;
    __half* dst = kh[b] + (size_t)r * hs;
    const __half* src = P.h + (int64_t)(id >= 0 ? id : 0) * P.dh;
    for (int ch = tid & 3; ch < nch; ch += 4) {
      if (id >= 0) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst + ch * 8)),
                     "l"(src + ch * 8)
                     : "memory");
      } else {
        *reinterpret_cast<uint4*>(dst + ch * 8) = make_uint4(0u, 0u, 0u, 0u);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (tid == 0) s_nql = 0;
  for (;;) {
    if (tid == 0) s_work = atomicAdd(p.counter, 1);
    __syncthreads();
    const int64_t w = s_work;
    if (w >= total) break;
    int lo = 0, hi = p.nlist;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (p.tile_ptr[mid] <= w) lo = mid; else hi = mid;
    }
    const int c = lo;
    const int64_t pb = p.pair_ptr[c] + (w - p.tile_ptr[c]) * TQ;
    const int nq = (int)lmin(TQ, p.pair_ptr[c + 1] - pb);
    const int64_t kb = p.list_ptr[c], ke = p.list_ptr[c + 1];
    const int ntile = (int)ceil_div(ke - kb, TK);
    // the first stages' keys start loading before the query tile is set up
    for (int st = 0; st < kTcStages - 1; ++st) {
      if (st < ntile) stage_keys(kb + (int64_t)st * TK, ke, st);
      else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    if (tid < TQ) {
      const int32_t e = tid < nq ? p.pair_ent[pb + tid] : -1;
      qent[tid] = e;
      const int32_t qr = e >= 0 ? (int32_t)(p.q0 + e / p.nprobe) : -1;
      qrow[tid] = qr;
      tn[tid] = 0;
      ccnt[tid] = 0;
      const float lq = qr >= 0 ? P.lres[qr] : 0.f;
      const float e_q = lq + lmax + lq * lmax + P.acc_err;
      eq[tid] = e_q;
      thr[tid] = -e_q;
      gt[tid] = e >= 0 ? fmaxf(-e_q, key_ord(p.qthr[e / p.nprobe])) : -e_q;
    }
    __syncthreads();
    for (int e = tid; e < TQ * nch; e += kT) {             // the tile's queries (fp16)
      const int r = e / nch, ch = e - r * nch;
      const int32_t qr = qrow[r];
      *reinterpret_cast<uint4*>(qh + (size_t)r * hs + ch * 8) =
          qr >= 0 ? *reinterpret_cast<const uint4*>(P.h + (int64_t)qr * P.dh + ch * 8) : make_uint4(0u, 0u, 0u, 0u);
    }
    for (int t = 0; t < ntile; ++t) {
      const int b = t % kTcStages;
      const int64_t k0 = kb + (int64_t)t * TK;
      const int nk = (int)lmin(TK, ke - k0);
      if (t + kTcStages - 1 < ntile) stage_keys(kb + (int64_t)(t + kTcStages - 1) * TK, ke, (t + kTcStages - 1) % kTcStages);
      else asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group %0;" ::"n"(kTcStages - 1) : "memory");
      __syncthreads();
      const int32_t* kid = kids[b];
      float acc[4][4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[nt][u] = 0.f;
      const __half* kb_ = kh[b];
      if constexpr (KS > 0) {
        if (t == 0) {                                          // qh complete (barrier above)
#pragma unroll
          for (int s = 0; s < KS; ++s) {
            if (16 * s >= (int)P.dh) break;
            const __half* qa = qh + (size_t)(wr + g) * hs + 16 * s + 2 * t4;
            areg[s][0] = *reinterpret_cast<const uint32_t*>(qa);
            areg[s][1] = *reinterpret_cast<const uint32_t*>(qa + 8 * hs);
            areg[s][2] = *reinterpret_cast<const uint32_t*>(qa + 8);
            areg[s][3] = *reinterpret_cast<const uint32_t*>(qa + 8 * hs + 8);
          }
        }
#pragma unroll
        for (int s = 0; s < KS; ++s) {
          if (16 * s < (int)P.dh) {
            uint32_t bf[4];
            ldsm_b2(kb_, hs, wc, 16 * s, lane, bf);
            mma16816(acc[0], areg[s], bf[0], bf[1]);
            mma16816(acc[1], areg[s], bf[2], bf[3]);
            ldsm_b2(kb_, hs, wc + 16, 16 * s, lane, bf);
            mma16816(acc[2], areg[s], bf[0], bf[1]);
            mma16816(acc[3], areg[s], bf[2], bf[3]);
          }
        }
      } else {
        for (int k = 0; k < (int)P.dh; k += 16) {
          uint32_t a[4];
          const __half* qa = qh + (size_t)(wr + g) * hs + k + 2 * t4;
          a[0] = *reinterpret_cast<const uint32_t*>(qa);
          a[1] = *reinterpret_cast<const uint32_t*>(qa + 8 * hs);
          a[2] = *reinterpret_cast<const uint32_t*>(qa + 8);
          a[3] = *reinterpret_cast<const uint32_t*>(qa + 8 * hs + 8);
          uint32_t bf[4];
          ldsm_b2(kb_, hs, wc, k, lane, bf);
          mma16816(acc[0], a, bf[0], bf[1]);
          mma16816(acc[1], a, bf[2], bf[3]);
          ldsm_b2(kb_, hs, wc + 16, k, lane, bf);
          mma16816(acc[2], a, bf[0], bf[1]);
          mma16816(acc[3], a, bf[2], bf[3]);
        }
      }
      // filter: lane holds rows wr+g, wr+g+8 and keys wc + 8 nt + 2 t4 + {0,1}
#pragma unroll
      for (int hrow = 0; hrow < 2; ++hrow) {
        const int q = wr + g + 8 * hrow;
        if (q >= nq) continue;
        const bool full = tn[q] == p.K2;
        const float ts_ = thr[q], g_ = gt[q];
        const int ti_ = full ? ti[q * p.K2 + p.K2 - 1] : 0;
        const int me = qrow[q];
        const float lo2 = fmaxf(g_, ts_);
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const float sv = acc[nt][2 * hrow + u];
            if (!(sv > g_) || sv < lo2 || (!full && !(sv > ts_))) continue;
            const int slot = wc + nt * 8 + 2 * t4 + u;
            const int id = kid[slot];
            if (slot >= nk || id < 0 || id == me) continue;
            if (full && !before(sv, id, ts_, ti_)) continue;
            const int pos = atomicAdd(&ccnt[q], 1);
            if (pos == 0) qlist[atomicAdd(&s_nql, 1)] = q;
            cbs[q * TK + pos] = sv;
            cbi[q * TK + pos] = (uint8_t)slot;
          }
      }
      __syncthreads();
      // no candidates in the tile: nothing to insert, and nothing read after
      // this barrier needs protecting before the next tile's top barrier
      const int nql = s_nql;
      if (nql == 0) continue;
      // warp-cooperative insertion (K2 <= 32: lane t holds entry t)
      for (int iq = warp; iq < nql; iq += kT / 32) {
        const int q = qlist[iq];
        const int nb = ccnt[q];
        if (nb == 0) continue;
        int cnt = tn[q];
        float es = lane < cnt ? ts[q * p.K2 + lane] : -FLT_MAX;
        int ei = lane < cnt ? ti[q * p.K2 + lane] : 0x7fffffff;
        for (int u = 0; u < nb; ++u) {
          const float sv = cbs[q * TK + u];
          const int id = kid[cbi[q * TK + u]];
          const float ls_ = __shfl_sync(0xffffffffu, es, p.K2 - 1);
          const int li_ = __shfl_sync(0xffffffffu, ei, p.K2 - 1);
          if (cnt == p.K2 && !before(sv, id, ls_, li_)) continue;
          const int pos = __popc(__ballot_sync(0xffffffffu, lane < cnt && before(es, ei, sv, id)));
          const float us = __shfl_up_sync(0xffffffffu, es, 1);
          const int ui = __shfl_up_sync(0xffffffffu, ei, 1);
          if (lane > pos) { es = us; ei = ui; }
          if (lane == pos) { es = sv; ei = id; }
          cnt = min(cnt + 1, p.K2);
        }
        if (lane < cnt) {
          ts[q * p.K2 + lane] = es;
          ti[q * p.K2 + lane] = ei;
        }
        const float last = __shfl_sync(0xffffffffu, es, p.K2 - 1);
        if (lane == 0) {
          tn[q] = cnt;
          ccnt[q] = 0;
          thr[q] = cnt == p.K2 ? last : -eq[q];
        }
      }
      __syncthreads();
      if (tid == 0) s_nql = 0;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (tid < nq) {
      const int r = tid;
      const int64_t base = (int64_t)qent[r] * p.K2;
      const int cnt = tn[r];
      for (int t = 0; t < p.K2; ++t) {
        p.part_s[base + t] = t < cnt ? ts[r * p.K2 + t] : -FLT_MAX;
        p.part_i[base + t] = t < cnt ? ti[r * p.K2 + t] : -1;
      }
      if (cnt == p.K2) atomicMax(p.qthr + qent[r] / p.nprobe, ord_key(ts[r * p.K2 + p.K2 - 1]));
    }
    __syncthreads();
  }
}

// ----------------------------------------------------------------- merge ---
struct MergeP {
  const float* xn;
  int64_t dp;
  int64_t q0, m;
  int32_t nprobe, K2, K;
  const float* part_s;
  const int32_t* part_i;
  float e;
  int32_t* ids;      // m x K (rows of this chunk)
  double* scores;
  int32_t* flagged;  // global row ids of uncertified rows
  int32_t* nflag;
  const float* lres;  // fp16 scan: per-row residual norms (e_q = l_q + l_max + l_q l_max + e)
  const unsigned* lmax_bits;
};

constexpr int kMergeWarps = 8;

__global__ void __launch_bounds__(32 * kMergeWarps) ivf_merge(MergeP p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* ws = reinterpret_cast<float*>(smem_raw) + (size_t)w * p.K2;
  int32_t* wi = reinterpret_cast<int32_t*>(reinterpret_cast<float*>(smem_raw) + kMergeWarps * p.K2) +
                (size_t)w * p.K2;
  double* wd = reinterpret_cast<double*>(smem_raw + align_dev((size_t)kMergeWarps * p.K2 * 8)) +
               (size_t)w * p.K2;
  for (int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; q < p.m;
       q += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t nc = (int64_t)p.nprobe * p.K2;
    const float* cs = p.part_s + q * nc;
    const int32_t* ci = p.part_i + q * nc;
    int cnt = 0;
    for (int64_t b = 0; b < nc; b += 32) {
      const int64_t j = b + lane;
      const int id = j < nc ? ci[j] : -1;
      const float s = j < nc ? cs[j] : -FLT_MAX;
      __syncwarp();
      const bool full = cnt == p.K2;
      const float ts_ = full ? ws[p.K2 - 1] : 0.0f;
      const int ti_ = full ? wi[p.K2 - 1] : 0;
      unsigned pass = __ballot_sync(0xffffffffu, id >= 0 && (!full || before(s, id, ts_, ti_)));
      while (pass) {
        const int src = __ffs(pass) - 1;
        pass &= pass - 1;
        const float s2 = __shfl_sync(0xffffffffu, s, src);
        const int id2 = __shfl_sync(0xffffffffu, id, src);
        if (lane == 0 && (cnt < p.K2 || before(s2, id2, ws[cnt - 1], wi[cnt - 1]))) {
          int pos = cnt < p.K2 ? cnt++ : p.K2 - 1;
          while (pos > 0 && before(s2, id2, ws[pos - 1], wi[pos - 1])) {
            ws[pos] = ws[pos - 1];
            wi[pos] = wi[pos - 1];
            --pos;
          }
          ws[pos] = s2;
          wi[pos] = id2;
        }
        cnt = __shfl_sync(0xffffffffu, cnt, 0);
      }
    }
    __syncwarp();
    // exact re-rank: f64 sums of the (exact) f32 x f32 products
    const int64_t gq = p.q0 + q;
    const float* xq = p.xn + gq * p.dp;
    for (int t = 0; t < cnt; ++t) {
      const float* xk = p.xn + (int64_t)wi[t] * p.dp;
      double a = 0.0;
      for (int64_t c = lane; c < p.dp; c += 32) a = fma((double)xq[c], (double)xk[c], a);
      a = warp_sum(a);
      if (lane == 0) wd[t] = a;
    }
    __syncwarp();
    if (lane == 0) {
      // sort the kept candidates by (f64 desc, id asc)
      for (int t = 1; t < cnt; ++t) {
        const double v = wd[t];
        const int id = wi[t];
        int u = t;
        while (u > 0 && (wd[u - 1] < v || (wd[u - 1] == v && wi[u - 1] > id))) {
          wd[u] = wd[u - 1];
          wi[u] = wi[u - 1];
          --u;
        }
        wd[u] = v;
        wi[u] = id;
      }
      // certificate: everything not kept scored (f32) <= the K2-th kept
      // f32 score, so its exact value is <= that + e
      const float last = cnt == p.K2 ? ws[p.K2 - 1] : -FLT_MAX;
      const double lmax = p.lres ? (double)__uint_as_float(*p.lmax_bits) : 0.0;
      const double eq = p.lres ? (double)p.lres[gq] + lmax + (double)p.lres[gq] * lmax + p.e
                               : (double)p.e;
      const double bound = (double)last + eq;
      int npos = 0, nabove = 0;
      for (int t = 0; t < cnt; ++t) {
        if (wd[t] > 0.0) ++npos;
        if (wd[t] > bound && wd[t] > 0.0) ++nabove;
      }
      const bool ok = cnt < p.K2 || bound <= 0.0 || nabove >= p.K;
      if (!ok) p.flagged[atomicAdd(p.nflag, 1)] = (int32_t)gq;
      const int take = min(npos, p.K);
      for (int t = 0; t < p.K; ++t) {
        p.ids[q * p.K + t] = t < take ? wi[t] : -1;
        p.scores[q * p.K + t] = t < take ? (double)fminf((float)wd[t], 1.0f) : 0.0;
      }
    }
    __syncwarp();
  }
}

// ivf_merge for K2 <= 32: the kept list spread over the warp (lane t holds
// entry t), inserts by one ballot + shift, the f64 re-rank order by ranks
// from shuffles -- the same lists, certificate and outputs as ivf_merge
// without its lane-0 serial inserts and sort
__global__ void __launch_bounds__(32 * kMergeWarps) ivf_merge_warp(MergeP p) {
  const int lane = threadIdx.x & 31;
  for (int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; q < p.m;
       q += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t nc = (int64_t)p.nprobe * p.K2;
    const float* cs = p.part_s + q * nc;
    const int32_t* ci = p.part_i + q * nc;
    float ls = -FLT_MAX;         // lane t < cnt: entry t of the kept list (f32 score, id)
    int li = -1;
    int cnt = 0;
    for (int64_t b = 0; b < nc; b += 32) {
      const int64_t j = b + lane;
      const int id = j < nc ? ci[j] : -1;
      const float s = j < nc ? cs[j] : -FLT_MAX;
      const bool full = cnt == p.K2;
      const float ts_ = __shfl_sync(0xffffffffu, ls, p.K2 - 1);
      const int ti_ = __shfl_sync(0xffffffffu, li, p.K2 - 1);
      unsigned pass = __ballot_sync(0xffffffffu, id >= 0 && (!full || before(s, id, ts_, ti_)));
      while (pass) {
        const int src = __ffs(pass) - 1;
        pass &= pass - 1;
        const float s2 = __shfl_sync(0xffffffffu, s, src);
        const int id2 = __shfl_sync(0xffffffffu, id, src);
        if (cnt == p.K2) {
          const float lsl = __shfl_sync(0xffffffffu, ls, p.K2 - 1);
          const int lil = __shfl_sync(0xffffffffu, li, p.K2 - 1);
          if (!before(s2, id2, lsl, lil)) continue;                 // warp-uniform
        }
        const int pos = __popc(__ballot_sync(0xffffffffu, lane < cnt && before(ls, li, s2, id2)));
        const float us = __shfl_up_sync(0xffffffffu, ls, 1);
        const int ui = __shfl_up_sync(0xffffffffu, li, 1);
        if (lane > pos && lane < p.K2) { ls = us; li = ui; }
        if (lane == pos) { ls = s2; li = id2; }
        cnt = min(cnt + 1, p.K2);
      }
    }
    // exact re-rank: f64 sums of the (exact) f32 x f32 products
    const int64_t gq = p.q0 + q;
    const float* xq = p.xn + gq * p.dp;
    double wd = 0.0;
    for (int t = 0; t < cnt; ++t) {
      const float* xk = p.xn + (int64_t)__shfl_sync(0xffffffffu, li, t) * p.dp;
      double a = 0.0;
      for (int64_t c = lane; c < p.dp; c += 32) a = fma((double)xq[c], (double)xk[c], a);
      a = warp_sum(a);
      if (lane == t) wd = a;
    }
    // certificate: everything not kept scored (f32) <= the K2-th kept
    // f32 score, so its exact value is <= that + e
    const float last = cnt == p.K2 ? __shfl_sync(0xffffffffu, ls, p.K2 - 1) : -FLT_MAX;
    const double lmax = p.lres ? (double)__uint_as_float(*p.lmax_bits) : 0.0;
    const double eq = p.lres ? (double)p.lres[gq] + lmax + (double)p.lres[gq] * lmax + p.e
                             : (double)p.e;
    const double bound = (double)last + eq;
    const bool mine = lane < cnt;
    const int npos = __popc(__ballot_sync(0xffffffffu, mine && wd > 0.0));
    const int nabove = __popc(__ballot_sync(0xffffffffu, mine && wd > bound && wd > 0.0));
    const bool ok = cnt < p.K2 || bound <= 0.0 || nabove >= p.K;
    if (lane == 0 && !ok) p.flagged[atomicAdd(p.nflag, 1)] = (int32_t)gq;
    // rank in (f64 desc, id asc) among the kept entries
    int rank = 0;
    for (int u = 0; u < cnt; ++u) {
      const double du = __shfl_sync(0xffffffffu, wd, u);
      const int iu = __shfl_sync(0xffffffffu, li, u);
      rank += (du > wd || (du == wd && iu < li)) ? 1 : 0;
    }
    const int take = min(npos, p.K);
    if (mine && rank < take) {
      p.ids[q * p.K + rank] = li;
      p.scores[q * p.K + rank] = (double)fminf((float)wd, 1.0f);
    }
    for (int t = take + lane; t < p.K; t += 32) {
      p.ids[q * p.K + t] = -1;
      p.scores[q * p.K + t] = 0.0;
    }
  }
}

// ------------------------------------------------------------ rows exact ---
// R query rows per CTA share one candidate stream (all keys, probes ==
// nullptr) or R = 1 with the row's own probe lists.  Every candidate scored
// with f64 accumulation; per row a top-K list (score desc, id asc) of the
// positive scores, self excluded.
constexpr int kRowsR = 16;

struct RowsP {
  const float* xn;
  int64_t dp, n;
  const int32_t* rows;  // global row ids
  int64_t nrows;
  const int32_t* probes;  // m x nprobe (row - q0), or nullptr: all keys
  int32_t nprobe;
  int64_t q0;
  const int32_t* perm;
  const int64_t* list_ptr;
  int32_t K;
  int32_t* ids;
  double* scores;
  int compact;  // output row b (audit) instead of rows[b] - q0
  int R;        // query rows per CTA (1 with probes)
  int nsplit;   // all-keys mode: key segments (blockIdx.y); > 1 writes exact partial lists
  double* seg_sc;   // nrows x nsplit x K partial scores (f64), ids below
  int32_t* seg_id;
};

__global__ void __launch_bounds__(kT) ivf_rows_exact(RowsP p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int R = p.R;
  double* ls = reinterpret_cast<double*>(smem_raw);                            // R x K
  int32_t* li = reinterpret_cast<int32_t*>(ls + (size_t)R * p.K);              // R x K
  // query rows held as f64 (exact widening, done once instead of per key)
  double* xq = reinterpret_cast<double*>(smem_raw + align_dev((size_t)R * p.K * 12));  // R x dp
  double* bs = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(xq) +
                                         align_dev((size_t)R * p.dp * 8));     // R x kT
  int32_t* bi = reinterpret_cast<int32_t*>(bs + (size_t)R * kT);
  __shared__ int bcnt[kRowsR], lcnt[kRowsR], qid[kRowsR];
  const int tid = threadIdx.x;
  const int64_t b0 = (int64_t)blockIdx.x * R;
  const int nr = (int)lmin(R, p.nrows - b0);
  if (nr <= 0) return;
  if (tid < R) {
    qid[tid] = tid < nr ? p.rows[b0 + tid] : -1;
    lcnt[tid] = 0;
  }
  __syncthreads();
  for (int64_t i = tid; i < (int64_t)R * p.dp; i += kT) {
    const int r = (int)(i / p.dp);
    xq[i] = qid[r] >= 0 ? (double)p.xn[(int64_t)qid[r] * p.dp + (i % p.dp)] : 0.0;
  }
  // candidate ranges: all keys, or the row's probe lists (through perm)
  const int nseg = p.probes ? p.nprobe : 1;
  for (int sg = 0; sg < nseg; ++sg) {
    int64_t cb = 0, ce = p.n;
    if (!p.probes && p.nsplit > 1) {          // this CTA's key segment
      const int64_t len = ceil_div(p.n, p.nsplit);
      cb = lmin(p.n, (int64_t)blockIdx.y * len);
      ce = lmin(p.n, cb + len);
    }
    if (p.probes) {
      const int c = p.probes[(int64_t)(qid[0] - p.q0) * p.nprobe + sg];
      cb = p.list_ptr[c];
      ce = p.list_ptr[c + 1];
    }
    for (int64_t j0 = cb; j0 < ce; j0 += kT) {
      if (tid < R) bcnt[tid] = 0;
      __syncthreads();
      const int64_t j = j0 + tid;
      if (j < ce) {
        const int id = p.probes ? p.perm[j] : (int)j;
        const float* xk = p.xn + (int64_t)id * p.dp;
        double a[kRowsR];
#pragma unroll
        for (int r = 0; r < kRowsR; ++r) a[r] = 0.0;
        for (int64_t c = 0; c < p.dp; c += 4) {
          const float4 v = *reinterpret_cast<const float4*>(xk + c);
          const double v0 = v.x, v1 = v.y, v2 = v.z, v3 = v.w;
#pragma unroll
          for (int r = 0; r < kRowsR; ++r) {
            if (r < R) {
              const double2 x01 = *reinterpret_cast<const double2*>(xq + (size_t)r * p.dp + c);
              const double2 x23 = *reinterpret_cast<const double2*>(xq + (size_t)r * p.dp + c + 2);
              a[r] = fma(x01.x, v0, a[r]);
              a[r] = fma(x01.y, v1, a[r]);
              a[r] = fma(x23.x, v2, a[r]);
              a[r] = fma(x23.y, v3, a[r]);
            }
          }
        }
#pragma unroll
        for (int r = 0; r < kRowsR; ++r) {
          if (r >= nr || id == qid[r] || !(a[r] > 0.0)) continue;
          const int cntr = lcnt[r];
          if (cntr == p.K) {
            const double lv = ls[(size_t)r * p.K + p.K - 1];
            const int lid = li[(size_t)r * p.K + p.K - 1];
            if (!(a[r] > lv || (a[r] == lv && id < lid))) continue;
          }
          const int slot = atomicAdd(&bcnt[r], 1);
          bs[(size_t)r * kT + slot] = a[r];
          bi[(size_t)r * kT + slot] = id;
        }
      }
      __syncthreads();
      if (tid < nr) {
        const int r = tid;
        double* L = ls + (size_t)r * p.K;
        int32_t* I = li + (size_t)r * p.K;
        int cnt = lcnt[r];
        for (int u = 0; u < bcnt[r]; ++u) {
          const double s = bs[(size_t)r * kT + u];
          const int id = bi[(size_t)r * kT + u];
          if (cnt == p.K && !(s > L[cnt - 1] || (s == L[cnt - 1] && id < I[cnt - 1]))) continue;
          int pos = cnt < p.K ? cnt++ : p.K - 1;
          while (pos > 0 && (s > L[pos - 1] || (s == L[pos - 1] && id < I[pos - 1]))) {
            L[pos] = L[pos - 1];
            I[pos] = I[pos - 1];
            --pos;
          }
          L[pos] = s;
          I[pos] = id;
        }
        lcnt[r] = cnt;
      }
      __syncthreads();
    }
  }
  if (tid < nr) {
    const int r = tid;
    if (!p.probes && p.nsplit > 1) {          // exact partial list of this key segment
      const int64_t base = ((b0 + r) * p.nsplit + blockIdx.y) * p.K;
      for (int t = 0; t < p.K; ++t) {
        const bool v = t < lcnt[r];
        p.seg_id[base + t] = v ? li[(size_t)r * p.K + t] : -1;
        p.seg_sc[base + t] = v ? ls[(size_t)r * p.K + t] : -INFINITY;
      }
      return;
    }
    const int64_t orow = p.compact ? b0 + r : (int64_t)qid[r] - p.q0;
    for (int t = 0; t < p.K; ++t) {
      const bool v = t < lcnt[r];
      p.ids[orow * p.K + t] = v ? li[(size_t)r * p.K + t] : -1;
      p.scores[orow * p.K + t] = v ? (double)fminf((float)ls[(size_t)r * p.K + t], 1.0f) : 0.0;
    }
  }
}

// merge of the key-segment partial lists (exact f64 scores): top-K by
// (score desc, id asc), one thread per row (compact output)
__global__ void ivf_rows_seg_merge(const double* __restrict__ seg_sc, const int32_t* __restrict__ seg_id,
                                   int64_t nrows, int nsplit, int K, int32_t* __restrict__ ids,
                                   double* __restrict__ scores) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  int head[64];
  for (int s = 0; s < nsplit; ++s) head[s] = 0;
  for (int t = 0; t < K; ++t) {
    int bs = -1;
    double bv = 0.0;
    int bi = 0x7fffffff;
    for (int s = 0; s < nsplit; ++s) {
      if (head[s] >= K) continue;
      const int64_t e = (r * nsplit + s) * K + head[s];
      const int id = seg_id[e];
      if (id < 0) continue;
      const double v = seg_sc[e];
      if (bs < 0 || v > bv || (v == bv && id < bi)) { bs = s; bv = v; bi = id; }
    }
    ids[r * K + t] = bs < 0 ? -1 : bi;
    scores[r * K + t] = bs < 0 ? 0.0 : (double)fminf((float)bv, 1.0f);
    if (bs >= 0) ++head[bs];
  }
}

size_t rows_smem(int R, int64_t dp, int K) {
  return align_dev((size_t)R * K * 12) + align_dev((size_t)R * dp * 8) + (size_t)R * kT * 12;
}

// ---------------------------------------------------------------- k-means ---
constexpr double kFx = 1099511627776.0;  // 2^40: |x| <= 1, <= 2^23 rows per centroid

__global__ void ivf_kmeans_accum(const float* __restrict__ S, int64_t lds, const int32_t* __restrict__ arows,
                                 int64_t m, const int32_t* __restrict__ labels, int64_t d,
                                 unsigned long long* __restrict__ sums, int32_t* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < m;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t ar = arows ? arows[r] : r;
    const int c = labels[r];
    for (int64_t k = lane; k < d; k += 32)
      atomicAdd(sums + (int64_t)c * d + k,
                (unsigned long long)(long long)llrint((double)S[ar * lds + k] * kFx));
    if (lane == 0) atomicAdd(counts + c, 1);
  }
}

// C[c] = sums / count (empty clusters keep their centre), bias[c] = -|C[c]|^2 / 2
__global__ void ivf_kmeans_finish(unsigned long long* __restrict__ sums, int32_t* __restrict__ counts,
                                  int32_t nlist, int64_t d, float* __restrict__ C, int64_t ldc,
                                  float* __restrict__ bias) {
  const int lane = threadIdx.x & 31;
  for (int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; c < nlist;
       c += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int cnt = counts ? counts[c] : 0;
    double q = 0.0;
    for (int64_t k = lane; k < d; k += 32) {
      float v = C[c * ldc + k];
      if (cnt > 0 && sums) v = (float)((double)(long long)sums[c * d + k] / kFx / (double)cnt);
      C[c * ldc + k] = v;
      q = fma((double)v, (double)v, q);
      if (sums) sums[c * d + k] = 0ull;
    }
    q = warp_sum(q);
    if (lane == 0) {
      bias[c] = (float)(-0.5 * q);
      if (counts) counts[c] = 0;
    }
  }
}

}  // namespace ivf
}  // namespace ancka

using namespace ancka;
using namespace ancka::ivf;

static int grid_for(int64_t work, int per_block, int cap = kNumSMs * 16) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(cap, ceil_div(work, per_block)));
}

extern "C" int ancka_ivf_normalize(const double* X, int64_t ldx, const int64_t* indptr,
                                   const int32_t* indices, const double* data, int64_t n,
                                   int64_t d, float* xn, int64_t dp, ancka_stream_t stream) {
  ANCKA_REQUIRE(n >= 0 && d >= 0 && dp >= d && dp % 4 == 0, ANCKA_ERR_ARG,
                "ivf_normalize: bad shape n=%lld d=%lld dp=%lld", (long long)n, (long long)d,
                (long long)dp);
  if (n == 0) return ANCKA_OK;
  const int g = grid_for(n * 32, kT);
  if (X)
    ivf_normalize_dense<<<g, kT, 0, as_stream(stream)>>>(X, ldx, n, d, xn, dp);
  else
    ivf_normalize_csr<<<g, kT, 0, as_stream(stream)>>>(indptr, indices, data, n, xn, dp);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

extern "C" int ancka_ivf_gemm(const float* A, int64_t lda, const int32_t* arows, int64_t m,
                              const float* B, int64_t ldb, int32_t nb, int64_t d,
                              const float* bias, float* C, int64_t ldc,
                              unsigned long long* argmax_keys, ancka_stream_t stream) {
  ANCKA_REQUIRE(m >= 0 && nb > 0 && d > 0 && (C || argmax_keys), ANCKA_ERR_ARG,
                "ivf_gemm: bad arguments");
  if (m == 0) return ANCKA_OK;
  ANCKA_REQUIRE(ceil_div(nb, GT) < 65536, ANCKA_ERR_ARG, "ivf_gemm: nb=%d too large", nb);
  GemmP p{A, lda, arows, m, B, ldb, nb, d, bias, C, ldc, argmax_keys};
  dim3 grid((unsigned)ceil_div(m, GT), (unsigned)ceil_div(nb, GT));
  ivf_gemm<<<grid, kT, 0, as_stream(stream)>>>(p);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

extern "C" int ancka_ivf_argmax_finish(unsigned long long* argmax_keys, int64_t m, int32_t* labels,
                                       int32_t* changed, ancka_stream_t stream) {
  if (m == 0) return ANCKA_OK;
  ivf_argmax_finish<<<grid_for(m, kT), kT, 0, as_stream(stream)>>>(argmax_keys, m, labels, changed);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

extern "C" int ancka_ivf_topsel(const float* S, int64_t lds, int64_t m, int32_t nb, int32_t nprobe,
                                int32_t* probes, ancka_stream_t stream) {
  ANCKA_REQUIRE(nprobe >= 1 && nprobe <= nb, ANCKA_ERR_ARG, "ivf_topsel: nprobe=%d nb=%d", nprobe, nb);
  if (m == 0) return ANCKA_OK;
  ivf_topsel<<<grid_for(m * 32, kT), kT, 0, as_stream(stream)>>>(S, lds, m, nb, nprobe, probes);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

extern "C" size_t ancka_ivf_bucket_workspace_size(int32_t nbuckets) {
  return align_up(sizeof(int32_t) * 2 * (size_t)nbuckets);
}

extern "C" int ancka_ivf_bucket(const int32_t* keys, int64_t count, int32_t nbuckets, int64_t* ptr,
                                int64_t* tiles, int32_t tile, int32_t* ent, void* workspace,
                                size_t workspace_bytes, ancka_stream_t stream) {
  ANCKA_REQUIRE(workspace_bytes >= ancka_ivf_bucket_workspace_size(nbuckets), ANCKA_ERR_ARG,
                "ivf_bucket: workspace too small");
  cudaStream_t st = as_stream(stream);
  int32_t* cnt = static_cast<int32_t*>(workspace);
  int32_t* cur = cnt + nbuckets;
  ANCKA_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * 2 * (size_t)nbuckets, st));
  if (count) {
    ivf_bucket_count<<<grid_for(count, kT), kT, 0, st>>>(keys, count, cnt);
    ANCKA_LAUNCHED();
  }
  ivf_bucket_scan<<<1, 1024, 0, st>>>(cnt, nbuckets, ptr, tiles, tile > 0 ? tile : 1);
  ANCKA_LAUNCHED();
  if (count) {
    ivf_bucket_fill<<<grid_for(count, kT), kT, 0, st>>>(keys, count, ptr, cur, ent);
    ANCKA_LAUNCHED();
  }
  return ANCKA_OK;
}

extern "C" int ancka_ivf_search(const float* xn, int64_t dp, const int32_t* perm,
                                const int64_t* list_ptr, const int64_t* pair_ptr,
                                const int32_t* pair_ent, const int64_t* tile_ptr, int32_t* counter,
                                int32_t nlist, int32_t nprobe, int64_t q0, int32_t K2, float err,
                                float* part_s, int32_t* part_i, uint32_t* qthr,
                                ancka_stream_t stream) {
  ANCKA_REQUIRE(K2 >= 1 && K2 <= 256 && dp % 4 == 0, ANCKA_ERR_ARG, "ivf_search: K2=%d dp=%lld", K2,
                (long long)dp);
  cudaStream_t st = as_stream(stream);
  const size_t smem = search_layout(dp, K2).total;
  ANCKA_REQUIRE(smem <= 227 * 1024, ANCKA_ERR_ARG, "ivf_search: K2=%d needs %zu B shared", K2, smem);
  ANCKA_CUDA(cudaMemsetAsync(counter, 0, sizeof(int32_t), st));
  SearchP p{xn, dp, perm, list_ptr, pair_ptr, pair_ent, tile_ptr, counter, nlist, nprobe, q0, K2, -err,
            part_s, part_i, qthr};
  auto kern = dp <= kResD ? ivf_search<true> : ivf_search<false>;
  ANCKA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  ANCKA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kT, smem));
  kern<<<kNumSMs * std::max(1, per_sm), kT, smem, st>>>(p);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

extern "C" int ancka_ivf_half_prep(const float* xn, int64_t n, int64_t dp, void* h, int64_t dh,
                                   float* lres, uint32_t* lmax_bits, ancka_stream_t stream) {
  ANCKA_REQUIRE(dh % 16 == 0 && dh >= dp, ANCKA_ERR_ARG, "ivf_half_prep: dh=%lld", (long long)dh);
  cudaStream_t st = as_stream(stream);
  ANCKA_CUDA(cudaMemsetAsync(lmax_bits, 0, sizeof(uint32_t), st));
  if (n == 0) return ANCKA_OK;
  ivf_half_prep<<<grid_for(n * 32, kT), kT, 0, st>>>(xn, n, dp, static_cast<__half*>(h), dh, lres,
                                                    reinterpret_cast<unsigned*>(lmax_bits));
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

// Probe split for the two-phase scan: own[] keeps, per query, the probe slot
// of its own list (the list it is assigned to, always among its probes) and
// -1 elsewhere; rest[] the other slots.  Scanning the own pairs first sets
// each query's shared threshold from a whole list before the other pairs.
__global__ void ivf_split_probes_kernel(const int32_t* __restrict__ probes, const int32_t* __restrict__ labels,
                                        int64_t q0, int64_t m, int nprobe, int32_t* __restrict__ own,
                                        int32_t* __restrict__ rest) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * nprobe;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = e / nprobe;
    const int32_t c = probes[e];
    const bool mine = c == labels[q0 + q];
    own[e] = mine ? c : -1;
    rest[e] = mine ? -1 : c;
  }
}

extern "C" int ancka_ivf_split_probes(const int32_t* probes, const int32_t* labels, int64_t q0,
                                      int64_t m, int32_t nprobe, int32_t* own, int32_t* rest,
                                      ancka_stream_t stream) {
  if (m == 0) return ANCKA_OK;
  ivf_split_probes_kernel<<<grid_for(m * nprobe, kT), kT, 0, as_stream(stream)>>>(probes, labels, q0, m,
                                                                                 nprobe, own, rest);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

extern "C" int ancka_ivf_search_tc(const void* h, int64_t dh, const float* lres,
                                   const uint32_t* lmax_bits, const int32_t* perm,
                                   const int64_t* list_ptr, const int64_t* pair_ptr,
                                   const int32_t* pair_ent, const int64_t* tile_ptr, int32_t* counter,
                                   int32_t nlist, int32_t nprobe, int64_t q0, int32_t K2, float acc_err,
                                   float* part_s, int32_t* part_i, uint32_t* qthr,
                                   ancka_stream_t stream) {
  ANCKA_REQUIRE(K2 >= 1 && K2 <= 32 && dh % 16 == 0 && dh <= kMaxDh, ANCKA_ERR_ARG,
                "ivf_search_tc: K2=%d dh=%lld", K2, (long long)dh);
  cudaStream_t st = as_stream(stream);
  const size_t smem = search_tc_smem(dh, K2);
  auto kern = dh <= 128 ? ivf_search_tc<8> : ivf_search_tc<0>;
  ANCKA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ANCKA_CUDA(cudaMemsetAsync(counter, 0, sizeof(int32_t), st));
  int per_sm = 0;
  ANCKA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kT, smem));
  SearchTcP P{};
  P.s = SearchP{nullptr, 0, perm, list_ptr, pair_ptr, pair_ent, tile_ptr, counter, nlist, nprobe, q0, K2,
                0.f, part_s, part_i, qthr};
  P.h = static_cast<const __half*>(h);
  P.dh = dh;
  P.lres = lres;
  P.lmax_bits = reinterpret_cast<const unsigned*>(lmax_bits);
  P.acc_err = acc_err;
  kern<<<kNumSMs * std::max(1, per_sm), kT, smem, st>>>(P);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

extern "C" int ancka_ivf_merge(const float* xn, int64_t dp, int64_t q0, int64_t m, int32_t nprobe,
                               int32_t K2, int32_t K, const float* part_s, const int32_t* part_i,
                               float err, int32_t* ids, double* scores, int32_t* flagged,
                               int32_t* nflag, const float* lres, const uint32_t* lmax_bits,
                               ancka_stream_t stream) {
  ANCKA_REQUIRE(K >= 1 && K2 >= K && K2 <= 256, ANCKA_ERR_ARG, "ivf_merge: K=%d K2=%d", K, K2);
  if (m == 0) return ANCKA_OK;
  MergeP p{xn, dp, q0, m, nprobe, K2, K, part_s, part_i, err, ids, scores, flagged, nflag, lres,
           reinterpret_cast<const unsigned*>(lmax_bits)};
  if (K2 <= 32) {
    ivf_merge_warp<<<grid_for(m * 32, 32 * kMergeWarps, kNumSMs * 32), 32 * kMergeWarps, 0,
                     as_stream(stream)>>>(p);
    ANCKA_LAUNCHED();
    return ANCKA_OK;
  }
  const size_t smem = align_dev((size_t)kMergeWarps * K2 * 8) + (size_t)kMergeWarps * K2 * 8;
  ANCKA_CUDA(cudaFuncSetAttribute(ivf_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ivf_merge<<<grid_for(m * 32, 32 * kMergeWarps, kNumSMs * 32), 32 * kMergeWarps, smem,
              as_stream(stream)>>>(p);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

extern "C" int ancka_ivf_rows_exact(const float* xn, int64_t dp, int64_t n, const int32_t* rows,
                                    int64_t nrows, const int32_t* probes, int32_t nprobe, int64_t q0,
                                    const int32_t* perm, const int64_t* list_ptr, int32_t K,
                                    int32_t* ids, double* scores, int32_t compact,
                                    ancka_stream_t stream) {
  ANCKA_REQUIRE(K >= 1 && K <= 1024 && dp % 4 == 0, ANCKA_ERR_ARG, "ivf_rows_exact: K=%d", K);
  if (nrows == 0) return ANCKA_OK;
  int R = probes ? 1 : kRowsR;
  while (R > 1 && rows_smem(R, dp, K) > 160 * 1024) R >>= 1;
  const size_t smem = rows_smem(R, dp, K);
  ANCKA_REQUIRE(smem <= 227 * 1024, ANCKA_ERR_ARG, "ivf_rows_exact: d=%lld K=%d exceed shared memory",
                (long long)dp, K);
  ANCKA_CUDA(cudaFuncSetAttribute(ivf_rows_exact, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  RowsP p{xn, dp, n, rows, nrows, probes, nprobe, q0, perm, list_ptr, K, ids, scores, compact, R,
          1, nullptr, nullptr};
  const int64_t gx = ceil_div(nrows, R);
  if (!probes && compact && gx < 4 * kNumSMs) {     // few rows: split the keys as well
    p.nsplit = (int)std::min<int64_t>(64, ceil_div(4 * kNumSMs, gx));
    ANCKA_CUDA(cudaMallocAsync(&p.seg_sc, sizeof(double) * nrows * p.nsplit * K, as_stream(stream)));
    ANCKA_CUDA(cudaMallocAsync(&p.seg_id, sizeof(int32_t) * nrows * p.nsplit * K, as_stream(stream)));
  }
  ivf_rows_exact<<<dim3((unsigned)gx, (unsigned)p.nsplit), kT, smem, as_stream(stream)>>>(p);
  ANCKA_LAUNCHED();
  if (p.nsplit > 1) {
    ivf_rows_seg_merge<<<(unsigned)ceil_div(nrows, 128), 128, 0, as_stream(stream)>>>(
        p.seg_sc, p.seg_id, nrows, p.nsplit, K, ids, scores);
    ANCKA_LAUNCHED();
    ANCKA_CUDA(cudaFreeAsync(p.seg_sc, as_stream(stream)));
    ANCKA_CUDA(cudaFreeAsync(p.seg_id, as_stream(stream)));
  }
  return ANCKA_OK;
}

extern "C" int ancka_ivf_kmeans_update(const float* S, int64_t lds, const int32_t* arows, int64_t m,
                                       const int32_t* labels, int32_t nlist, int64_t d,
                                       unsigned long long* sums, int32_t* counts, float* C,
                                       int64_t ldc, float* bias, ancka_stream_t stream) {
  cudaStream_t st = as_stream(stream);
  if (sums && m) {
    ivf_kmeans_accum<<<grid_for(m * 32, kT), kT, 0, st>>>(S, lds, arows, m, labels, d, sums, counts);
    ANCKA_LAUNCHED();
  }
  ivf_kmeans_finish<<<grid_for((int64_t)nlist * 32, kT), kT, 0, st>>>(sums, counts, nlist, d, C, ldc,
                                                                      bias);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}
