// Exact KNN on the 5th-gen tensor cores for integer-valued attributes
// (bag-of-words and other count data): knn.py:112-140 with the ordering of
// _ordered_top_k (knn.py:83-98), computed exactly.
//
// X is quantised losslessly (|x| <= 16 -> e4m3 fp8, |x| <= 256 -> bf16) and
// S = X X^T is contracted by tcgen05.mma into f32 TMEM accumulators, which
// are exact integers (row sums of squares < 2^24).  Cosine order is decided
// by exact integer arithmetic: s_j > s_l  <=>  c_j^2 a_l > c_l^2 a_j  with
// c = dot count and a = squared norm, ties by smaller index -- the canonical
// order the reference's f64 arithmetic approximates.  The n x n similarity
// matrix never leaves TMEM/registers.
//
// Pipeline (TMA producer, tcgen05 issuer, TMEM double buffer): knn_tc.cuh.
// Epilogue warps stream each query row's accumulator columns into a
// register-resident exact top-K list.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp8.h>
#include <cstdlib>

#include "common.cuh"
#include "knn.cuh"
#include "knn_tc.cuh"
#include "sm100.cuh"

namespace ancka {
using namespace sm100;


struct Entry {
  uint32_t c;  // exact dot count (0 = empty slot)
  uint32_t a;  // squared norm of the neighbour
  int32_t j;   // neighbour index
};

// exact: c1/sqrt(a1) > c2/sqrt(a2), ties -> smaller index; c2 == 0 is empty
__device__ __forceinline__ bool better(uint32_t c1, uint32_t a1, int32_t j1, uint32_t c2,
                                       uint32_t a2, int32_t j2) {
  if (c2 == 0) return true;
  const uint64_t l = (uint64_t)c1 * c1, r = (uint64_t)c2 * c2;
  const uint64_t lh = __umul64hi(l, (uint64_t)a2), ll = l * (uint64_t)a2;
  const uint64_t rh = __umul64hi(r, (uint64_t)a1), rl = r * (uint64_t)a1;
  if (lh != rh) return lh > rh;
  if (ll != rl) return ll > rl;
  return j1 < j2;
}

// f32 keys c * rsqrt(a) carry < 3e-7 relative error, so two keys whose f32
// values differ by more than kBand relative are ordered by the f32 compare;
// only keys inside the band need the exact integer comparison.
constexpr float kBand = 4e-6f;

// Register-resident exact top-K.  The list always has KMAX slots; the first
// KMAX-K are padding with key +inf (never displaced) and the K live entries
// occupy slots KMAX-K..KMAX-1, best first.  The K-th entry is therefore
// always slot KMAX-1 and no slot is ever addressed by a runtime index, which
// keeps the arrays in registers.
template <int KMAX>
struct TopK {
  uint32_t c[KMAX], a[KMAX];
  int32_t j[KMAX];
  float f[KMAX];           // f32 keys: +inf padding, 0 empty
  float thr_lo, thr_hi;    // band around the K-th key (-1 while not full)
  float floor_lo;          // shared lower bound of the row's true K-th key (banded)

  __device__ __forceinline__ void clear(int K) {
#pragma unroll
    for (int t = 0; t < KMAX; ++t) {
      const bool pad = t < KMAX - K;
      c[t] = 0; a[t] = 1; j[t] = -1;
      f[t] = pad ? __int_as_float(0x7f800000) : 0.f;
    }
    thr_lo = thr_hi = -1.f;
    floor_lo = -1.f;
  }

  // raise the pruning floor to a bound learned elsewhere (another list of
  // the same row): any key below it cannot be among the row's top K
  __device__ __forceinline__ void raise_floor(float bound) {
    const float lo = bound * (1.f - kBand);
    floor_lo = fmaxf(floor_lo, lo);
    thr_lo = fmaxf(thr_lo, floor_lo);
  }

  // does the candidate rank before entry t?  ff_lo / ff_hi = ff (1 -/+ 2 kBand)
  // bracket the band once per insert: f2 < ff_lo implies ff > f2 (1 + kBand),
  // f2 > ff_hi implies ff < f2 (1 - kBand); equal (c, a) -- the common exact
  // tie of binary attributes -- is decided by the index without products
  __device__ __forceinline__ static bool above(float ff_lo, float ff_hi, uint32_t cc, uint32_t aa,
                                               int32_t jj, float f2, uint32_t c2, uint32_t a2,
                                               int32_t j2) {
    if (f2 == 0.f) return true;                       // empty slot
    if (f2 < ff_lo) return true;
    if (f2 > ff_hi) return false;                     // includes +inf padding
    if (cc == c2 && aa == a2) return jj < j2;
    return better(cc, aa, jj, c2, a2, j2);
  }

  // Does the candidate enter the list?  a_norm is read only inside the band.
  __device__ __forceinline__ bool admits(float ff, uint32_t cc, int32_t jj,
                                         const uint32_t* __restrict__ a_norm) const {
    if (ff < thr_lo) return false;
    const float fk = f[KMAX - 1];
    if (fk == 0.f || ff > thr_hi) return true;
    const uint32_t aa = __ldg(a_norm + jj);
    if (cc == c[KMAX - 1] && aa == a[KMAX - 1]) return jj < j[KMAX - 1];  // exact (c, a) tie
    return better(cc, aa, jj, c[KMAX - 1], a[KMAX - 1], j[KMAX - 1]);
  }

  // rank against every slot with independent compares, then shift with
  // fixed-index selects
  __device__ __forceinline__ void insert(float ff, uint32_t cc, uint32_t aa, int32_t jj) {
    int pos = 0;
    const float ff_lo = ff * (1.f - 2.f * kBand), ff_hi = ff * (1.f + 2.f * kBand);
#pragma unroll
    for (int t = 0; t < KMAX; ++t) pos += above(ff_lo, ff_hi, cc, aa, jj, f[t], c[t], a[t], j[t]) ? 0 : 1;
#pragma unroll
    for (int t = KMAX - 1; t > 0; --t) {
      const bool sh = t > pos, put = t == pos;
      c[t] = sh ? c[t - 1] : (put ? cc : c[t]);
      a[t] = sh ? a[t - 1] : (put ? aa : a[t]);
      j[t] = sh ? j[t - 1] : (put ? jj : j[t]);
      f[t] = sh ? f[t - 1] : (put ? ff : f[t]);
    }
    if (pos == 0) { c[0] = cc; a[0] = aa; j[0] = jj; f[0] = ff; }
    const float fk = f[KMAX - 1];
    thr_lo = fmaxf(fk == 0.f ? -1.f : fk * (1.f - kBand), floor_lo);
    thr_hi = fk == 0.f ? -1.f : fk * (1.f + kBand);
  }

  // entry r (0 = best) of the K live entries, written without runtime indexing
  template <typename F>
  __device__ __forceinline__ void emit(int K, F&& out) const {
#pragma unroll
    for (int t = 0; t < KMAX; ++t)
      if (t >= KMAX - K) out(t - (KMAX - K), c[t], a[t], j[t]);
  }
};

struct TcParams {
  int64_t n;
  int d;              // attribute columns: MMA k-steps past d are skipped
  int nkb;            // k-blocks of 128 bytes along d
  int K;
  int key_tiles;      // end key tile (exclusive) of BN
  int kt_base;        // first key tile
  int tiles_per_seg;
  int nseg;
  const uint32_t* a_norm;   // n_pad
  const float* inv_sqrt;    // n_pad
  int2* partial;            // n x nseg x K  (c, j)
  int debug;                // 0 normal; 1 skip epilogue math; 2 skip MMA issue
  int64_t q_begin, q_end;   // query rows handled by this launch (row sharding)
  int* row_bound;           // n: best known K-th key per row (f32 bits, atomicMax)
};

template <bool FP8, int KMAX>
__global__ void __launch_bounds__(tc::THREADS, 1)
knn_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              TcParams p) {
  using namespace tc;
  extern __shared__ __align__(1024) unsigned char smraw[];
  const Pipe P = setup(smraw, &tmA, &tmB);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t q0 = p.q_begin + (int64_t)blockIdx.x * BM;
  const int seg = blockIdx.y;
  const int kt0 = p.kt_base + seg * p.tiles_per_seg;
  const int kt1 = min(p.key_tiles, kt0 + p.tiles_per_seg);
  const int ntiles = kt1 - kt0;
  const uint32_t tmem = P.tmem;

  if (warp == 0) {
    if (lane == 0)
      producer(P, &tmA, &tmB, kt0, ntiles, p.nkb, (int)q0, [](int kb, int& ca, int& cb) {
        ca = cb = kb * ROW_BYTES / (FP8 ? 1 : 2);
      });
  } else if (warp == 1) {
    if (lane == 0) mma_issuer<FP8>(P, ntiles, p.nkb, p.debug == 2, p.d);
  } else {
    // ------------------------------------------------------ epilogue
    const int ew = warp - 2;                      // epilogue warp 0..EPI_WARPS-1
    const int quarter = warp & 3;                 // TMEM lane quarter of this warp
    const int half = ew / 4;                      // which column range of the tile
    const int row = quarter * 32 + lane;
    const int64_t i = q0 + row;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    TopK<KMAX> L;
    L.clear(p.K);
    float published = 0.f;
    float* stash = P.stash_base + (threadIdx.x - 64) * 33;
    // shared floor read one tile ahead (the L2 round trip overlaps the tile)
    int floor_next = i < p.q_end ? __ldcg(p.row_bound + (i - p.q_begin)) : 0;
    for (int t = 0; t < ntiles; ++t) {
      const int acc = t & 1;
      const uint32_t acc_phase = (t >> 1) & 1;
      mbar_wait_sleep(&P.tfull[acc], acc_phase);
      if (i < p.q_end) {
        L.raise_floor(__int_as_float(floor_next));
        floor_next = __ldcg(p.row_bound + (i - p.q_begin));
      }
      tc_fence_after();
      const int64_t j0 = (int64_t)(kt0 + t) * BN + half * EPI_COLS;
#pragma unroll 1
      for (int ch = 0; ch < EPI_COLS / 32; ++ch) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_off + acc * BN + half * EPI_COLS + ch * 32, r);
        tmem_ld_wait();
        if (ch == EPI_COLS / 32 - 1) {     // this warp's share is in registers
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&P.tempty[acc]);
        }
        if (p.debug == 1) continue;
        // fast filter (branch-free, unrolled): candidate bitmask against the
        // current K-th key; the rare survivors take one out-of-line slow path.
        // (A max-tree pre-test as in the real-valued kernel does not pay here:
        // binary attributes give large exact tie groups at the K-th key, so
        // most 32-column chunks hold a key inside the band.)
        const int64_t jb = j0 + ch * 32;
        uint32_t mask = 0;
        // the 32 key scales as eight 16-byte loads (jb is a multiple of 32;
        // inv_sqrt is padded to n_pad), the same addresses for the whole warp
        const float4* is4 = reinterpret_cast<const float4*>(p.inv_sqrt + jb);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 sc = __ldg(is4 + q);
          const float s4[4] = {sc.x, sc.y, sc.z, sc.w};
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            const int u = 4 * q + w;
            const float v = __uint_as_float(r[u]);
            const bool keep = (v > 0.5f) & (v * s4[w] >= L.thr_lo);
            mask |= (uint32_t)keep << u;
          }
        }
        if (i >= jb && i < jb + 32) mask &= ~(1u << (int)(i - jb));   // j != i
        if (jb + 32 > p.n) mask &= p.n > jb ? (1u << (int)(p.n - jb)) - 1u : 0u;
        if (mask) {
#pragma unroll
          for (int u = 0; u < 32; ++u) stash[u] = __uint_as_float(r[u]);
        }
#pragma unroll 1
        while (mask) {
          const int u = __ffs(mask) - 1;
          mask &= mask - 1;
          const float v = stash[u];
          const int32_t j = (int32_t)(jb + u);
          const float kf = v * __ldg(p.inv_sqrt + j);
          const uint32_t cc = (uint32_t)(v + 0.5f);
          if (L.admits(kf, cc, j, p.a_norm)) {
            L.insert(kf, cc, __ldg(p.a_norm + j), j);
            const float fk = L.f[KMAX - 1];
            if (fk > published) {        // share the row's improved bound
              atomicMax(p.row_bound + (i - p.q_begin), __float_as_int(fk));
              published = fk;
            }
          }
        }
      }
    }
    if (i < p.q_end) {
      const int lists = p.nseg * (EPI_WARPS / 4);
      int2* out = p.partial + ((size_t)(i - p.q_begin) * lists + seg * (EPI_WARPS / 4) + half) * p.K;
      L.emit(p.K, [&](int r, uint32_t c, uint32_t, int32_t j) {
        out[r] = make_int2((int)c, c ? j : -1);
      });
    }
  }
  teardown(P);
}

// Merge the per-segment lists (exact order) and emit ids / f64 cosines.
template <int KMAX>
__global__ void knn_tc_merge_kernel(const int2* __restrict__ partial, int64_t q_begin, int64_t nq,
                                    int nseg, int K,
                                    const uint32_t* __restrict__ a_norm,
                                    const float* __restrict__ inv_sqrt, int32_t* __restrict__ ids,
                                    double* __restrict__ scores) {
  for (int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; li < nq;
       li += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q_begin + li;
    TopK<KMAX> L;
    L.clear(K);
    for (int s = 0; s < nseg; ++s) {
      const int2* src = partial + ((size_t)li * nseg + s) * K;
      for (int t = 0; t < K; ++t) {
        const int2 e = src[t];
        if (e.x <= 0) break;
        const float kf = (float)e.x * inv_sqrt[e.y];
        if (L.admits(kf, (uint32_t)e.x, e.y, a_norm))
          L.insert(kf, (uint32_t)e.x, a_norm[e.y], e.y);
      }
    }
    const double ai = (double)a_norm[i];
    L.emit(K, [&](int r, uint32_t c, uint32_t a, int32_t j) {
      const bool ok = c != 0;
      ids[li * K + r] = ok ? j : -1;
      scores[li * K + r] = ok ? fmin((double)c / sqrt(ai * (double)a), 1.0) : 0.0;
    });
  }
}

// f64 dense X -> padded fp8/bf16 rows + exact squared norms.
template <bool FP8>
__global__ void knn_tc_prep_kernel(const double* __restrict__ X, int64_t n, int64_t d, int64_t ldx,
                                   int64_t n_pad, int64_t d_pad, void* __restrict__ xq,
                                   uint32_t* __restrict__ a_norm, float* __restrict__ inv_sqrt) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < n_pad; r += nwarps) {
    double s = 0.0;
    for (int64_t c = lane; c < d_pad; c += 32) {
      const double v = (r < n && c < d) ? X[r * ldx + c] : 0.0;
      s += v * v;
      if (FP8) reinterpret_cast<__nv_fp8_e4m3*>(xq)[r * d_pad + c] = __nv_fp8_e4m3((float)v);
      else reinterpret_cast<__nv_bfloat16*>(xq)[r * d_pad + c] = __float2bfloat16_rn((float)v);
    }
    s = warp_sum(s);
    if (lane == 0) {
      a_norm[r] = (uint32_t)s;
      inv_sqrt[r] = s > 0 ? (float)(1.0 / sqrt(s)) : 0.f;
    }
  }
}

// --------------------------------------------------------------- host side
struct TcLayout {
  bool fp8;
  int64_t n_pad, d_pad, d;
  int nseg, tiles_per_seg, key_tiles, q_tiles;
  KeyRange kr;
};

static TcLayout tc_layout(int64_t n, int64_t d, bool fp8, int64_t nq, KeyRange kr = {0, -1}) {
  TcLayout L;
  L.fp8 = fp8;
  L.n_pad = ceil_div(n, tc::BN) * tc::BN;
  const int64_t elems_per_row = tc::ROW_BYTES / (fp8 ? 1 : 2);
  L.d_pad = ceil_div(d, elems_per_row) * elems_per_row;
  L.d = d;
  const TcGrid g = tc_grid(n, nq, kr);
  L.kr = {kr.k0, kr.k1 < 0 ? n : kr.k1};
  L.q_tiles = g.q_tiles;
  L.key_tiles = g.key_tiles;
  L.nseg = g.nseg;
  L.tiles_per_seg = g.tiles_per_seg;
  return L;
}

static void carve_tc(Carver& cv, const TcLayout& L, int64_t n, int K, void** xq, uint32_t** an,
                     float** isq, int** rb, int2** part) {
  *xq = cv.take<unsigned char>((size_t)L.n_pad * L.d_pad * (L.fp8 ? 1 : 2));
  *an = cv.take<uint32_t>(L.n_pad);
  *isq = cv.take<float>(L.n_pad);
  *rb = cv.take<int>(L.n_pad);
  // nq * nseg <= n + 8 * 148 * BM for every query range (nseg ~ 8*148 / q_tiles)
  *part = cv.take<int2>(((size_t)n + 8 * kNumSMs * tc::BM) * (tc::EPI_WARPS / 4) * K);
}

// the fp8 path is taken when the host asserts |x| <= 16 via integer_exact == 2
size_t knn_tc_workspace(int64_t n, int64_t d, int K) {
  Carver cv(nullptr, 0);
  TcLayout L = tc_layout(n, d, false, n);  // bf16 bound covers fp8
  void* xq;
  uint32_t* an;
  float* isq;
  int* rb;
  int2* part;
  carve_tc(cv, L, n, K, &xq, &an, &isq, &rb, &part);
  return cv.used;
}

template <bool FP8, int KMAX>
static int launch_tc(const CUtensorMap& ma, const CUtensorMap& mb, const TcParams& p,
                     const TcLayout& L, cudaStream_t st) {
  auto kern = knn_tc_kernel<FP8, KMAX>;
  ANCKA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc::SMEM));
  dim3 grid(L.q_tiles, L.nseg);
  kern<<<grid, tc::THREADS, tc::SMEM, st>>>(ma, mb, p);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

// CSR X -> zero-filled padded fp8/bf16 rows + exact squared norms (warp per row)
template <bool FP8>
__global__ void knn_tc_prep_csr_kernel(const int64_t* __restrict__ indptr,
                                       const int32_t* __restrict__ indices,
                                       const double* __restrict__ data, int64_t n, int64_t n_pad,
                                       int64_t d_pad, void* __restrict__ xq,
                                       uint32_t* __restrict__ a_norm, float* __restrict__ inv_sqrt) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < n_pad; r += nwarps) {
    double s = 0.0;
    if (r < n) {
      for (int64_t q = indptr[r] + lane; q < indptr[r + 1]; q += 32) {
        const double v = data[q];
        const int64_t c = indices[q];
        s += v * v;
        if (FP8) reinterpret_cast<__nv_fp8_e4m3*>(xq)[r * d_pad + c] = __nv_fp8_e4m3((float)v);
        else reinterpret_cast<__nv_bfloat16*>(xq)[r * d_pad + c] = __float2bfloat16_rn((float)v);
      }
    }
    s = warp_sum(s);
    if (lane == 0) {
      a_norm[r] = (uint32_t)s;
      inv_sqrt[r] = s > 0 ? (float)(1.0 / sqrt(s)) : 0.f;
    }
  }
}

static int knn_tc_main(void* xq, uint32_t* an, float* isq, int* rb, int2* part, const TcLayout& L,
                       int64_t n, int K, int64_t q_begin, int64_t q_end, int32_t* ids,
                       double* scores, cudaStream_t st, bool fp8);

int knn_tc_csr(const int64_t* indptr, const int32_t* indices, const double* data, int64_t n,
               int64_t d, int K, int64_t q_begin, int64_t q_end, int32_t* ids, double* scores,
               void* ws, size_t wsb, cudaStream_t st, bool fp8, KeyRange kr) {
  ANCKA_REQUIRE(K <= 32, ANCKA_ERR_UNSUPPORTED, "tensor-core KNN supports K <= 32 (got %d)", K);
  ANCKA_REQUIRE(n < (1ll << 31), ANCKA_ERR_UNSUPPORTED, "tensor-core KNN: n too large");
  TcLayout L = tc_layout(n, d, fp8, q_end - q_begin, kr);
  Carver cv(ws, wsb);
  void* xq;
  uint32_t* an;
  float* isq;
  int* rb;
  int2* part;
  carve_tc(cv, L, n, K, &xq, &an, &isq, &rb, &part);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "knn_tc: workspace too small");
  ANCKA_CUDA(cudaMemsetAsync(xq, 0, (size_t)L.n_pad * L.d_pad * (fp8 ? 1 : 2), st));
  const int pg = (int)std::min<int64_t>(ceil_div(L.n_pad * 32, 256), 16 * kNumSMs);
  if (fp8)
    knn_tc_prep_csr_kernel<true><<<pg, 256, 0, st>>>(indptr, indices, data, n, L.n_pad, L.d_pad, xq, an, isq);
  else
    knn_tc_prep_csr_kernel<false><<<pg, 256, 0, st>>>(indptr, indices, data, n, L.n_pad, L.d_pad, xq, an, isq);
  ANCKA_LAUNCHED();
  return knn_tc_main(xq, an, isq, rb, part, L, n, K, q_begin, q_end, ids, scores, st, fp8);
}

int knn_tc(const double* X, int64_t n, int64_t d, int64_t ldx, int K, int64_t q_begin,
           int64_t q_end, int32_t* ids, double* scores, void* ws, size_t wsb, cudaStream_t st,
           bool fp8, KeyRange kr) {
  ANCKA_REQUIRE(K <= 32, ANCKA_ERR_UNSUPPORTED, "tensor-core KNN supports K <= 32 (got %d)", K);
  ANCKA_REQUIRE(n < (1ll << 31), ANCKA_ERR_UNSUPPORTED, "tensor-core KNN: n too large");
  TcLayout L = tc_layout(n, d, fp8, q_end - q_begin, kr);
  Carver cv(ws, wsb);
  void* xq;
  uint32_t* an;
  float* isq;
  int* rb;
  int2* part;
  carve_tc(cv, L, n, K, &xq, &an, &isq, &rb, &part);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "knn_tc: workspace too small");
  const int pg = (int)std::min<int64_t>(ceil_div(L.n_pad * 32, 256), 16 * kNumSMs);
  if (fp8)
    knn_tc_prep_kernel<true><<<pg, 256, 0, st>>>(X, n, d, ldx, L.n_pad, L.d_pad, xq, an, isq);
  else
    knn_tc_prep_kernel<false><<<pg, 256, 0, st>>>(X, n, d, ldx, L.n_pad, L.d_pad, xq, an, isq);
  ANCKA_LAUNCHED();
  return knn_tc_main(xq, an, isq, rb, part, L, n, K, q_begin, q_end, ids, scores, st, fp8);
}

static int knn_tc_main(void* xq, uint32_t* an, float* isq, int* rb, int2* part, const TcLayout& L,
                       int64_t n, int K, int64_t q_begin, int64_t q_end, int32_t* ids,
                       double* scores, cudaStream_t st, bool fp8) {
  CUtensorMap ma, mb;
  ANCKA_TRY(tc_make_map(&ma, xq, fp8, L.n_pad, L.d_pad, tc::BM));
  ANCKA_TRY(tc_make_map(&mb, xq, fp8, L.n_pad, L.d_pad, tc::BN));
  TcParams p;
  p.n = L.kr.k1;                      // key index bound (masking)
  p.kt_base = (int)(L.kr.k0 / tc::BN);
  p.d = (int)L.d;
  p.q_begin = q_begin;
  p.q_end = q_end;
  p.nkb = (int)(L.d_pad * (fp8 ? 1 : 2) / tc::ROW_BYTES);
  p.K = K;
  p.key_tiles = p.kt_base + L.key_tiles;
  p.tiles_per_seg = L.tiles_per_seg;
  p.nseg = L.nseg;
  p.a_norm = an;
  p.inv_sqrt = isq;
  p.partial = part;
  p.row_bound = rb;
  ANCKA_CUDA(cudaMemsetAsync(rb, 0, sizeof(int) * (q_end - q_begin), st));
  p.debug = getenv("ANCKA_KNN_DEBUG") ? atoi(getenv("ANCKA_KNN_DEBUG")) : 0;
  if (fp8) {
    if (K <= 10) { ANCKA_TRY((launch_tc<true, 10>(ma, mb, p, L, st))); }
    else if (K <= 12) { ANCKA_TRY((launch_tc<true, 12>(ma, mb, p, L, st))); }
    else if (K <= 16) { ANCKA_TRY((launch_tc<true, 16>(ma, mb, p, L, st))); }
    else { ANCKA_TRY((launch_tc<true, 32>(ma, mb, p, L, st))); }
  } else {
    if (K <= 10) { ANCKA_TRY((launch_tc<false, 10>(ma, mb, p, L, st))); }
    else if (K <= 12) { ANCKA_TRY((launch_tc<false, 12>(ma, mb, p, L, st))); }
    else if (K <= 16) { ANCKA_TRY((launch_tc<false, 16>(ma, mb, p, L, st))); }
    else { ANCKA_TRY((launch_tc<false, 32>(ma, mb, p, L, st))); }
  }
  const int64_t nq = q_end - q_begin;
  const int mg = (int)std::min<int64_t>(ceil_div(nq, 128), 8 * kNumSMs);
  if (K <= 10)
    knn_tc_merge_kernel<10><<<mg, 128, 0, st>>>(part, q_begin, nq, L.nseg * (tc::EPI_WARPS / 4), K, an, isq, ids, scores);
  else if (K <= 16)
    knn_tc_merge_kernel<16><<<mg, 128, 0, st>>>(part, q_begin, nq, L.nseg * (tc::EPI_WARPS / 4), K, an, isq, ids, scores);
  else
    knn_tc_merge_kernel<32><<<mg, 128, 0, st>>>(part, q_begin, nq, L.nseg * (tc::EPI_WARPS / 4), K, an, isq, ids, scores);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

}  // namespace ancka
