// Shared tcgen05 / TMA pipeline of the tensor-core KNN kernels.
//
// CTA = 2 + EPI_WARPS warps, one 128-row query tile x one key segment:
//   warp 0     TMA producer (A: 128 x 128B, B: 256 x 128B per stage, SW128)
//   warp 1     TMEM allocator + single-thread MMA issuer (M=128, N=256)
//   warps 2..  epilogue (kernel specific): thread owns query row (TMEM lane)
//              and streams accumulator columns of each key tile out of the
//              double-buffered TMEM accumulator.
// The k-loop walks `nkb` 128-byte k-blocks; a column map gives, per k-block,
// the element column of the A (query) and B (key) tiles, which lets the
// split-precision kernel contract [hi|hi|lo] against [hi|lo|hi] out of one
// stored [hi|lo] matrix.
#pragma once
#include <cuda.h>

#include <cstdlib>

#include "common.cuh"
#include "sm100.cuh"

namespace ancka {
namespace tc {
constexpr int BM = 128, BN = 256;
constexpr int STAGES = 4;
constexpr int ROW_BYTES = 128;                    // one SW128 row per stage
constexpr int A_BYTES = BM * ROW_BYTES;           // 16 KB
constexpr int B_BYTES = BN * ROW_BYTES;           // 32 KB
constexpr int EPI_WARPS = 8;                      // two per TMEM lane quarter
constexpr int THREADS = 64 + 32 * EPI_WARPS;
constexpr int EPI_COLS = BN / (EPI_WARPS / 4);    // accumulator columns per epilogue warp
constexpr int TMEM_COLS = 512;                    // 2 accumulators x 256 columns
constexpr size_t SMEM = 1024 + STAGES * (A_BYTES + B_BYTES) + 256 + 32 * EPI_WARPS * 33 * 4;

struct Pipe {
  unsigned char *sA, *sB;
  uint64_t *full, *empty, *tfull, *tempty;
  uint32_t* tmem_slot;
  float* stash_base;   // EPI_WARPS * 32 threads x 33 floats
  uint32_t tmem;
};

// carve shared memory, init barriers, allocate TMEM (all threads call)
__device__ __forceinline__ Pipe setup(unsigned char* smraw, const CUtensorMap* ma,
                                      const CUtensorMap* mb) {
  using namespace sm100;
  Pipe P;
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  P.sA = base;
  P.sB = base + STAGES * A_BYTES;
  P.full = reinterpret_cast<uint64_t*>(P.sB + STAGES * B_BYTES);
  P.empty = P.full + STAGES;
  P.tfull = P.empty + STAGES;
  P.tempty = P.tfull + 2;
  P.tmem_slot = reinterpret_cast<uint32_t*>(P.tempty + 2);
  P.stash_base = reinterpret_cast<float*>(P.tmem_slot + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch(ma);
    tma_prefetch(mb);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&P.full[s], 1); mbar_init(&P.empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&P.tfull[s], 1); mbar_init(&P.tempty[s], EPI_WARPS); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<TMEM_COLS>(P.tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  P.tmem = *P.tmem_slot;
  return P;
}

// warp 0, lane 0: stream A/B k-blocks of every key tile of the segment
template <typename ColMap>
__device__ __forceinline__ void producer(const Pipe& P, const CUtensorMap* ma,
                                         const CUtensorMap* mb, int kt0, int ntiles, int nkb,
                                         int q0, const ColMap& cols) {
  using namespace sm100;
  int stage = 0;
  uint32_t phase = 0;
  for (int t = 0; t < ntiles; ++t) {
    const int krow = (kt0 + t) * BN;
    for (int kb = 0; kb < nkb; ++kb) {
      int ca, cb;
      cols(kb, ca, cb);
      mbar_wait_sleep(&P.empty[stage], phase ^ 1);
      mbar_arrive_expect_tx(&P.full[stage], A_BYTES + B_BYTES);
      tma_load_2d(P.sA + stage * A_BYTES, ma, &P.full[stage], ca, q0);
      tma_load_2d(P.sB + stage * B_BYTES, mb, &P.full[stage], cb, krow);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
  }
}

// warp 1, lane 0: one 128 x 256 accumulator per key tile, alternating halves
template <bool FP8>
__device__ __forceinline__ void mma_issuer(const Pipe& P, int ntiles, int nkb, bool skip,
                                           int k_elems = 1 << 30) {
  using namespace sm100;
  constexpr uint32_t idesc = make_idesc(FP8 ? 0u : 1u, BM, BN);
  int stage = 0;
  uint32_t phase = 0;
  for (int t = 0; t < ntiles; ++t) {
    const int acc = t & 1;
    const uint32_t acc_phase = (t >> 1) & 1;
    mbar_wait_sleep(&P.tempty[acc], acc_phase ^ 1);
    tc_fence_after();
    const uint32_t dtm = P.tmem + acc * BN;
    for (int kb = 0; kb < nkb; ++kb) {
      mbar_wait_sleep(&P.full[stage], phase);
      tc_fence_after();
      const uint32_t a_addr = smem_u32(P.sA + stage * A_BYTES);
      const uint32_t b_addr = smem_u32(P.sB + stage * B_BYTES);
#pragma unroll
      for (int k = 0; k < 4; ++k) {  // 4 x 32 bytes of K per 128-byte row
        const uint64_t ad = sw128_kmajor_desc(a_addr + k * 32);
        const uint64_t bd = sw128_kmajor_desc(b_addr + k * 32);
        // k-steps entirely in the zero padding past the last column are skipped
        if (skip || (kb * 4 + k) * (FP8 ? 32 : 16) >= k_elems) continue;
        if (FP8) mma_f8_ss(dtm, ad, bd, idesc, (kb | k) != 0);
        else mma_f16_ss(dtm, ad, bd, idesc, (kb | k) != 0);
      }
      mma_commit(&P.empty[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
    mma_commit(&P.tfull[acc]);
  }
}

__device__ __forceinline__ void teardown(const Pipe& P) {
  using namespace sm100;
  tc_fence_before();
  __syncthreads();
  if ((threadIdx.x >> 5) == 1) tmem_dealloc<TMEM_COLS>(P.tmem);
}

// order-preserving f32 <-> u32 map, so atomicMax on u32 orders signed floats
// (0 = "no bound yet", below every encoded value)
__device__ __forceinline__ uint32_t f2ord(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t u) {
  if (u == 0) return -__int_as_float(0x7f800000);
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}
}  // namespace tc

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn tc_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D map over a row-major [rows x row_elems] fp8/bf16 matrix, box = one
// 128-byte k-block x box_rows rows, 128-byte swizzle
inline int tc_make_map(CUtensorMap* m, void* ptr, bool fp8, int64_t rows, int64_t row_elems,
                       int box_rows) {
  EncodeTiledFn enc = tc_encode_fn();
  ANCKA_REQUIRE(enc != nullptr, ANCKA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int esz = fp8 ? 1 : 2;
  cuuint64_t gdim[2] = {(cuuint64_t)row_elems, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)(row_elems * esz)};
  cuuint32_t box[2] = {(cuuint32_t)(tc::ROW_BYTES / esz), (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, fp8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   ptr, gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  ANCKA_REQUIRE(r == CUDA_SUCCESS, ANCKA_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return ANCKA_OK;
}

// query tiles x key segments: enough CTAs for ~8 waves of 148 SMs
struct TcGrid {
  int q_tiles, key_tiles, nseg, tiles_per_seg;
};
// keys: rows [k0, k1) of the key matrix, k0 a multiple of BN (the query-row
// x key-block products of the multi-GPU ring); key_tiles then counts the
// tiles of the range and kt_base is the first one
struct KeyRange {
  int64_t k0, k1;
};
inline TcGrid tc_grid(int64_t n, int64_t nq, KeyRange kr = {0, -1}) {
  TcGrid g;
  const int64_t k1 = kr.k1 < 0 ? n : kr.k1;
  g.q_tiles = (int)ceil_div(nq, tc::BM);
  g.key_tiles = (int)(ceil_div(k1, tc::BN) - kr.k0 / tc::BN);
  static const int waves = getenv("ANCKA_KNN_WAVES") ? atoi(getenv("ANCKA_KNN_WAVES")) : 8;
  int nseg = (int)ceil_div((int64_t)waves * kNumSMs, g.q_tiles);
  nseg = std::max(1, std::min(nseg, g.key_tiles));
  g.tiles_per_seg = (int)ceil_div(g.key_tiles, nseg);
  g.nseg = (int)ceil_div(g.key_tiles, g.tiles_per_seg);
  return g;
}
}  // namespace ancka
