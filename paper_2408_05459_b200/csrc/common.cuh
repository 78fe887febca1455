// Shared helpers for the ANCKA B200 kernels: status/error plumbing, workspace
// carving, deterministic reductions.
#pragma once

#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/ancka_b200.h"

namespace ancka {

void set_error(const char* fmt, ...);
void note_launch();  // counts kernel launches issued by this library

#define ANCKA_CUDA(expr)                                                         \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess) {                                                          \
      ::ancka::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return ANCKA_ERR_CUDA;                                                          \
    }                                                                                 \
  } while (0)

#define ANCKA_LAUNCHED()                                                              \
  do {                                                                                \
    ::ancka::note_launch();                                                           \
    cudaError_t _e = cudaGetLastError();                                              \
    if (_e != cudaSuccess) {                                                          \
      ::ancka::set_error("%s:%d launch: %s", __FILE__, __LINE__, cudaGetErrorString(_e)); \
      return ANCKA_ERR_CUDA;                                                          \
    }                                                                                 \
  } while (0)

#define ANCKA_REQUIRE(cond, code, ...)                                                \
  do {                                                                                \
    if (!(cond)) {                                                                    \
      ::ancka::set_error(__VA_ARGS__);                                                \
      return (code);                                                                  \
    }                                                                                 \
  } while (0)

#define ANCKA_TRY(expr)                                                               \
  do {                                                                                \
    int _s = (expr);                                                                  \
    if (_s != ANCKA_OK) return _s;                                                    \
  } while (0)

inline cudaStream_t as_stream(ancka_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kNumSMs = 148;

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ constexpr size_t align_dev(size_t v) { return (v + 15) & ~size_t(15); }
inline size_t align_up(size_t v, size_t a = 256) { return (v + a - 1) / a * a; }

// Bump allocator over a caller-provided workspace.  With base == nullptr it
// only measures (used by the *_workspace_size functions).
struct Carver {
  char* base;
  size_t used = 0;
  size_t cap;
  Carver(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
  template <typename T>
  T* take(size_t count) {
    size_t off = align_up(used);
    used = off + align_up(count * sizeof(T));
    return base ? reinterpret_cast<T*>(base + off) : nullptr;
  }
  bool ok() const { return base == nullptr || used <= cap; }
};

// ---------------------------------------------------------------- device ---
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (fixed shuffle tree, fixed warp order).  All threads
// of the block must call it; the result is valid in every thread.
template <typename T>
__device__ T block_sum(T v, T* smem /* >= 32 */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) smem[warp] = v;
  __syncthreads();
  T r = 0;
  if (warp == 0) {
    r = lane < nwarps ? smem[lane] : T(0);
    r = warp_sum(r);
    if (lane == 0) smem[0] = r;
  }
  __syncthreads();
  r = smem[0];
  __syncthreads();
  return r;
}

// numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
// pairwise_sum) as used by np.add.reduce / reduceat: r = a[0] + pw(a[1:]).
// Reproducing it makes row sums bit-identical to scipy's csr.sum(axis=1).
template <typename G>
__device__ __forceinline__ double np_pairwise_rec_g(const G& a, int64_t o, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, a(o + i));
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a(o + j);
  int64_t i;
  for (i = 8; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a(o + i + j));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, a(o + i));
  return res;
}

// pairwise_sum over elements a(o .. o+n-1): the recursive halving
//   sum(o, n) = sum(o, n2) + sum(o + n2, n - n2),  n2 = n/2 - (n/2) % 8
// evaluated with an explicit stack; leaves of <= 128 elements use the
// 8-accumulator loop above.
template <typename G>
__device__ inline double np_pairwise_sum_g(const G& a, int64_t n) {
  struct Frame { int64_t o, n; int dep; };
  Frame stack[64];
  double vals[64];
  int vdepth[64];
  int sp = 0, vp = 0;
  stack[sp++] = {0, n, 0};
  while (sp) {
    Frame f = stack[--sp];
    int dep = f.dep;
    if (f.n <= 128) {
      double v = np_pairwise_rec_g(a, f.o, f.n);
      while (vp > 0 && vdepth[vp - 1] == dep) {   // combine with finished left sibling
        v = __dadd_rn(vals[vp - 1], v);
        --vp;
        --dep;
      }
      vals[vp] = v;
      vdepth[vp] = dep;
      ++vp;
    } else {
      int64_t n2 = f.n / 2;
      n2 -= n2 % 8;
      stack[sp++] = {f.o + n2, f.n - n2, f.dep + 1};   // right, evaluated second
      stack[sp++] = {f.o, n2, f.dep + 1};
    }
  }
  return vals[0];
}

__device__ inline double np_pairwise_sum(const double* a, int64_t n) {
  return np_pairwise_sum_g([a](int64_t i) { return a[i]; }, n);
}

}  // namespace ancka
