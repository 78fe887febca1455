// Tensor-pipe peak microbenchmark (roofline denominators):
// one CTA per SM issues back-to-back tcgen05.mma (M = 128, N = 256, the KNN
// kernels' tile) on operand tiles resident in shared memory (SW128 K-major,
// the same descriptors as the KNN kernels), accumulating into one TMEM
// buffer, with one commit per 4 k-steps so the issue queue never drains.
// fmt 0: kind::f8f6f4 (e4m3, K = 32 per instruction), 1: kind::f16 (bf16,
// K = 16).  Reports FLOP = 2 x 128 x 256 x K per instruction.  No data
// leaves TMEM; the operands are zeros (the pipe's rate is data-independent).
#include "common.cuh"
#include "sm100.cuh"

namespace ancka {
namespace {
using namespace sm100;

constexpr int kPM = 128, kPN = 256;
constexpr int kPA = kPM * 128, kPB = kPN * 128;   // one 128-byte K block per row

__global__ void __launch_bounds__(128, 1) tc_peak_kernel(int fmt, int iters, long long* cycles) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = base;
  unsigned char* sB = base + kPA;
  __shared__ uint64_t done;
  __shared__ uint32_t tmem;
  for (int e = threadIdx.x; e < (kPA + kPB) / 16; e += blockDim.x)
    reinterpret_cast<uint4*>(base)[e] = make_uint4(0u, 0u, 0u, 0u);
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  if ((threadIdx.x >> 5) == 0) tmem_alloc<256>(&tmem);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = tmem;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    const uint32_t a_addr = smem_u32(sA), b_addr = smem_u32(sB);
    const uint32_t idesc = fmt == 0 ? make_idesc(0u, kPM, kPN) : make_idesc(1u, kPM, kPN);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t ad = sw128_kmajor_desc(a_addr + k * 32);
        const uint64_t bd = sw128_kmajor_desc(b_addr + k * 32);
        if (fmt == 0) mma_f8_ss(d, ad, bd, idesc, (it | k) != 0);
        else mma_f16_ss(d, ad, bd, idesc, (it | k) != 0);
      }
    }
    mma_commit(&done);
  }
  mbar_wait(&done, 0);
  const long long t1 = clock64();
  tc_fence_before();
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) tmem_dealloc<256>(d);
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}
}  // namespace
}  // namespace ancka

using namespace ancka;

/* Runs the microbenchmark on all SMs: flop_out = FLOP issued, *ms_out =
 * kernel time measured with events on `stream` (synchronises). */
extern "C" int ancka_tc_peak(int32_t fmt, int32_t iters, double* flop_out, double* ms_out,
                             long long* cycles, ancka_stream_t stream) {
  ANCKA_REQUIRE(fmt == 0 || fmt == 1, ANCKA_ERR_ARG, "tc_peak: fmt 0 (fp8) or 1 (bf16)");
  cudaStream_t st = as_stream(stream);
  const size_t smem = kPA + kPB + 1024;
  ANCKA_CUDA(cudaFuncSetAttribute(tc_peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t a, b;
  ANCKA_CUDA(cudaEventCreate(&a));
  ANCKA_CUDA(cudaEventCreate(&b));
  ANCKA_CUDA(cudaEventRecord(a, st));
  tc_peak_kernel<<<kNumSMs, 128, smem, st>>>(fmt, iters, cycles);
  ANCKA_LAUNCHED();
  ANCKA_CUDA(cudaEventRecord(b, st));
  ANCKA_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  ANCKA_CUDA(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  const double kk = fmt == 0 ? 32.0 : 16.0;
  *flop_out = 2.0 * kPM * kPN * kk * 4.0 * (double)iters * kNumSMs;
  *ms_out = ms;
  return ANCKA_OK;
}

// L2 read-bandwidth microbenchmark (the SpMM gather's roofline): every
// thread walks rows of a table that fits L2, reading one float4 per row
// chunk -- sequential (row = thread index stride) or gathered (row =
// hash of the index, rows of `row_floats` floats as the SpMM's Q rows).
namespace ancka {
namespace {
__global__ void __launch_bounds__(256) l2_read_kernel(const float4* __restrict__ tab, int64_t rows,
                                                      int row_f4, int iters, int gather,
                                                      float* __restrict__ sink) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const uint32_t nthreads = gridDim.x * blockDim.x;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t total = (uint32_t)(rows * row_f4);
  const uint32_t mask = (uint32_t)rows - 1u;     // rows: a power of two
  for (int it = 0; it < iters; ++it) {
    uint32_t e = tid;
    for (; e + 3 * nthreads < total; e += 4 * nthreads) {   // four loads in flight
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t ee = e + u * nthreads;
        uint32_t r = ee / (uint32_t)row_f4;
        const uint32_t c = ee - r * (uint32_t)row_f4;
        if (gather) r = ((r + (uint32_t)it) * 2654435761u) & mask;
        v[u] = __ldcg(tab + (size_t)r * row_f4 + c);           // L2, not L1
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
    }
    for (; e < total; e += nthreads) {
      uint32_t r = e / (uint32_t)row_f4;
      const uint32_t c = e - r * (uint32_t)row_f4;
      if (gather) r = ((r + (uint32_t)it) * 2654435761u) & mask;
      const float4 v = __ldcg(tab + (size_t)r * row_f4 + c);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  if (acc.x + acc.y + acc.z + acc.w == 1.2345f) sink[0] = acc.x;   // keep the loads
}
}  // namespace
}  // namespace ancka

/* L2 read bandwidth: bytes read and event-timed ms for `iters` sweeps over a
 * rows x row_floats f32 table (device memory, fits L2), sequential or
 * gathered rows. */
extern "C" int ancka_l2_read(const float* table, int64_t rows, int32_t row_floats, int32_t iters,
                             int32_t gather, float* sink, double* bytes_out, double* ms_out,
                             ancka_stream_t stream) {
  ANCKA_REQUIRE(row_floats % 4 == 0 && rows > 0 && (rows & (rows - 1)) == 0, ANCKA_ERR_ARG,
                "l2_read: row_floats a multiple of 4, rows a power of two");
  cudaStream_t st = as_stream(stream);
  cudaEvent_t a, b;
  ANCKA_CUDA(cudaEventCreate(&a));
  ANCKA_CUDA(cudaEventCreate(&b));
  ANCKA_CUDA(cudaEventRecord(a, st));
  l2_read_kernel<<<kNumSMs * 8, 256, 0, st>>>(reinterpret_cast<const float4*>(table), rows,
                                             row_floats / 4, iters, gather, sink);
  ANCKA_LAUNCHED();
  ANCKA_CUDA(cudaEventRecord(b, st));
  ANCKA_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  ANCKA_CUDA(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *bytes_out = 4.0 * (double)rows * row_floats * iters;
  *ms_out = ms;
  return ANCKA_OK;
}
