// Multi-hop conductance (engine.py:291-299) and greedy BCM initialisation
// (engine.py:87-127) on top of the fused SpMM epilogues.
#include <climits>

#include "common.cuh"
#include "spmm.cuh"

namespace ancka {

__global__ void cluster_sizes_kernel(const int32_t* __restrict__ labels, int64_t n, int k,
                                     int64_t* __restrict__ sizes) {
  extern __shared__ unsigned long long hist[];
  for (int c = threadIdx.x; c < k; c += blockDim.x) hist[c] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int l = labels[i];
    if (l >= 0 && l < k) atomicAdd(&hist[l], 1ull);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x)
    if (hist[c]) atomicAdd(reinterpret_cast<unsigned long long*>(sizes + c), hist[c]);
}

int cluster_sizes(const int32_t* labels, int64_t n, int k, int64_t* sizes, cudaStream_t st) {
  ANCKA_CUDA(cudaMemsetAsync(sizes, 0, sizeof(int64_t) * k, st));
  const int grid = (int)std::min<int64_t>(ceil_div(n, 256), 2 * kNumSMs);
  cluster_sizes_kernel<<<std::max(grid, 1), 256, k * sizeof(unsigned long long), st>>>(labels, n, k, sizes);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

// tagval[c] = alpha * (1 / sqrt(size_c))   (f0 = alpha * yhat, engine.py:294)
template <typename T>
__global__ void mhc_tagval_kernel(const int64_t* __restrict__ sizes, int k, double alpha,
                                  T* __restrict__ tagval, double* __restrict__ yhat) {
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    const double y = sizes[c] > 0 ? 1.0 / sqrt((double)sizes[c]) : 0.0;
    yhat[c] = y;
    tagval[c] = (T)(alpha * y);
  }
}

// F[i, c] = (c == label[i]) ? tagval[c] : 0
template <typename T>
__global__ void fill_tag_kernel(const int32_t* __restrict__ tag, int64_t n, int64_t ld, int c,
                                const T* __restrict__ tagval, T* __restrict__ F) {
  const int64_t total = n * ld;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / ld;
    const int col = (int)(e - i * ld);
    const int t = tag[i];
    F[e] = (col < c && col == t) ? tagval[col] : T(0);
  }
}

// psi partials: sum_i yhat[lab_i] * F[i, lab_i]
template <typename T>
__global__ void __launch_bounds__(256)
mhc_trace_kernel(const T* __restrict__ F, int64_t n, int64_t ld, const int32_t* __restrict__ lab,
                 const double* __restrict__ yhat, double* __restrict__ partial) {
  __shared__ double red[32];
  const int64_t rpb = ceil_div(n, gridDim.x);
  const int64_t r0 = (int64_t)blockIdx.x * rpb, r1 = lmin(n, r0 + rpb);
  double s = 0.0;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    const int l = lab[i];
    s += yhat[l] * (double)F[i * ld + l];
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void mhc_finish_kernel(const double* __restrict__ partial, int nblk,
                                  const int64_t* __restrict__ sizes, int k,
                                  double* __restrict__ phi) {
  __shared__ double red[32];
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) s += partial[b];
  s = block_sum(s, red);
  if (threadIdx.x == 0) {
    bool empty = false;
    for (int c = 0; c < k; ++c) empty |= sizes[c] == 0;
    *phi = empty ? nan("") : 1.0 - s / (double)k;
  }
}

constexpr int kTraceBlocks = 2 * kNumSMs;

template <typename T>
struct MhcWs {
  T* F0;
  T* F1;
  T* scratch;
  T* tagval;
  double* yhat;
  double* partial;
  unsigned long long* hist;
};

// one cooperative kernel for narrow f32 blocks on graph / hypergraph walks
template <typename T>
static bool mhc_fused(const ancka_operator* op, int k) {
  static const bool off = getenv("ANCKA_MHC_UNFUSED") != nullptr;
  return sizeof(T) == 4 && k <= 8 && op->kind != ANCKA_MULTIPLEX && !off;
}

template <typename T>
static int64_t mhc_ld(const ancka_operator* op, int k) {
  const int W = sizeof(T) == 4 ? 4 : 2;
  return mhc_fused<T>(op, k) ? 8 : (k + W - 1) / W * W;
}

template <typename T>
static void carve_mhc(Carver& cv, MhcWs<T>& w, const ancka_operator* op, int k) {
  const int64_t ld = mhc_ld<T>(op, k);
  w.F0 = cv.take<T>((size_t)op->n * ld);
  w.F1 = cv.take<T>((size_t)op->n * ld);
  w.scratch = cv.take<T>(op->kind == ANCKA_HYPERGRAPH ? (size_t)op->m * ld : 1);
  w.tagval = cv.take<T>(k);
  w.yhat = cv.take<double>(k);
  w.partial = cv.take<double>(std::max(kTraceBlocks, mhc_fused_grid_cap()));
  w.hist = cv.take<unsigned long long>(k);
}

template <typename T>
static int mhc_t(const ancka_operator* op, const int32_t* labels, int k, double alpha, int gamma,
                 double* phi, int64_t* sizes, void* ws, size_t wsb, cudaStream_t st) {
  Carver cv(ws, wsb);
  MhcWs<T> w;
  carve_mhc<T>(cv, w, op, k);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "mhc: workspace too small");
  const int64_t ld = mhc_ld<T>(op, k);
  const int64_t n = op->n;
  if constexpr (sizeof(T) == 4) {
    if (mhc_fused<T>(op, k))
      return mhc_fused_f32(op, labels, k, alpha, gamma, phi, sizes, w.F0, w.F1, w.scratch, w.hist,
                           w.partial, st);
  }
  ANCKA_TRY(cluster_sizes(labels, n, k, sizes, st));
  mhc_tagval_kernel<T><<<1, 256, 0, st>>>(sizes, k, alpha, w.tagval, w.yhat);
  ANCKA_LAUNCHED();
  const int fg = (int)std::min<int64_t>(ceil_div(n * ld, 256), 16 * kNumSMs);
  fill_tag_kernel<T><<<std::max(fg, 1), 256, 0, st>>>(labels, n, ld, k, w.tagval, w.F0);
  ANCKA_LAUNCHED();
  EpilogueTag<T> epi{labels, w.tagval, (T)(1.0 - alpha)};
  T* cur = w.F0;
  T* nxt = w.F1;
  for (int g = 0; g < gamma; ++g) {
    ANCKA_TRY(op_apply_t<T>(op, cur, ld, k, nxt, ld, w.scratch, st, &epi));
    std::swap(cur, nxt);
  }
  mhc_trace_kernel<T><<<kTraceBlocks, 256, 0, st>>>(cur, n, ld, labels, w.yhat, w.partial);
  ANCKA_LAUNCHED();
  mhc_finish_kernel<<<1, 256, 0, st>>>(w.partial, kTraceBlocks, sizes, k, phi);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

// ------------------------------------------------------------------ init ---
__global__ void center_of_kernel(const int64_t* __restrict__ centers, int k, int64_t n,
                                 int32_t* __restrict__ center_of, double* __restrict__ tagval,
                                 double alpha) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    center_of[i] = -1;
  __syncthreads();
  if (blockIdx.x == 0)
    for (int c = threadIdx.x; c < k; c += blockDim.x) tagval[c] = alpha;  // pi0 = alpha * z0
}

__global__ void center_set_kernel(const int64_t* __restrict__ centers, int k,
                                  int32_t* __restrict__ center_of) {
  for (int c = threadIdx.x; c < k; c += blockDim.x) center_of[centers[c]] = c;
}

// first-max argmax over the k centres (np.argmax(pi, axis=0), engine.py:119)
__global__ void argmax_rows_kernel(const double* __restrict__ P, int64_t n, int64_t ld, int k,
                                   int32_t* __restrict__ labels) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double* r = P + i * ld;
    double best = r[0];
    int arg = 0;
    for (int c = 1; c < k; ++c)
      if (r[c] > best) { best = r[c]; arg = c; }
    labels[i] = arg;
  }
}

struct InitWs {
  double* P0;
  double* P1;
  double* scratch;
  double* tagval;
  int32_t* center_of;
};

static void carve_init(Carver& cv, InitWs& w, const ancka_operator* op, int k) {
  const int64_t ld = (k + 1) / 2 * 2;
  w.P0 = cv.take<double>((size_t)op->n * ld);
  w.P1 = cv.take<double>((size_t)op->n * ld);
  w.scratch = cv.take<double>(op->kind == ANCKA_HYPERGRAPH ? (size_t)op->m * ld : 1);
  w.tagval = cv.take<double>(k);
  w.center_of = cv.take<int32_t>(op->n);
}

}  // namespace ancka

using namespace ancka;

namespace ancka {
// Q0 = [1/sqrt(n) | Yhat0] (engine.py:368-371): row i gets first_col in
// column 0 and 1/sqrt(|C_l|) in column l+1 (l = label, l + 1 < c); every other
// entry of the n x ld block is zero
__global__ void bcm_block_kernel(const int32_t* __restrict__ labels, int64_t n, int c,
                                 const int64_t* __restrict__ sizes, double first_col,
                                 double* __restrict__ q, int64_t ldq) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * ldq;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / ldq;
    const int j = (int)(e - i * ldq);
    double v = 0.0;
    if (j == 0) {
      v = first_col;
    } else if (j < c) {
      const int l = labels[i];
      if (l + 1 == j && sizes[l] > 0) v = 1.0 / sqrt((double)sizes[l]);
    }
    q[e] = v;
  }
}
}  // namespace ancka

extern "C" int ancka_bcm_block(const int32_t* labels, int64_t n, int32_t c, const int64_t* sizes,
                               double first_col, double* q, int64_t ldq, ancka_stream_t stream) {
  ANCKA_REQUIRE(n >= 1 && c >= 1 && ldq >= c, ANCKA_ERR_ARG, "bcm_block: bad sizes");
  const int grid = (int)std::min<int64_t>(ceil_div(n * ldq, 256), 16 * kNumSMs);
  bcm_block_kernel<<<grid, 256, 0, as_stream(stream)>>>(labels, n, c, sizes, first_col, q, ldq);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

extern "C" int ancka_cluster_sizes(const int32_t* labels, int64_t n, int32_t k, int64_t* sizes_out,
                                   ancka_stream_t stream) {
  return cluster_sizes(labels, n, k, sizes_out, as_stream(stream));
}

extern "C" size_t ancka_mhc_workspace_size(const ancka_operator* op, int32_t k) {
  Carver cv(nullptr, 0);
  if (op->dtype == ANCKA_F64) { MhcWs<double> w; carve_mhc<double>(cv, w, op, k); }
  else { MhcWs<float> w; carve_mhc<float>(cv, w, op, k); }
  return cv.used;
}

extern "C" int ancka_mhc(const ancka_operator* op, const int32_t* labels, int32_t k, double alpha,
                         int32_t gamma, double* phi_out, int64_t* sizes_out, void* workspace,
                         size_t workspace_bytes, ancka_stream_t stream) {
  ANCKA_REQUIRE(op && k >= 1, ANCKA_ERR_ARG, "mhc: bad arguments");
  auto st = as_stream(stream);
  if (op->dtype == ANCKA_F64)
    return mhc_t<double>(op, labels, k, alpha, gamma, phi_out, sizes_out, workspace,
                         workspace_bytes, st);
  return mhc_t<float>(op, labels, k, alpha, gamma, phi_out, sizes_out, workspace,
                      workspace_bytes, st);
}

extern "C" size_t ancka_init_workspace_size(const ancka_operator* op, int32_t k) {
  Carver cv(nullptr, 0);
  InitWs w;
  carve_init(cv, w, op, k);
  return cv.used;
}

extern "C" int ancka_init_bcm(const ancka_operator* op64, const int64_t* centers, int32_t k,
                              int32_t t_i, double alpha, int32_t* labels_out, void* workspace,
                              size_t workspace_bytes, ancka_stream_t stream) {
  ANCKA_REQUIRE(op64 && op64->dtype == ANCKA_F64, ANCKA_ERR_ARG, "init_bcm needs the f64 operator");
  Carver cv(workspace, workspace_bytes);
  InitWs w;
  carve_init(cv, w, op64, k);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "init_bcm: workspace too small");
  auto st = as_stream(stream);
  const int64_t n = op64->n;
  const int64_t ld = (k + 1) / 2 * 2;
  const int g = (int)std::min<int64_t>(ceil_div(n, 256), 8 * kNumSMs);
  center_of_kernel<<<std::max(g, 1), 256, 0, st>>>(centers, k, n, w.center_of, w.tagval, alpha);
  ANCKA_LAUNCHED();
  center_set_kernel<<<1, 256, 0, st>>>(centers, k, w.center_of);
  ANCKA_LAUNCHED();
  const int fg = (int)std::min<int64_t>(ceil_div(n * ld, 256), 16 * kNumSMs);
  fill_tag_kernel<double><<<std::max(fg, 1), 256, 0, st>>>(w.center_of, n, ld, k, w.tagval, w.P0);
  ANCKA_LAUNCHED();
  EpilogueTag<double> epi{w.center_of, w.tagval, 1.0 - alpha};
  double* cur = w.P0;
  double* nxt = w.P1;
  for (int t = 0; t < t_i; ++t) {
    ANCKA_TRY(op_apply_struct_t_t<double>(op64, cur, ld, k, nxt, ld, w.scratch, st, &epi));
    std::swap(cur, nxt);
  }
  argmax_rows_kernel<<<std::max(g, 1), 256, 0, st>>>(cur, n, ld, k, labels_out);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

// ------------------------------------------------------- same partition ---
// a and b (labels in [0, k)) describe the same partition up to relabelling
// iff every cluster of a maps to one cluster of b (min == max of b over its
// rows) and the map is injective; phi is a function of the partition (the
// walk's columns and the trace's per-row terms do not depend on the ids), so
// the MHC of a relabelled partition repeats the previous value bit for bit.
namespace {
constexpr int kSameSmemK = 4096;

__global__ void same_init_kernel(int32_t* __restrict__ mn, int32_t* __restrict__ mx, int k) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < k; c += gridDim.x * blockDim.x) {
    mn[c] = INT_MAX;
    mx[c] = INT_MIN;
  }
}

__global__ void __launch_bounds__(256)
same_minmax_kernel(const int32_t* __restrict__ a, const int32_t* __restrict__ b, int64_t n, int k,
                   int32_t* __restrict__ mn, int32_t* __restrict__ mx) {
  __shared__ int32_t smn[kSameSmemK], smx[kSameSmemK];
  const bool loc = k <= kSameSmemK;
  if (loc)
    for (int c = threadIdx.x; c < k; c += blockDim.x) { smn[c] = INT_MAX; smx[c] = INT_MIN; }
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t x = a[i], y = b[i];
    if (x < 0 || x >= k) { atomicMin(mn, INT_MIN); continue; }   // out of range: never "same"
    if (loc) { atomicMin(&smn[x], y); atomicMax(&smx[x], y); }
    else { atomicMin(&mn[x], y); atomicMax(&mx[x], y); }
  }
  __syncthreads();
  if (loc)
    for (int c = threadIdx.x; c < k; c += blockDim.x)
      if (smx[c] != INT_MIN) { atomicMin(&mn[c], smn[c]); atomicMax(&mx[c], smx[c]); }
}

__global__ void __launch_bounds__(256)
same_finish_kernel(const int32_t* __restrict__ mn, const int32_t* __restrict__ mx, int k,
                   int32_t* __restrict__ same) {
  __shared__ unsigned bits[kSameSmemK / 32];
  __shared__ int ok;
  if (threadIdx.x == 0) ok = k <= kSameSmemK;
  for (int w = threadIdx.x; w < kSameSmemK / 32; w += blockDim.x) bits[w] = 0u;
  __syncthreads();
  if (ok)
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
      const int32_t lo = mn[c], hi = mx[c];
      if (lo != hi || lo < 0 || lo >= k) { ok = 0; continue; }   // split, empty or out of range
      if (atomicOr(&bits[lo >> 5], 1u << (lo & 31)) & (1u << (lo & 31))) ok = 0;   // not injective
    }
  __syncthreads();
  if (threadIdx.x == 0) *same = ok;
}
}  // namespace

extern "C" int ancka_same_partition(const int32_t* a, const int32_t* b, int64_t n, int32_t k,
                                    int32_t* minmax_ws, int32_t* same_out, ancka_stream_t stream) {
  ANCKA_REQUIRE(k >= 1 && n >= 0, ANCKA_ERR_ARG, "same_partition: n=%lld k=%d", (long long)n, k);
  auto st = as_stream(stream);
  int32_t* mn = minmax_ws;
  int32_t* mx = minmax_ws + k;
  same_init_kernel<<<(int)std::min<int64_t>(ceil_div(k, 256), 64), 256, 0, st>>>(mn, mx, k);
  ANCKA_LAUNCHED();
  if (n > 0) {
    same_minmax_kernel<<<(int)std::min<int64_t>(ceil_div(n, 256), 2 * kNumSMs), 256, 0, st>>>(
        a, b, n, k, mn, mx);
    ANCKA_LAUNCHED();
  }
  same_finish_kernel<<<1, 256, 0, st>>>(mn, mx, k, same_out);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}
