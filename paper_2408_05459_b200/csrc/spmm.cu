// Walk-operator application (subsystem 2): CSR SpMM against a dense n x c
// block with the joint-walk mix, self-loops and the MHC / init epilogues
// fused (walk.py:135-190, engine.py:116-117,
// engine.py:296-297).
//
// Mapping: one thread owns (row, V-wide column chunk) and walks the row's
// nonzeros in index order.  Threads of one row read the same index/value
// (broadcast) and gather one contiguous c-wide row of the source per
// nonzero, so a row gather is one coalesced transaction group.  The f64
// instantiation accumulates sequentially with non-contracted mul/add, i.e.
// in exactly scipy csr_matvecs' order, giving bit-identical results.
#include "common.cuh"
#include <cub/device/device_radix_sort.cuh>

#include "spmm.cuh"

namespace ancka {

template <typename T> struct Vec;
template <> struct Vec<float> { using type = float4; static constexpr int W = 4; };
template <> struct Vec<double> { using type = double2; static constexpr int W = 2; };

__device__ __forceinline__ float4 ldv(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ double2 ldv(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }

__device__ __forceinline__ void fma_acc(float4& acc, float w, float4 x) {
  acc.x = fmaf(w, x.x, acc.x); acc.y = fmaf(w, x.y, acc.y);
  acc.z = fmaf(w, x.z, acc.z); acc.w = fmaf(w, x.w, acc.w);
}
// f64: keep the multiply and the add separately rounded (scipy order).
__device__ __forceinline__ void fma_acc(double2& acc, double w, double2 x) {
  acc.x = __dadd_rn(acc.x, __dmul_rn(w, x.x));
  acc.y = __dadd_rn(acc.y, __dmul_rn(w, x.y));
}
__device__ __forceinline__ void add_acc(float4& acc, float4 x) {
  acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
}
__device__ __forceinline__ void add_acc(double2& acc, double2 x) {
  acc.x = __dadd_rn(acc.x, x.x); acc.y = __dadd_rn(acc.y, x.y);
}
__device__ __forceinline__ void div_acc(float4& acc, float d) {
  acc.x /= d; acc.y /= d; acc.z /= d; acc.w /= d;
}
__device__ __forceinline__ void div_acc(double2& acc, double d) {
  acc.x = __ddiv_rn(acc.x, d); acc.y = __ddiv_rn(acc.y, d);
}

template <typename T, typename VT>
__device__ __forceinline__ VT seg_sum(const SegArgs<T>& s, int64_t row, int64_t coloff) {
  VT acc;
  memset(&acc, 0, sizeof(acc));
  if (s.rowptr == nullptr) return acc;
  const int64_t b = __ldg(s.rowptr + row), e = __ldg(s.rowptr + row + 1);
  const T* src = s.src + coloff;
  int64_t p = b;
  // 4-way unrolled: loads issued together, adds kept in order.
  for (; p + 4 <= e; p += 4) {
    int32_t j0 = __ldg(s.colidx + p), j1 = __ldg(s.colidx + p + 1);
    int32_t j2 = __ldg(s.colidx + p + 2), j3 = __ldg(s.colidx + p + 3);
    T w0 = s.values ? __ldg(s.values + p) : T(1);
    T w1 = s.values ? __ldg(s.values + p + 1) : T(1);
    T w2 = s.values ? __ldg(s.values + p + 2) : T(1);
    T w3 = s.values ? __ldg(s.values + p + 3) : T(1);
    VT x0 = ldv(src + (int64_t)j0 * s.ld);
    VT x1 = ldv(src + (int64_t)j1 * s.ld);
    VT x2 = ldv(src + (int64_t)j2 * s.ld);
    VT x3 = ldv(src + (int64_t)j3 * s.ld);
    fma_acc(acc, w0, x0);
    fma_acc(acc, w1, x1);
    fma_acc(acc, w2, x2);
    fma_acc(acc, w3, x3);
  }
  for (; p < e; ++p) {
    int32_t j = __ldg(s.colidx + p);
    T w = s.values ? __ldg(s.values + p) : T(1);
    fma_acc(acc, w, ldv(src + (int64_t)j * s.ld));
  }
  return acc;
}

template <typename T>
__device__ __forceinline__ T comp(const typename Vec<T>::type& v, int i);
template <> __device__ __forceinline__ float comp<float>(const float4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}
template <> __device__ __forceinline__ double comp<double>(const double2& v, int i) {
  return i == 0 ? v.x : v.y;
}
__device__ __forceinline__ void set_comp(float4& v, int i, float x) {
  if (i == 0) v.x = x; else if (i == 1) v.y = x; else if (i == 2) v.z = x; else v.w = x;
}
__device__ __forceinline__ void set_comp(double2& v, int i, double x) {
  if (i == 0) v.x = x; else v.y = x;
}
__device__ __forceinline__ float dmul(float a, float b) { return a * b; }
__device__ __forceinline__ float dadd(float a, float b) { return a + b; }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

// self-loop, beta mix, tag epilogue and store of one (row, chunk)
template <typename T, typename VT>
__device__ __forceinline__ void finish_row(const SpmmArgs<T>& a, int64_t row, int64_t coloff,
                                           VT s, VT k) {
  constexpr int W = Vec<T>::W;
  if (a.selfloop && a.selfloop[row]) add_acc(s, ldv(a.self_src + row * a.self_ld + coloff));
  VT out = s;
  if (a.beta) {
    const T b = __ldg(a.beta + row);
    const T omb = dadd(T(1), -b);   // 1.0 - beta, as (1.0 - op.beta)
#pragma unroll
    for (int i = 0; i < W; ++i)
      set_comp(out, i, dadd(dmul(omb, comp<T>(s, i)), dmul(b, comp<T>(k, i))));
  }
  if (a.tag) {  // out = scale * out + (col == tag[row] ? tagval[col] : 0)
    const int t = __ldg(a.tag + row);
#pragma unroll
    for (int i = 0; i < W; ++i) {
      const int col = (int)coloff + i;
      T v = dmul(a.scale, comp<T>(out, i));
      const T add = (col == t && col < a.c) ? a.tagval[col] : T(0);
      set_comp(out, i, dadd(v, add));
    }
  }
  // padding columns stay exactly zero
#pragma unroll
  for (int i = 0; i < W; ++i)
    if ((int)coloff + i >= a.c) set_comp(out, i, T(0));
  *reinterpret_cast<VT*>(a.out + row * a.ldo + coloff) = out;
}

// A long row summed by a whole warp.  Lanes are (slot, chunk) with `lpr`
// lanes per nonzero (the column chunks, rounded up to a power of two), so the
// lanes reading one gathered row read its consecutive 16-byte chunks
// (coalesced), and 32 / lpr nonzeros are in flight per step.  The slot
// partial sums are combined by a fixed butterfly (deterministic).
__device__ __forceinline__ float4 warp_rows_sum(const SegArgs<float>& s, int64_t row,
                                                int64_t coloff, int slot, int nslot, bool act) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (s.rowptr == nullptr) return acc;
  const int64_t b = __ldg(s.rowptr + row), e = __ldg(s.rowptr + row + 1);
  const float* src = s.src + coloff;
  int64_t p = b + slot;
  for (; p + nslot < e; p += 2 * nslot) {
    const int32_t j0 = __ldg(s.colidx + p), j1 = __ldg(s.colidx + p + nslot);
    const float w0 = s.values ? __ldg(s.values + p) : 1.f;
    const float w1 = s.values ? __ldg(s.values + p + nslot) : 1.f;
    if (act) {
      const float4 x0 = ldv(src + (int64_t)j0 * s.ld), x1 = ldv(src + (int64_t)j1 * s.ld);
      fma_acc(acc, w0, x0);
      fma_acc(acc, w1, x1);
    }
  }
  if (p < e && act)
    fma_acc(acc, s.values ? __ldg(s.values + p) : 1.f, ldv(src + (int64_t)__ldg(s.colidx + p) * s.ld));
  return acc;
}

__device__ __forceinline__ void slot_reduce(float4& v, int lpr) {
  for (int o = lpr; o < 32; o <<= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    v.z += __shfl_xor_sync(0xffffffffu, v.z, o);
    v.w += __shfl_xor_sync(0xffffffffu, v.w, o);
  }
}

template <typename T>
__global__ void __launch_bounds__(256)
spmm_kernel(SpmmArgs<T> a) {
  using VT = typename Vec<T>::type;
  constexpr int W = Vec<T>::W;
  // long rows (KNN / graph hubs) take the first blocks, a warp per row, so
  // the heaviest rows start first instead of forming the tail
  const int64_t long_blocks = ceil_div(a.n_long, (int64_t)(blockDim.x >> 5));
  if constexpr (std::is_same<T, float>::value) {
    if (blockIdx.x < long_blocks) {
      const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
      if (w >= a.n_long) return;
      const int lane = threadIdx.x & 31;
      const int64_t row = a.long_rows[w];
      for (int cb = 0; cb < a.nchunk; cb += 32) {      // column chunks in blocks of <= 32
        const int nc = min(32, a.nchunk - cb);
        int lpr = 1;
        while (lpr < nc) lpr <<= 1;
        const int sub = lane & (lpr - 1), slot = lane / lpr, nslot = 32 / lpr;
        const bool act = sub < nc;
        const int64_t coloff = (int64_t)(cb + sub) * W;
        float4 s = warp_rows_sum(a.s, row, coloff, slot, nslot, act);
        float4 k = make_float4(0.f, 0.f, 0.f, 0.f);
        if (a.beta) k = warp_rows_sum(a.k, row, coloff, slot, nslot, act);
        slot_reduce(s, lpr);
        slot_reduce(k, lpr);
        if (act && slot == 0) finish_row<T, VT>(a, row, coloff, s, k);
      }
      return;
    }
  }
  const int64_t gid = (int64_t)(blockIdx.x - long_blocks) * blockDim.x + threadIdx.x;
  const int64_t slot = gid / a.nchunk;
  if (slot >= a.rows) return;
  // rows in a locality order (grouped by cluster): the rows in flight share
  // their neighbours' gathered rows in L2.  Each row's sum is unchanged.
  const int64_t row = a.order ? (int64_t)__ldg(a.order + slot) : slot;
  if (a.skip && a.skip[row]) return;            // long row: the warp path
  const int chunk = (int)(gid - slot * a.nchunk);
  const int64_t coloff = (int64_t)chunk * W;
  VT s = seg_sum<T, VT>(a.s, row, coloff);
  if (a.nl > 1) {   // multiplex: (sum_l P_l M) / L, layers added in order (walk.py:143-147)
    for (int l = 0; l < a.nl - 1; ++l) add_acc(s, seg_sum<T, VT>(a.lay[l], row, coloff));
    div_acc(s, T(a.nl));
  }
  VT k;
  if (a.beta) k = seg_sum<T, VT>(a.k, row, coloff);
  else memset(&k, 0, sizeof(k));
  finish_row<T, VT>(a, row, coloff, s, k);
}

template <typename T>
int launch_spmm(const SpmmArgs<T>& args, cudaStream_t st) {
  if (args.rows == 0) return ANCKA_OK;
  const int64_t threads = args.rows * args.nchunk;
  const int bs = 256;
  // blocks of 8 long-row warps, then the regular blocks
  const int64_t grid = ceil_div(threads, bs) + ceil_div(args.n_long, (int64_t)(bs / 32));
  ANCKA_REQUIRE(grid < (1ll << 31), ANCKA_ERR_ARG, "spmm grid too large");
  spmm_kernel<T><<<(unsigned)grid, bs, 0, st>>>(args);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

template int launch_spmm<float>(const SpmmArgs<float>&, cudaStream_t);
template int launch_spmm<double>(const SpmmArgs<double>&, cudaStream_t);

// ---------------------------------------------------------------------------
template <typename T>
static SegArgs<T> seg_of(const ancka_csr& m, const T* src, int64_t ld) {
  SegArgs<T> s{};
  if (m.rowptr == nullptr) return s;
  s.rowptr = m.rowptr;
  s.colidx = m.colidx;
  s.values = static_cast<const T*>(m.values);
  s.src = src;
  s.ld = ld;
  return s;
}

template <typename T>
static int set_layers(SpmmArgs<T>& a, int nl, const ancka_csr* layers, const T* src, int64_t ld) {
  ANCKA_REQUIRE(nl >= 1 && nl <= ANCKA_MAX_LAYERS && layers != nullptr, ANCKA_ERR_ARG,
                "multiplex operator needs 1..%d layers (got %d)", ANCKA_MAX_LAYERS, nl);
  a.s = seg_of<T>(layers[0], src, ld);
  for (int l = 1; l < nl; ++l) a.lay[l - 1] = seg_of<T>(layers[l], src, ld);
  a.nl = nl;
  return ANCKA_OK;
}

template <typename T>
int op_apply_t(const ancka_operator* op, const T* Q, int64_t ldq, int c, T* Z, int64_t ldz,
               T* scratch, cudaStream_t st, const EpilogueTag<T>* epi) {
  constexpr int W = Vec<T>::W;
  ANCKA_REQUIRE(ldq % W == 0 && ldz % W == 0 && ldq >= c && ldz >= c, ANCKA_ERR_ARG,
                "op_apply: leading dims must be multiples of %d and >= c", W);
  const int nchunk = (int)ceil_div(c, W);
  SpmmArgs<T> a{};
  a.c = c;
  a.nchunk = nchunk;
  if (op->kind == ANCKA_HYPERGRAPH) {
    ANCKA_REQUIRE(scratch != nullptr, ANCKA_ERR_ARG, "hypergraph apply needs scratch");
    // stage 1: T = P_E Q   (m x c)
    SpmmArgs<T> s1{};
    s1.c = c;
    s1.nchunk = nchunk;
    s1.rows = op->m;
    s1.s = seg_of<T>(op->p_e, Q, ldq);
    s1.out = scratch;
    s1.ldo = ldq;
    ANCKA_TRY(launch_spmm<T>(s1, st));
    a.s = seg_of<T>(op->p_v, scratch, ldq);
  } else if (op->kind == ANCKA_MULTIPLEX) {
    ANCKA_TRY(set_layers<T>(a, op->n_layers, op->layers, Q, ldq));
  } else {
    a.s = seg_of<T>(op->p_n, Q, ldq);
  }
  a.rows = op->n;
  a.selfloop = op->selfloop;
  a.self_src = Q;
  a.self_ld = ldq;
  a.k = seg_of<T>(op->p_k, Q, ldq);
  a.beta = static_cast<const T*>(op->beta);
  a.out = Z;
  a.ldo = ldz;
  if (epi) {
    a.tag = epi->tag;
    a.tagval = epi->tagval;
    a.scale = epi->scale;
  }
  if constexpr (std::is_same<T, float>::value) {
    if (op->split.n_long > 0) {   // long rows by whole warps in the same launch
      a.skip = op->split.is_long;
      a.long_rows = op->split.long_rows;
      a.n_long = op->split.n_long;
    }
    if (op->kind == ANCKA_GRAPH) a.order = op->split.locality_order;
  }
  return launch_spmm<T>(a, st);
}

template <typename T>
int op_apply_struct_t_t(const ancka_operator* op, const T* Q, int64_t ldq, int c, T* Z,
                        int64_t ldz, T* scratch, cudaStream_t st, const EpilogueTag<T>* epi) {
  constexpr int W = Vec<T>::W;
  ANCKA_REQUIRE(ldq % W == 0 && ldz % W == 0, ANCKA_ERR_ARG, "struct_t: bad leading dims");
  const int nchunk = (int)ceil_div(c, W);
  SpmmArgs<T> a{};
  a.c = c;
  a.nchunk = nchunk;
  if (op->kind == ANCKA_HYPERGRAPH) {
    ANCKA_REQUIRE(scratch != nullptr, ANCKA_ERR_ARG, "hypergraph apply needs scratch");
    // (p_e^T @ (p_v^T @ m)): stage A U = P_V^T Q (m x c), stage B P_E^T U
    SpmmArgs<T> s1{};
    s1.c = c;
    s1.nchunk = nchunk;
    s1.rows = op->m;
    s1.s = seg_of<T>(op->t_a, Q, ldq);
    s1.out = scratch;
    s1.ldo = ldq;
    ANCKA_TRY(launch_spmm<T>(s1, st));
    a.s = seg_of<T>(op->t_b, scratch, ldq);
  } else if (op->kind == ANCKA_MULTIPLEX) {
    ANCKA_TRY(set_layers<T>(a, op->n_layers, op->layers_t, Q, ldq));
  } else {
    a.s = seg_of<T>(op->t_a, Q, ldq);
  }
  a.rows = op->n;
  a.selfloop = op->selfloop;
  a.self_src = Q;
  a.self_ld = ldq;
  a.out = Z;
  a.ldo = ldz;
  if (epi) {
    a.tag = epi->tag;
    a.tagval = epi->tagval;
    a.scale = epi->scale;
  }
  return launch_spmm<T>(a, st);
}

template int op_apply_t<float>(const ancka_operator*, const float*, int64_t, int, float*, int64_t,
                               float*, cudaStream_t, const EpilogueTag<float>*);
template int op_apply_t<double>(const ancka_operator*, const double*, int64_t, int, double*,
                                int64_t, double*, cudaStream_t, const EpilogueTag<double>*);
template int op_apply_struct_t_t<float>(const ancka_operator*, const float*, int64_t, int, float*,
                                        int64_t, float*, cudaStream_t, const EpilogueTag<float>*);
template int op_apply_struct_t_t<double>(const ancka_operator*, const double*, int64_t, int,
                                         double*, int64_t, double*, cudaStream_t,
                                         const EpilogueTag<double>*);

}  // namespace ancka

extern "C" int ancka_op_apply(const ancka_operator* op, const void* Q, int64_t ldq, int32_t c,
                              void* Z, int64_t ldz, void* scratch, ancka_stream_t stream) {
  if (!op) { ancka::set_error("null operator"); return ANCKA_ERR_ARG; }
  auto st = ancka::as_stream(stream);
  if (op->dtype == ANCKA_F64)
    return ancka::op_apply_t<double>(op, (const double*)Q, ldq, c, (double*)Z, ldz,
                                     (double*)scratch, st, nullptr);
  return ancka::op_apply_t<float>(op, (const float*)Q, ldq, c, (float*)Z, ldz, (float*)scratch,
                                  st, nullptr);
}

extern "C" int ancka_op_apply_struct_t(const ancka_operator* op, const void* Q, int64_t ldq,
                                       int32_t c, void* Z, int64_t ldz, void* scratch,
                                       ancka_stream_t stream) {
  if (!op) { ancka::set_error("null operator"); return ANCKA_ERR_ARG; }
  auto st = ancka::as_stream(stream);
  if (op->dtype == ANCKA_F64)
    return ancka::op_apply_struct_t_t<double>(op, (const double*)Q, ldq, c, (double*)Z, ldz,
                                              (double*)scratch, st, nullptr);
  return ancka::op_apply_struct_t_t<float>(op, (const float*)Q, ldq, c, (float*)Z, ldz,
                                           (float*)scratch, st, nullptr);
}

// Generic two-segment SpMM (the building block of the row-partitioned
// multi-GPU operator): rows of out = epi( mix( S_rows . S_src (+ self),
// K_rows . K_src ) ).  S/K are row slices whose column indices address the
// full (gathered) sources; `row_offset` maps local row r to the global row
// used for the self-loop source.  beta == NULL: structure only (no K term).
extern "C" int ancka_spmm2(int32_t dtype, int64_t rows, int32_t c, const ancka_csr* S,
                           const void* s_src, int64_t lds, const ancka_csr* K, const void* k_src,
                           int64_t ldk, const void* beta, const uint8_t* selfloop,
                           const void* self_src, int64_t ld_self, int64_t row_offset,
                           const int32_t* tag, const void* tagval, double scale, void* out,
                           int64_t ldo, const int32_t* order, ancka_stream_t stream) {
  using namespace ancka;
  auto st = as_stream(stream);
  auto fill = [&](auto* tp) -> int {
    using T = std::remove_pointer_t<decltype(tp)>;
    constexpr int W = sizeof(T) == 4 ? 4 : 2;
    SpmmArgs<T> a{};
    a.rows = rows;
    a.c = c;
    a.nchunk = (int)ceil_div(c, W);
    if (S && S->rowptr) {
      a.s.rowptr = S->rowptr; a.s.colidx = S->colidx;
      a.s.values = static_cast<const T*>(S->values);
      a.s.src = static_cast<const T*>(s_src); a.s.ld = lds;
    }
    if (K && K->rowptr) {
      a.k.rowptr = K->rowptr; a.k.colidx = K->colidx;
      a.k.values = static_cast<const T*>(K->values);
      a.k.src = static_cast<const T*>(k_src); a.k.ld = ldk;
    }
    a.beta = static_cast<const T*>(beta);
    a.selfloop = selfloop;
    a.self_src = self_src ? static_cast<const T*>(self_src) + row_offset * ld_self : nullptr;
    a.self_ld = ld_self;
    a.tag = tag;
    a.tagval = static_cast<const T*>(tagval);
    a.scale = (T)scale;
    a.out = static_cast<T*>(out);
    a.ldo = ldo;
    if constexpr (sizeof(T) == 4) a.order = order;   // row processing order (sums unchanged)
    return launch_spmm<T>(a, st);
  };
  if (dtype == ANCKA_F64) return fill((double*)nullptr);
  return fill((float*)nullptr);
}

// ---------------------------------------------------------------------------
// rows grouped by label: order = rows sorted by (label, row) (radix sort)
using namespace ancka;

extern "C" size_t ancka_locality_order_workspace_size(int64_t n) {
  size_t bytes = 0;
  cub::DoubleBuffer<int32_t> kb(nullptr, nullptr), vb(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, kb, vb, (int)n, 0, 32);
  return bytes + 3 * (size_t)n * sizeof(int32_t) + 1024;
}

static __global__ void iota_labels_kernel(const int32_t* __restrict__ labels, int64_t n,
                                   int32_t* __restrict__ keys, int32_t* __restrict__ vals) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = labels[i];
    vals[i] = (int32_t)i;
  }
}

extern "C" int ancka_locality_order(const int32_t* labels, int64_t n, int32_t k, int32_t* order_out,
                                    void* workspace, size_t workspace_bytes,
                                    ancka_stream_t stream) {
  ANCKA_REQUIRE(n >= 1 && n < (1ll << 31) && k >= 1, ANCKA_ERR_ARG, "locality_order: bad sizes");
  Carver cv(workspace, workspace_bytes);
  int32_t* k0 = cv.take<int32_t>(n);
  int32_t* k1 = cv.take<int32_t>(n);
  int32_t* v0 = cv.take<int32_t>(n);
  size_t bytes = 0;
  cub::DoubleBuffer<int32_t> kb(k0, k1), vb(v0, order_out);
  ANCKA_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kb, vb, (int)n, 0, 32));
  void* tmp = cv.take<char>(bytes);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "locality_order: workspace too small");
  auto st = as_stream(stream);
  int bits = 1;
  while ((1 << bits) <= k) ++bits;
  iota_labels_kernel<<<(int)std::min<int64_t>(ceil_div(n, 256), 16 * kNumSMs), 256, 0, st>>>(
      labels, n, k0, v0);
  ANCKA_LAUNCHED();
  ANCKA_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, kb, vb, (int)n, 0, bits, st));
  if (vb.Current() != order_out)
    ANCKA_CUDA(cudaMemcpyAsync(order_out, vb.Current(), sizeof(int32_t) * n,
                               cudaMemcpyDeviceToDevice, st));
  return ANCKA_OK;
}
