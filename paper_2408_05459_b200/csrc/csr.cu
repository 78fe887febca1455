// Structural-factor construction on the device (walk.py:38-79, 153-174):
// row normalisation D^-1 A of a CSR matrix with numpy's row-sum order, CSR
// transpose by a stable radix sort of the column keys (rows stay ascending
// inside every transposed row, i.e. scipy's sorted CSR), column scaling, and
// the attribute checks that pick the KNN path (integer-exact levels).
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

namespace ancka {

// rs_i = a[b] + pairwise(a[b+1:e]) -- scipy's csr.sum(axis=1) (see knn_graph.cu);
// out = (1 / rs_i) * a  where rs_i > 0, else 0  (diags(inv) @ a)
__global__ void row_normalize_kernel(const int64_t* __restrict__ rowptr,
                                     const double* __restrict__ vals, int64_t rows,
                                     double* __restrict__ out, double* __restrict__ inv_out) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = rowptr[r], e = rowptr[r + 1];
    double rs = 0.0;
    if (e > b) rs = __dadd_rn(vals[b], np_pairwise_sum(vals + b + 1, e - b - 1));
    const double inv = rs > 0.0 ? 1.0 / rs : 0.0;
    for (int64_t p = b; p < e; ++p) out[p] = __dmul_rn(inv, vals[p]);
    if (inv_out) inv_out[r] = inv;
  }
}

__global__ void col_scale_kernel(const int32_t* __restrict__ colidx, const double* __restrict__ vals,
                                 int64_t nnz, const double* __restrict__ scale,
                                 double* __restrict__ out) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz;
       p += (int64_t)gridDim.x * blockDim.x)
    out[p] = __dmul_rn(scale[colidx[p]], vals[p]);
}

__global__ void row_ids_kernel(const int64_t* __restrict__ rowptr, int64_t rows,
                               int32_t* __restrict__ rid) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x)
    for (int64_t p = rowptr[r]; p < rowptr[r + 1]; ++p) rid[p] = (int32_t)r;
}

__global__ void iota_kernel(int64_t nnz, int64_t* __restrict__ perm) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz;
       p += (int64_t)gridDim.x * blockDim.x)
    perm[p] = p;
}

// sorted column keys -> transposed row pointers; permutation -> row ids, values
__global__ void transpose_finish_kernel(const int32_t* __restrict__ skeys,
                                        const int64_t* __restrict__ perm, int64_t nnz, int64_t cols,
                                        const int32_t* __restrict__ rid,
                                        const double* __restrict__ vals,
                                        int64_t* __restrict__ t_rowptr,
                                        int32_t* __restrict__ t_colidx,
                                        double* __restrict__ t_vals) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p <= nnz;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t prev = p == 0 ? -1 : skeys[p - 1];
    const int64_t cur = p == nnz ? cols : skeys[p];
    for (int64_t c = prev + 1; c <= cur && c <= cols; ++c) t_rowptr[c] = p;
    if (p < nnz) {
      const int64_t src = perm[p];
      t_colidx[p] = rid[src];
      if (t_vals) t_vals[p] = vals[src];
    }
  }
}

// attribute checks: [0] 1 if every entry is an integer, [1] max |x|,
// [2] max row sum of squares (exact for integer data)
__global__ void attr_check_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colidx,
                                  const double* __restrict__ vals, int64_t rows, int64_t ld,
                                  int64_t d, double* __restrict__ out) {
  __shared__ double red[32];
  double mx = 0.0, sq = 0.0;
  int nonint = 0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    if (rowptr) {
      for (int64_t p = rowptr[r]; p < rowptr[r + 1]; ++p) {
        const double v = vals[p];
        nonint |= v != rint(v);
        mx = fmax(mx, fabs(v));
        s += v * v;
      }
    } else {
      for (int64_t c = 0; c < d; ++c) {
        const double v = vals[r * ld + c];
        nonint |= v != rint(v);
        mx = fmax(mx, fabs(v));
        s += v * v;
      }
    }
    sq = fmax(sq, s);
  }
  (void)colidx;
  const int any_nonint = __syncthreads_or(nonint);
  // block max of mx and sq via the generic block reduction on negated sums
  __shared__ double smx, ssq;
  if (threadIdx.x == 0) { smx = 0.0; ssq = 0.0; }
  __syncthreads();
  // f64 max through 64-bit integer atomics (values are >= 0)
  atomicMax(reinterpret_cast<unsigned long long*>(&smx), (unsigned long long)__double_as_longlong(mx));
  atomicMax(reinterpret_cast<unsigned long long*>(&ssq), (unsigned long long)__double_as_longlong(sq));
  __syncthreads();
  (void)red;
  if (threadIdx.x == 0) {
    if (any_nonint) atomicExch(reinterpret_cast<unsigned long long*>(out), (unsigned long long)__double_as_longlong(1.0));
    atomicMax(reinterpret_cast<unsigned long long*>(out + 1), (unsigned long long)__double_as_longlong(smx));
    atomicMax(reinterpret_cast<unsigned long long*>(out + 2), (unsigned long long)__double_as_longlong(ssq));
  }
}

static int grid_for(int64_t items) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(items, 256), 16 * kNumSMs));
}

}  // namespace ancka

using namespace ancka;

extern "C" int ancka_csr_row_normalize(const ancka_csr* A, double* out_values, double* inv_rows,
                                       ancka_stream_t stream) {
  ANCKA_REQUIRE(A && A->rowptr && (A->nnz == 0 || A->values), ANCKA_ERR_ARG, "row_normalize: bad CSR");
  auto st = as_stream(stream);
  row_normalize_kernel<<<grid_for(A->rows), 256, 0, st>>>(
      (const int64_t*)A->rowptr, (const double*)A->values, A->rows, out_values, inv_rows);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

extern "C" int ancka_csr_col_scale(const ancka_csr* A, const double* col_scale, double* out_values,
                                   ancka_stream_t stream) {
  ANCKA_REQUIRE(A && col_scale, ANCKA_ERR_ARG, "col_scale: bad arguments");
  if (A->nnz == 0) return ANCKA_OK;
  auto st = as_stream(stream);
  col_scale_kernel<<<grid_for(A->nnz), 256, 0, st>>>((const int32_t*)A->colidx,
                                                     (const double*)A->values, A->nnz, col_scale,
                                                     out_values);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

static int bits_for_cols(int64_t cols) {
  int b = 1;
  while ((1ll << b) <= cols) ++b;
  return b;
}

static size_t transpose_ws(int64_t rows, int64_t cols, int64_t nnz, size_t* sort_bytes) {
  (void)rows;
  size_t sb = 0;
  cub::DoubleBuffer<int32_t> kb(nullptr, nullptr);
  cub::DoubleBuffer<int64_t> vb(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, sb, kb, vb, (int64_t)std::max<int64_t>(nnz, 1), 0,
                                  bits_for_cols(cols));
  if (sort_bytes) *sort_bytes = sb;
  Carver cv(nullptr, 0);
  cv.take<int32_t>(nnz + 1);   // keys 0
  cv.take<int32_t>(nnz + 1);   // keys 1
  cv.take<int64_t>(nnz + 1);   // perm 0
  cv.take<int64_t>(nnz + 1);   // perm 1
  cv.take<int32_t>(nnz + 1);   // row ids
  cv.take<unsigned char>(sb);
  return cv.used;
}

extern "C" size_t ancka_csr_transpose_workspace_size(int64_t rows, int64_t cols, int64_t nnz) {
  return transpose_ws(rows, cols, nnz, nullptr);
}

extern "C" int ancka_csr_transpose(const ancka_csr* A, int64_t* t_rowptr, int32_t* t_colidx,
                                   double* t_values, void* workspace, size_t workspace_bytes,
                                   ancka_stream_t stream) {
  ANCKA_REQUIRE(A && A->rowptr && t_rowptr && t_colidx, ANCKA_ERR_ARG, "transpose: bad arguments");
  ANCKA_REQUIRE(A->rows < (1ll << 31) && A->cols < (1ll << 31), ANCKA_ERR_UNSUPPORTED,
                "transpose: dimensions exceed int32");
  auto st = as_stream(stream);
  const int64_t nnz = A->nnz;
  size_t sb = 0;
  transpose_ws(A->rows, A->cols, nnz, &sb);
  Carver cv(workspace, workspace_bytes);
  int32_t* k0 = cv.take<int32_t>(nnz + 1);
  int32_t* k1 = cv.take<int32_t>(nnz + 1);
  int64_t* p0 = cv.take<int64_t>(nnz + 1);
  int64_t* p1 = cv.take<int64_t>(nnz + 1);
  int32_t* rid = cv.take<int32_t>(nnz + 1);
  void* tmp = cv.take<unsigned char>(sb);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "transpose: workspace too small");
  if (nnz == 0) {
    ANCKA_CUDA(cudaMemsetAsync(t_rowptr, 0, sizeof(int64_t) * (A->cols + 1), st));
    return ANCKA_OK;
  }
  ANCKA_CUDA(cudaMemcpyAsync(k0, A->colidx, sizeof(int32_t) * nnz, cudaMemcpyDeviceToDevice, st));
  iota_kernel<<<grid_for(nnz), 256, 0, st>>>(nnz, p0);
  ANCKA_LAUNCHED();
  row_ids_kernel<<<grid_for(A->rows), 256, 0, st>>>((const int64_t*)A->rowptr, A->rows, rid);
  ANCKA_LAUNCHED();
  cub::DoubleBuffer<int32_t> kb(k0, k1);
  cub::DoubleBuffer<int64_t> vb(p0, p1);
  ANCKA_CUDA(cub::DeviceRadixSort::SortPairs(tmp, sb, kb, vb, nnz, 0, bits_for_cols(A->cols), st));
  note_launch();
  transpose_finish_kernel<<<grid_for(nnz + 1), 256, 0, st>>>(
      kb.Current(), vb.Current(), nnz, A->cols, rid, (const double*)A->values, t_rowptr, t_colidx,
      t_values);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

extern "C" int ancka_attr_check(const int64_t* rowptr, const double* values, int64_t rows,
                                int64_t ld, int64_t d, double* out3, ancka_stream_t stream) {
  ANCKA_REQUIRE(values && out3, ANCKA_ERR_ARG, "attr_check: bad arguments");
  auto st = as_stream(stream);
  ANCKA_CUDA(cudaMemsetAsync(out3, 0, 3 * sizeof(double), st));
  attr_check_kernel<<<grid_for(rows), 256, 0, st>>>(rowptr, nullptr, values, rows, ld, d, out3);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}

namespace ancka {
// beta_vector (walk.py:47-57) and the self-loop flags (walk.py:123)
__global__ void beta_vector_kernel(const double* __restrict__ degrees,
                                   const uint8_t* __restrict__ knn_zero, int64_t n, double beta,
                                   double* __restrict__ b64, float* __restrict__ b32,
                                   uint8_t* __restrict__ selfloop) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool isolated = degrees[i] == 0.0;
    double b = isolated ? 1.0 : beta;
    if (knn_zero[i]) b = 0.0;
    b64[i] = b;
    b32[i] = (float)b;
    selfloop[i] = (isolated && b == 0.0) ? 1 : 0;
  }
}
}  // namespace ancka

extern "C" int ancka_beta_vector(const double* degrees, const uint8_t* knn_zero_rows, int64_t n,
                                 double beta, double* beta64_out, float* beta32_out,
                                 uint8_t* selfloop_out, ancka_stream_t stream) {
  ANCKA_REQUIRE(n >= 1, ANCKA_ERR_ARG, "beta_vector: empty");
  const int grid = (int)std::min<int64_t>(ceil_div(n, 256), 4 * kNumSMs);
  beta_vector_kernel<<<grid, 256, 0, as_stream(stream)>>>(degrees, knn_zero_rows, n, beta,
                                                          beta64_out, beta32_out, selfloop_out);
  ANCKA_LAUNCHED();
  return ANCKA_OK;
}
