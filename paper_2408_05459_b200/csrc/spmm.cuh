// Internal interface of the walk-operator SpMM (spmm.cu).
#pragma once
#include <type_traits>

#include "common.cuh"

namespace ancka {

template <typename T>
struct SegArgs {
  const int64_t* rowptr = nullptr;  // nullptr: empty segment
  const int32_t* colidx = nullptr;
  const T* values = nullptr;        // nullptr: unit weights
  const T* src = nullptr;           // gathered block
  int64_t ld = 0;
};

// out[row] = epilogue( mix( s_row (+ self), k_row ) )
template <typename T>
struct SpmmArgs {
  int64_t rows = 0;
  int c = 0, nchunk = 0;
  SegArgs<T> s, k;
  int nl = 0;                       // multiplex: layers (s = layer 0, lay[] = 1..nl-1)
  SegArgs<T> lay[ANCKA_MAX_LAYERS - 1];
  const uint8_t* selfloop = nullptr;
  const T* self_src = nullptr;
  int64_t self_ld = 0;
  const T* beta = nullptr;          // nullptr: no mix (structure only)
  const uint8_t* skip = nullptr;    // long rows: handled by the warp path below
  const int32_t* order = nullptr;   // regular rows processed in this order (locality)
  const int32_t* long_rows = nullptr;  // f32: rows done by a warp per (row, column chunk)
  int64_t n_long = 0;
  const int32_t* tag = nullptr;     // epilogue: out = scale*out + (col==tag ? tagval[col] : 0)
  const T* tagval = nullptr;
  T scale = T(1);
  T* out = nullptr;
  int64_t ldo = 0;
};

template <typename T>
struct EpilogueTag {
  const int32_t* tag;
  const T* tagval;
  T scale;
};

template <typename T> int launch_spmm(const SpmmArgs<T>& args, cudaStream_t st);

template <typename T>
int op_apply_t(const ancka_operator* op, const T* Q, int64_t ldq, int c, T* Z, int64_t ldz,
               T* scratch, cudaStream_t st, const EpilogueTag<T>* epi);
template <typename T>
int op_apply_struct_t_t(const ancka_operator* op, const T* Q, int64_t ldq, int c, T* Z,
                        int64_t ldz, T* scratch, cudaStream_t st, const EpilogueTag<T>* epi);

// fused multi-hop conductance for k <= 8 (orth_fused.cu); F0/F1 n x 8, T m x 8
constexpr int mhc_fused_grid_cap() { return 4 * kNumSMs; }
int mhc_fused_f32(const ancka_operator* op, const int32_t* labels, int k, double alpha, int gamma,
                  double* phi, int64_t* sizes, float* F0, float* F1, float* T,
                  unsigned long long* hist, double* part, cudaStream_t st);

}  // namespace ancka
