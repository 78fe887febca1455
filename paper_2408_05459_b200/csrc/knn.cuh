// Internal interface of the KNN kernels.
#pragma once
#include "common.cuh"
#include "knn_tc.cuh"

namespace ancka {
int normalize_rows_f64(const double* X, int64_t n, int64_t d, int64_t ldx, double* xn, int64_t ldn,
                       double* norms, cudaStream_t st);
size_t knn_simt_smem(int K);
int knn_simt(const double* xn, int64_t n, int64_t ldn, const double* norms, int K,
             int64_t q_begin, int64_t q_end, int32_t* ids, double* scores, cudaStream_t st);
size_t knn_simt_list_workspace(int K);
int knn_simt_list(const double* xn, int64_t n, int64_t ldn, const double* norms, int K,
                  int64_t q_begin, const int32_t* qlist, const int* qcount, int32_t* ids,
                  double* scores, void* ws, size_t wsb, cudaStream_t st);

// tcgen05 split-bf16 certified path for real-valued attributes (knn_tc_real.cu)
size_t knn_real_workspace(int64_t n, int64_t d, int K);
int knn_real(const double* X, int64_t n, int64_t d, int64_t ldx, int K, int64_t q_begin,
             int64_t q_end, int32_t* ids, double* scores, void* ws, size_t wsb, cudaStream_t st,
             KeyRange kr = {0, -1});
int knn_real_flag_count(void* ws, size_t wsb, int64_t n, int64_t d, int K, int64_t q_begin,
                        int64_t q_end, int* out_host);
int knn_real_flag_count_async(void* ws, size_t wsb, int64_t n, int64_t d, int K, int64_t q_begin,
                              int64_t q_end, int* out_dev, cudaStream_t st);

// tcgen05 integer-exact path (knn_tc.cu)
size_t knn_tc_workspace(int64_t n, int64_t d, int K);
int knn_tc(const double* X, int64_t n, int64_t d, int64_t ldx, int K, int64_t q_begin,
           int64_t q_end, int32_t* ids, double* scores, void* ws, size_t wsb, cudaStream_t st,
           bool fp8, KeyRange kr = {0, -1});
int knn_tc_csr(const int64_t* indptr, const int32_t* indices, const double* data, int64_t n,
               int64_t d, int K, int64_t q_begin, int64_t q_end, int32_t* ids, double* scores,
               void* ws, size_t wsb, cudaStream_t st, bool fp8, KeyRange kr = {0, -1});
}  // namespace ancka
