// C-ABI entry points that are not owned by a subsystem file, plus the KNN
// dispatcher (tensor-core integer-exact path vs f64 CUDA-core path).
#include <atomic>
#include <cstdarg>

#include "common.cuh"
#include "knn.cuh"

namespace ancka {

static thread_local char g_err[1024] = "";
static std::atomic<long long> g_launches{0};

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

}  // namespace ancka

using namespace ancka;

extern "C" const char* ancka_last_error(void) { return g_err; }
extern "C" int ancka_abi_version(void) { return ANCKA_ABI_VERSION; }
extern "C" int64_t ancka_launch_count(void) { return g_launches.load(); }

extern "C" int ancka_device_check(void) {
  int dev = 0;
  ANCKA_CUDA(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  ANCKA_CUDA(cudaGetDeviceProperties(&prop, dev));
  ANCKA_REQUIRE(prop.major == 10, ANCKA_ERR_UNSUPPORTED,
                "device %s is sm_%d%d; this library is built for sm_100a only", prop.name,
                prop.major, prop.minor);
  return ANCKA_OK;
}

static void carve_knn_simt(Carver& cv, int64_t n, int64_t d, double** xn, double** norms,
                           int64_t* ldn) {
  *ldn = (d + 15) / 16 * 16;
  *xn = cv.take<double>((size_t)n * *ldn);
  *norms = cv.take<double>(n);
}

extern "C" size_t ancka_knn_workspace_size(int64_t n, int64_t d, int32_t K, int32_t integer_exact) {
  if (integer_exact > 0) return knn_tc_workspace(n, d, K);
  if (integer_exact == 0) return knn_real_workspace(n, d, K);
  Carver cv(nullptr, 0);
  double *xn, *nr;
  int64_t ldn;
  carve_knn_simt(cv, n, d, &xn, &nr, &ldn);
  return cv.used;
}

extern "C" int ancka_knn_exact(const double* X, int64_t n, int64_t d, int64_t ldx, int32_t K,
                               int32_t integer_exact, int64_t q_begin, int64_t q_end, int32_t* ids,
                               double* scores, void* workspace, size_t workspace_bytes,
                               ancka_stream_t stream) {
  ANCKA_REQUIRE(K < n, ANCKA_ERR_NETWORK, "K=%d must be smaller than n=%lld", K, (long long)n);
  ANCKA_REQUIRE(K >= 1 && d >= 1, ANCKA_ERR_ARG, "knn: bad sizes");
  auto st = as_stream(stream);
  ANCKA_REQUIRE(0 <= q_begin && q_begin < q_end && q_end <= n, ANCKA_ERR_ARG, "knn: bad query range");
  if (integer_exact > 0)
    return knn_tc(X, n, d, ldx, K, q_begin, q_end, ids, scores, workspace, workspace_bytes, st,
                  integer_exact == 2);
  if (integer_exact == 0)
    return knn_real(X, n, d, ldx, K, q_begin, q_end, ids, scores, workspace, workspace_bytes, st);
  Carver cv(workspace, workspace_bytes);
  double *xn, *nr;
  int64_t ldn;
  carve_knn_simt(cv, n, d, &xn, &nr, &ldn);
  ANCKA_REQUIRE(cv.ok(), ANCKA_ERR_ARG, "knn: workspace too small");
  ANCKA_TRY(normalize_rows_f64(X, n, d, ldx, xn, ldn, nr, st));
  return knn_simt(xn, n, ldn, nr, K, q_begin, q_end, ids, scores, st);
}

extern "C" int ancka_knn_exact_csr(const int64_t* indptr, const int32_t* indices, const double* data,
                                   int64_t n, int64_t d, int32_t K, int32_t integer_exact,
                                   int64_t q_begin, int64_t q_end, int32_t* ids, double* scores,
                                   void* workspace, size_t workspace_bytes, ancka_stream_t stream) {
  ANCKA_REQUIRE(K < n, ANCKA_ERR_NETWORK, "K=%d must be smaller than n=%lld", K, (long long)n);
  ANCKA_REQUIRE(integer_exact == 1 || integer_exact == 2, ANCKA_ERR_UNSUPPORTED,
                "CSR attributes are supported on the integer-exact tensor-core path only");
  ANCKA_REQUIRE(0 <= q_begin && q_begin < q_end && q_end <= n, ANCKA_ERR_ARG, "knn: bad query range");
  return knn_tc_csr(indptr, indices, data, n, d, K, q_begin, q_end, ids, scores, workspace,
                    workspace_bytes, as_stream(stream), integer_exact == 2);
}

// Query rows [q_begin, q_end) against the key rows [k0, k1) only (k0 a
// multiple of 256): the own-rows x visiting-block products of the multi-GPU
// key ring.  Rows the real-valued certificate rejects are rescanned against
// all n keys (callers merge lists with de-duplication).
extern "C" int ancka_knn_exact_keys(const double* X, int64_t n, int64_t d, int64_t ldx, int32_t K,
                                    int32_t integer_exact, int64_t q_begin, int64_t q_end,
                                    int64_t k0, int64_t k1, int32_t* ids, double* scores,
                                    void* workspace, size_t workspace_bytes,
                                    ancka_stream_t stream) {
  ANCKA_REQUIRE(K >= 1 && d >= 1 && K < n, ANCKA_ERR_ARG, "knn: bad sizes");
  ANCKA_REQUIRE(0 <= q_begin && q_begin < q_end && q_end <= n, ANCKA_ERR_ARG, "knn: bad query range");
  ANCKA_REQUIRE(k0 >= 0 && k0 % 256 == 0 && k0 < k1 && k1 <= n, ANCKA_ERR_ARG, "knn: bad key range");
  auto st = as_stream(stream);
  const KeyRange kr{k0, k1};
  if (integer_exact > 0)
    return knn_tc(X, n, d, ldx, K, q_begin, q_end, ids, scores, workspace, workspace_bytes, st,
                  integer_exact == 2, kr);
  ANCKA_REQUIRE(integer_exact == 0, ANCKA_ERR_UNSUPPORTED, "key ranges need a tensor-core path");
  return knn_real(X, n, d, ldx, K, q_begin, q_end, ids, scores, workspace, workspace_bytes, st, kr);
}

extern "C" int ancka_knn_exact_csr_keys(const int64_t* indptr, const int32_t* indices,
                                        const double* data, int64_t n, int64_t d, int32_t K,
                                        int32_t integer_exact, int64_t q_begin, int64_t q_end,
                                        int64_t k0, int64_t k1, int32_t* ids, double* scores,
                                        void* workspace, size_t workspace_bytes,
                                        ancka_stream_t stream) {
  ANCKA_REQUIRE(K >= 1 && K < n, ANCKA_ERR_ARG, "knn: bad sizes");
  ANCKA_REQUIRE(integer_exact == 1 || integer_exact == 2, ANCKA_ERR_UNSUPPORTED,
                "CSR attributes are supported on the integer-exact tensor-core path only");
  ANCKA_REQUIRE(0 <= q_begin && q_begin < q_end && q_end <= n, ANCKA_ERR_ARG, "knn: bad query range");
  ANCKA_REQUIRE(k0 >= 0 && k0 % 256 == 0 && k0 < k1 && k1 <= n, ANCKA_ERR_ARG, "knn: bad key range");
  return knn_tc_csr(indptr, indices, data, n, d, K, q_begin, q_end, ids, scores, workspace,
                    workspace_bytes, as_stream(stream), integer_exact == 2, KeyRange{k0, k1});
}

extern "C" int ancka_knn_fallback_rows(void* workspace, size_t workspace_bytes, int64_t n, int64_t d,
                                       int32_t K, int64_t q_begin, int64_t q_end,
                                       int32_t* out_rows) {
  ANCKA_REQUIRE(out_rows != nullptr, ANCKA_ERR_ARG, "knn_fallback_rows: null output");
  return knn_real_flag_count(workspace, workspace_bytes, n, d, K, q_begin, q_end, out_rows);
}

extern "C" int ancka_knn_fallback_rows_async(void* workspace, size_t workspace_bytes, int64_t n,
                                             int64_t d, int32_t K, int64_t q_begin, int64_t q_end,
                                             int32_t* out_rows_dev, ancka_stream_t stream) {
  ANCKA_REQUIRE(out_rows_dev != nullptr, ANCKA_ERR_ARG, "knn_fallback_rows_async: null output");
  return knn_real_flag_count_async(workspace, workspace_bytes, n, d, K, q_begin, q_end, out_rows_dev,
                                   as_stream(stream));
}
