/*
 * ancka_b200.h -- C ABI of the B200-native ANCKA clustering hot path.
 *
 * Plain C: device pointers, sizes and an opaque CUDA stream handle; no torch
 * or C++ types cross this boundary.  Every entry point returns an ANCKA_*
 * status; on failure `ancka_last_error()` returns a thread-local message.
 * The Python package `paper_2408_05459_b200` binds these with ctypes and
 * keeps the reference's Python API (ancka/__init__.py:12-99) on top.
 *
 * Each function names the reference interface it replaces (paths relative
 * to /root/reference/pkg/src/ancka).  All work is enqueued on `stream`; no
 * function synchronises the device unless documented ("syncs").
 */
#ifndef ANCKA_B200_H
#define ANCKA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ANCKA_ABI_VERSION 1

typedef void* ancka_stream_t; /* cudaStream_t */

enum ancka_status {
  ANCKA_OK = 0,
  ANCKA_ERR_ARG = 1,      /* maps to ValueError                       */
  ANCKA_ERR_CUDA = 2,     /* maps to RuntimeError                     */
  ANCKA_ERR_NETWORK = 3,  /* maps to ancka.NetworkError (network.py:39) */
  ANCKA_ERR_UNSUPPORTED = 4
};

enum ancka_dtype { ANCKA_F32 = 0, ANCKA_F64 = 1 };
enum ancka_kind { ANCKA_GRAPH = 0, ANCKA_HYPERGRAPH = 1, ANCKA_MULTIPLEX = 2 };
#define ANCKA_MAX_LAYERS 8

/* Sparse row matrix on the device.  values == NULL means every stored entry
 * is 1 (index-only storage of an unweighted factor). */
typedef struct {
  int64_t rows, cols, nnz;
  const int64_t* rowptr; /* rows + 1 */
  const int32_t* colidx; /* nnz, sorted within each row */
  const void* values;    /* nnz of the operator dtype, or NULL */
} ancka_csr;

/* Load-balancing plan for the f32 operator application: rows whose
 * structural + KNN nonzeros exceed a threshold ("long" rows, e.g. KNN hubs)
 * are summed by a whole warp each (lanes strided over the nonzeros, fixed
 * butterfly combine: deterministic) in the same launch as the regular rows.
 * All pointers NULL / n_long 0 disable it.  The f64 path ignores it (it keeps
 * scipy's sequential order). */
typedef struct {
  int64_t n_long;
  const uint8_t* is_long;     /* n                                        */
  const int32_t* long_rows;   /* n_long                                   */
  const int32_t* row_order;   /* n rows by descending cost (optional): the
                                 fused narrow-block kernel deals rows to its
                                 lane groups in this order (balanced tails) */
  const int32_t* locality_order; /* n rows grouped by cluster (optional, graph
                                 operators): the f32 apply processes rows in
                                 this order, so the rows in flight share their
                                 neighbours' gathered rows in L2; results are
                                 unchanged (each row's sum is the same) */
} ancka_row_split;

/* Device-resident WalkOperator (walk.py:89-104).  Index arrays are shared by
 * the f32 and f64 instances; `dtype` selects the value arrays. */
typedef struct {
  int32_t kind;           /* ancka_kind                                  */
  int32_t dtype;          /* ancka_dtype of values/beta                  */
  int64_t n, m;           /* nodes, hyperedges (0 for graphs)            */
  ancka_csr p_n;          /* graph: P_N = D^-1 A            (n x n)       */
  ancka_csr p_e;          /* hypergraph: P_E = D_E^-1 H     (m x n)       */
  ancka_csr p_v;          /* hypergraph: P_V = D_V^-1 H^T   (n x m)       */
  ancka_csr p_k;          /* P_K = D_K^-1 A_K               (n x n)       */
  ancka_csr t_a;          /* init transposes: graph P_N^T (n x n);
                             hypergraph P_V^T (m x n)                     */
  ancka_csr t_b;          /* hypergraph P_E^T (n x m); unused for graphs  */
  const void* beta;       /* n, beta_vector (walk.py:47-57)              */
  const uint8_t* selfloop;/* n, 1 where walk.py:123 adds a self-loop     */
  ancka_row_split split;  /* f32 load balancing of the n-row pass         */
  int32_t n_layers;       /* multiplex: L <= ANCKA_MAX_LAYERS (0 otherwise) */
  const ancka_csr* layers;   /* multiplex: host array of L CSR views of
                                P_l = D_l^-1 A_l (walk.py:82-86); the
                                structural term is (sum_l P_l M) / L     */
  const ancka_csr* layers_t; /* multiplex: P_l^T, for the rowvec apply    */
} ancka_operator;

const char* ancka_last_error(void);
int ancka_abi_version(void);
/* Number of kernels this library has enqueued (stream capture counts once;
 * CUDA-graph replays are not seen here). */
int64_t ancka_launch_count(void);
/* Fails unless a compute-capability 10.x device is current. */
int ancka_device_check(void);

/* ---- subsystem 1: exact KNN graph (knn.py:112-140, 294-324) ------------ */

/* Exact top-K cosine neighbours of every row of a dense n x d matrix X (row
 * stride ldx elements, dtype f64).  Selection and order follow
 * _ordered_top_k (knn.py:83-98): strictly positive similarities only, j != i,
 * order (similarity desc, index asc); an all-zero row gets an empty list.
 * `integer_exact` selects the path:
 *   2 / 1  every X entry is an integer with |x| <= 16 (e4m3) / <= 256 (bf16)
 *          and every row's sum of squares < 2^24: tcgen05 computes exact
 *          integer dot products, ranked by exact rational comparison;
 *   0      real-valued X: tcgen05 split-bf16 (hi/lo) contraction with a
 *          rigorous error bound selects candidates, which are re-ranked with
 *          exact f64 dots; rows the bound cannot certify are recomputed by
 *          the f64 CUDA-core scan (ancka_knn_fallback_rows reports how many);
 *  -1      the f64 CUDA-core scan for every row.
 * Only query rows [q_begin, q_end) are computed (against all n keys): the
 * query-row sharding of the multi-GPU path; [0, n) is the whole matrix.
 * Outputs: ids ((q_end-q_begin) x K int32, -1 padded), scores (same shape,
 * f64, 0 padded, min(s, 1) as knn.py:139).  ANCKA_ERR_NETWORK if K >= n. */
size_t ancka_knn_workspace_size(int64_t n, int64_t d, int32_t K, int32_t integer_exact);
int ancka_knn_exact(const double* X, int64_t n, int64_t d, int64_t ldx, int32_t K,
                    int32_t integer_exact, int64_t q_begin, int64_t q_end, int32_t* ids,
                    double* scores, void* workspace, size_t workspace_bytes,
                    ancka_stream_t stream);

/* Diagnostics of the last integer_exact == 0 call that used this workspace
 * (same sizes): number of query rows the tensor-core certificate rejected
 * and the f64 scan recomputed.  Synchronises with the device. */
int ancka_knn_fallback_rows(void* workspace, size_t workspace_bytes, int64_t n, int64_t d,
                            int32_t K, int64_t q_begin, int64_t q_end, int32_t* out_rows);
/* Same count copied to device memory on `stream` (no synchronisation). */
int ancka_knn_fallback_rows_async(void* workspace, size_t workspace_bytes, int64_t n, int64_t d,
                                  int32_t K, int64_t q_begin, int64_t q_end, int32_t* out_rows_dev,
                                  ancka_stream_t stream);

/* Same, with X given as a CSR matrix (indptr n+1, sorted indices, f64 data):
 * the quantised tensor-core operand is built directly from the nonzeros (no
 * dense f64 copy).  Integer-exact path only (integer_exact = 1 bf16, 2 fp8);
 * the workspace is ancka_knn_workspace_size(n, d, K, integer_exact). */
int ancka_knn_exact_csr(const int64_t* indptr, const int32_t* indices, const double* data,
                        int64_t n, int64_t d, int32_t K, int32_t integer_exact, int64_t q_begin,
                        int64_t q_end, int32_t* ids, double* scores, void* workspace,
                        size_t workspace_bytes, ancka_stream_t stream);

/* Same searches restricted to the key rows [k0, k1) (k0 a multiple of 256):
 * the query-stationary ring of the multi-GPU path computes its own rows
 * against each visiting key block once (reference knn.py:112-140 blocked
 * over keys).  Rows the real-valued certificate rejects are rescanned
 * against all keys; merge with ancka_knn_merge_lists (de-duplicating). */
int ancka_knn_exact_keys(const double* X, int64_t n, int64_t d, int64_t ldx, int32_t K,
                         int32_t integer_exact, int64_t q_begin, int64_t q_end, int64_t k0,
                         int64_t k1, int32_t* ids, double* scores, void* workspace,
                         size_t workspace_bytes, ancka_stream_t stream);
int ancka_knn_exact_csr_keys(const int64_t* indptr, const int32_t* indices, const double* data,
                             int64_t n, int64_t d, int32_t K, int32_t integer_exact,
                             int64_t q_begin, int64_t q_end, int64_t k0, int64_t k1, int32_t* ids,
                             double* scores, void* workspace, size_t workspace_bytes,
                             ancka_stream_t stream);

/* Per row, merge two neighbour lists (each ordered by score desc, id asc,
 * -1 padded) into the first K of their union by the same order, dropping
 * repeated ids (knn.py:83-98 applied across key blocks).  In place into
 * (ids_a, scores_a). */
int ancka_knn_merge_lists(int32_t* ids_a, double* scores_a, const int32_t* ids_b,
                          const double* scores_b, int64_t nq, int32_t K, ancka_stream_t stream);

/* KNN-graph rows from COO entries (local row, global column, score): the
 * per-rank rows of A_K = M + M^T after the all-to-all of transposed
 * triples, then P_K rows (same sums/normalisation as ancka_knn_graph).
 * Capacities: colidx/val arrays hold E entries. */
size_t ancka_knn_graph_coo_workspace_size(int64_t E);
int ancka_knn_graph_coo(const int32_t* rows, const int32_t* cols, const double* vals, int64_t E,
                        int64_t nrows, int64_t ncols, int64_t* rowptr, int32_t* colidx,
                        double* a_k, double* p_k64, float* p_k32, uint8_t* zero_rows,
                        int64_t* nnz_out, void* workspace, size_t workspace_bytes,
                        ancka_stream_t stream);

/* build_knn_adjacency + knn_transition (knn.py:294-324): A_K = M + M^T as a
 * sorted CSR and P_K = D_K^-1 A_K with row sums summed exactly as numpy's
 * pairwise reduction (so f64 values are bit-identical to scipy's).
 * Capacities: colidx/val arrays hold 2*n*K entries.  nnz_out is a device
 * int64.  zero_rows[i] = 1 where row i of A_K is empty. */
size_t ancka_knn_graph_workspace_size(int64_t n, int32_t K);
int ancka_knn_graph(const int32_t* ids, const double* scores, int64_t n, int32_t K,
                    int64_t* rowptr, int32_t* colidx, double* a_k, double* p_k64,
                    float* p_k32, uint8_t* zero_rows, int64_t* nnz_out,
                    void* workspace, size_t workspace_bytes, ancka_stream_t stream);

/* ---- structural factors (walk.py:38-79, 153-174) ----------------------- */

/* _row_normalize (walk.py:38-44): out = (1/rs_i) * a_ij with rs_i the row
 * sum in numpy/scipy's order (a[b] + pairwise(a[b+1:e])); rows with rs = 0
 * stay zero.  A is f64 (values required); inv_rows (optional, rows) gets
 * 1/rs_i (0 for empty rows).  Bit-identical to scipy's diags(inv) @ a. */
int ancka_csr_row_normalize(const ancka_csr* A, double* out_values, double* inv_rows,
                            ancka_stream_t stream);

/* out[p] = col_scale[colidx[p]] * values[p]: A D (e.g. P_V^T from H). */
int ancka_csr_col_scale(const ancka_csr* A, const double* col_scale, double* out_values,
                        ancka_stream_t stream);

/* CSR transpose (scipy's a.T.tocsr()): t_rowptr (cols+1 int64), t_colidx
 * (nnz int32, ascending within each row), t_values (nnz f64, optional). */
size_t ancka_csr_transpose_workspace_size(int64_t rows, int64_t cols, int64_t nnz);
int ancka_csr_transpose(const ancka_csr* A, int64_t* t_rowptr, int32_t* t_colidx,
                        double* t_values, void* workspace, size_t workspace_bytes,
                        ancka_stream_t stream);

/* Attribute checks that select the KNN path (integer_exact levels): out3 =
 * {1 if some entry is not an integer else 0, max |x|, max row sum of x^2}.
 * CSR (rowptr != NULL, values = nonzeros) or dense (rowptr NULL, ld, d). */
int ancka_attr_check(const int64_t* rowptr, const double* values, int64_t rows, int64_t ld,
                     int64_t d, double* out3, ancka_stream_t stream);

/* ---- subsystem 2: walk operator application ---------------------------- */

/* apply_joint_transition (walk.py:177-190): Z = (I-B) P_struct Q + B P_K Q,
 * Q and Z row-major n x c with leading dims ldq/ldz (multiples of 4 for f32,
 * 2 for f64; padding columns are read/written as zeros).  `scratch` holds the
 * hypergraph intermediate P_E Q (m x ldq elements).  With f64 the summation
 * order equals scipy's csr_matvecs, so results are bit-identical. */
int ancka_op_apply(const ancka_operator* op, const void* Q, int64_t ldq, int32_t c,
                   void* Z, int64_t ldz, void* scratch, ancka_stream_t stream);

/* apply_structure_rowvec (walk.py:153-174) in column form: Z = P_struct^T Q
 * (+ self-loops). */
int ancka_op_apply_struct_t(const ancka_operator* op, const void* Q, int64_t ldq, int32_t c,
                            void* Z, int64_t ldz, void* scratch, ancka_stream_t stream);

/* Generic two-segment SpMM, the building block of the row-partitioned
 * multi-GPU operator (walk.py:135-190 on a row slice):
 *   out[r] = epi( mix( S[r] . s_src (+ self), K[r] . k_src ) ),  r < rows
 * S, K: row slices (rows x *) whose column indices address the full
 * gathered sources; mix = (1-beta_r) s + beta_r k when beta != NULL, else s;
 * self-loop rows add self_src[row_offset + r]; epi: scale*x + (col == tag[r]
 * ? tagval[col] : 0) when tag != NULL.  dtype ANCKA_F32 / ANCKA_F64. */
int ancka_spmm2(int32_t dtype, int64_t rows, int32_t c, const ancka_csr* S, const void* s_src,
                int64_t lds, const ancka_csr* K, const void* k_src, int64_t ldk, const void* beta,
                const uint8_t* selfloop, const void* self_src, int64_t ld_self, int64_t row_offset,
                const int32_t* tag, const void* tagval, double scale, void* out, int64_t ldo,
                const int32_t* order, ancka_stream_t stream);

/* Split Cholesky-QR for row-partitioned blocks: G = Z^T Z of the local rows
 * (packed upper, f64, c(c+1)/2), all-reduced by the caller, then factor +
 * Q_out = Z R^-1 + local ||Q_out - Q_prev||^2 into stats[0] (stats as
 * ancka_orth_step_f32).  Workspace: ancka_orth_workspace_size(NULL, c). */
int ancka_gram_f32(const float* Z, int64_t n, int64_t ld, int32_t c, double* G,
                   void* workspace, size_t workspace_bytes, ancka_stream_t stream);
int ancka_cholqr_apply_f32(const float* Z, const float* Q_prev, float* Q_out, int64_t n, int64_t ld,
                           int32_t c, const double* G, double* stats, void* workspace,
                           size_t workspace_bytes, ancka_stream_t stream);

/* ---- wide-block discretisation (k > 16; engine.py:183-263) ------------- */
/* The n-sized per-round work of _alternate_rounding on the device; the host
 * runs the k x k SVD (np.linalg.svd, as the reference) between rounds.
 * q~ = q / ||q|| (numpy's pairwise norm) as f32 rows of stride ldt >= k;
 * zero_rows (device int32) counts all-zero rows. */
int ancka_disc_normalize(const float* Q, int64_t ldq, int64_t col0, int64_t n, int32_t k,
                         float* qt, int64_t ldt, int32_t* zero_rows, ancka_stream_t stream);
/* labels = first argmax_j (q~ R)[i, j], margin = second-largest score. */
int ancka_disc_score(const float* qt, int64_t ldt, int64_t n, int32_t k, const float* R,
                     int64_t ldr, int32_t* labels, float* margin, ancka_stream_t stream);
/* S[l*k + j] = sum over rows with label l of llrint(q~[i][j] * scale) (int64),
 * counts[l] = cluster sizes.  Integer sums: bit-reproducible. */
int ancka_disc_accumulate(const float* qt, int64_t ldt, int64_t n, int32_t k,
                          const int32_t* labels, double scale, int64_t* S, int64_t* counts,
                          ancka_stream_t stream);
/* acc[i] += |q~_i . rcol| (f64): one greedy pass of _prototype_rotation. */
int ancka_disc_proto_pass(const float* qt, int64_t ldt, int64_t n, int32_t k,
                          const double* rcol, double* acc, ancka_stream_t stream);

/* ---- engine pieces (engine.py) ----------------------------------------- */

/* init_bcm (engine.py:87-127) after centre selection: t_i restart-walk steps
 * on the transposed structure (f64) and the first-max argmax over centres.
 * centers: device int64[k] sorted.  labels_out: int32[n]. */
size_t ancka_init_workspace_size(const ancka_operator* op, int32_t k);
int ancka_init_bcm(const ancka_operator* op64, const int64_t* centers, int32_t k, int32_t t_i,
                   double alpha, int32_t* labels_out, void* workspace, size_t workspace_bytes,
                   ancka_stream_t stream);

/* orthogonal_step (engine.py:130-149), f32 fast path: Z = apply(Q_prev);
 * Cholesky-QR with an f64 Gram and f64 k x k factor; Q_out = Z R^-1 (diag R
 * > 0 by construction, the reference's sign convention).  stats (device
 * f64[4]): [0] = ||Q_out - Q_prev||_F^2 (overwritten each step),
 * [1] = min(stats[1], min pivot ratio R_jj^2 / G_jj), [2] += number of
 * suspect pivots (ratio <= 1e-9); the caller resets [1] = 1, [2] = 0.
 * [3] reserved. */
size_t ancka_orth_workspace_size(const ancka_operator* op, int32_t c);
int ancka_orth_step_f32(const ancka_operator* op32, const float* Q_prev, float* Q_out,
                        float* Z, int64_t ld, int32_t c, double* stats,
                        void* workspace, size_t workspace_bytes, ancka_stream_t stream);

/* `steps` consecutive f32 orthogonal steps in ONE cooperative kernel for
 * narrow blocks (c <= 8, ld == 8): Q0 is the input, the result lands in Q0
 * if `steps` is even and Q1 if odd.  stats as ancka_orth_step_f32 ([0] is
 * the last step's ||dQ||_F^2).  Returns ANCKA_ERR_UNSUPPORTED for other
 * shapes (callers then use ancka_orth_step_f32). */
size_t ancka_orth_block_workspace_size(const ancka_operator* op);
int ancka_orth_block_f32(const ancka_operator* op32, float* Q0, float* Q1, float* Z, int64_t ld,
                         int32_t c, int32_t steps, double* stats, void* workspace,
                         size_t workspace_bytes, ancka_stream_t stream);

/* Thin QR in f64 by classical Gram-Schmidt with re-orthogonalisation
 * (Householder-equivalent Q/|R_jj| for full-rank columns; the reference's
 * rank test engine.py:141-142 is applied by the caller on rdiag).
 * Z (n x c, ld) is overwritten by Q.  rdiag: device f64[c]. */
size_t ancka_qr_f64_workspace_size(int64_t n, int32_t c);
int ancka_qr_f64(double* Z, int64_t n, int64_t ld, int32_t c, double* rdiag,
                 void* workspace, size_t workspace_bytes, ancka_stream_t stream);

/* discretize + repair_empty_clusters (engine.py:162-288) on columns
 * [col0, col0+k) of Q (f32, n x ldq): two alternating-rounding runs (identity
 * and prototype start), up to max_iter rounds each, |d obj| < tol.
 * 1 <= k <= 192: k <= 64 one cooperative kernel; 64 < k <= 192 device-driven
 * rounds (the call synchronises the stream once every 8 rounds to read the
 * convergence flag; no host arithmetic).
 * labels_out: int32[n]; info (device f64[8 + 2*max_iter + 2*k*k]):
 *   [0] final objective  [1] rounds  [2] converged  [3] winning run (0 id, 1 proto)
 *   [4] empty clusters left (repair impossible -> NetworkError)
 *   [5] zero rows  [6] rounds of run 0  [7] rounds of run 1
 *   [8 ...] objective trace of run 0 (max_iter slots) then run 1,
 *   then the final k x k rotation R of run 0 and of run 1 (row-major). */
size_t ancka_discretize_workspace_size(int64_t n, int32_t k, int32_t max_iter);
int ancka_discretize(const float* Q, int64_t ldq, int64_t col0, int64_t n, int32_t k,
                     int32_t max_iter, double tol, int32_t* labels_out, double* info,
                     void* workspace, size_t workspace_bytes, ancka_stream_t stream);

/* calc_mhc (engine.py:291-299): phi = 1 - tr(Yhat^T F)/k after gamma steps of
 * F <- (1-alpha) apply(F) + alpha Yhat.  phi_out: device f64[1]; sizes_out:
 * device int64[k] (cluster sizes; an empty cluster -> phi = NaN). */
size_t ancka_mhc_workspace_size(const ancka_operator* op, int32_t k);
int ancka_mhc(const ancka_operator* op, const int32_t* labels, int32_t k, double alpha,
              int32_t gamma, double* phi_out, int64_t* sizes_out,
              void* workspace, size_t workspace_bytes, ancka_stream_t stream);
/* same_out (device int32) = 1 iff labels a and b (int32[n] in [0, k), every
 * cluster nonempty) are the same partition up to relabelling -- the MHC of
 * b then repeats the MHC of a exactly (calc_mhc depends on the partition
 * only).  minmax_ws: device int32[2k] scratch. */
int ancka_same_partition(const int32_t* a, const int32_t* b, int64_t n, int32_t k,
                         int32_t* minmax_ws, int32_t* same_out, ancka_stream_t stream);

/* Diagnostics of the fused MHC kernel (k <= 8, set ANCKA_MHC_TIMING=1 before
 * the first call): copies the phase timers (host u64[64 + 9 * 1024]: per
 * phase CTA-0 ns and max-over-CTAs ns, per-CTA ns, per-CTA nonzeros) and
 * optionally resets them.  Synchronises the device.  Not used on the
 * clustering path. */
void ancka_mhc_timing(unsigned long long* out, int reset);

/* Load-balancing plan (ancka_row_split) of the f32 operator pass, from the
 * structural row pointers `srp` (P_N, or P_V for hypergraphs) and the KNN
 * row pointers `krp`.  No reference counterpart: the reference's scipy SpMM
 * is sequential per row (walk.py:135-190); this only schedules the same sums.
 * Writes row_order (n, descending cost, stable), is_long (n, cost > thr),
 * long_rows (capacity n, ascending) and *n_long_out (device int64). */
size_t ancka_row_split_workspace_size(int64_t n);
int ancka_row_split_plan(const int64_t* srp, const int64_t* krp, int64_t n, double thr,
                         int32_t* order_out, uint8_t* is_long_out, int32_t* long_rows_out,
                         int64_t* n_long_out, void* workspace, size_t workspace_bytes,
                         ancka_stream_t stream);

/* Rows sorted by (label, row): the locality order of ancka_row_split. */
size_t ancka_locality_order_workspace_size(int64_t n);
int ancka_locality_order(const int32_t* labels, int64_t n, int32_t k, int32_t* order_out,
                         void* workspace, size_t workspace_bytes, ancka_stream_t stream);

/* The first iterate Q0 = [1/sqrt(n) | Yhat0] (engine.py:368-371, Yhat by
 * normalize_bcm, engine.py:75-84) as an n x ldq f64 block, from device labels
 * and cluster sizes; first_col = 1/sqrt(n); columns past c are zero. */
int ancka_bcm_block(const int32_t* labels, int64_t n, int32_t c, const int64_t* sizes,
                    double first_col, double* q, int64_t ldq, ancka_stream_t stream);

/* beta_vector (walk.py:47-57: beta, 1 for degree-0 nodes, 0 for empty KNN
 * rows) in f64 and f32, and the self-loop flags of walk.py:123 (degree 0 and
 * beta_i = 0), from the node degrees and the KNN zero-row flags. */
int ancka_beta_vector(const double* degrees, const uint8_t* knn_zero_rows, int64_t n, double beta,
                      double* beta64_out, float* beta32_out, uint8_t* selfloop_out,
                      ancka_stream_t stream);

/* Cluster sizes (BcmMatrix.cluster_sizes, network.py:176-177). */
int ancka_cluster_sizes(const int32_t* labels, int64_t n, int32_t k, int64_t* sizes_out,
                        ancka_stream_t stream);

/* ---- approximate KNN: inverted-file index (knn.py:143-280, knn_search_approx;
 * csrc/knn_ivf.cu).  xn is the n x dp f32 copy of the row-normalised
 * attributes (dp = d rounded up to 4, zero padded), the matrix the reference
 * searches (knn.py:172-174). */
/* xn = f32(x * (1/||x||)) from dense f64 X (X != NULL) or CSR attributes. */
int ancka_ivf_normalize(const double* X, int64_t ldx, const int64_t* indptr,
                        const int32_t* indices, const double* data, int64_t n, int64_t d,
                        float* xn, int64_t dp, ancka_stream_t stream);
/* S = A[arows] B^T + bias (f32): stored to C (m x ldc) when C != NULL, and/or
 * reduced to a first-max argmax per row into argmax_keys (zeroed u64, packed
 * score | ~column; decode with ancka_ivf_argmax_finish).  knn.py:216-222
 * (_batched_argmax_assign) and the probe scores of knn.py:246. */
int ancka_ivf_gemm(const float* A, int64_t lda, const int32_t* arows, int64_t m, const float* B,
                   int64_t ldb, int32_t nb, int64_t d, const float* bias, float* C, int64_t ldc,
                   unsigned long long* argmax_keys, ancka_stream_t stream);
/* labels[r] = argmax column; counts label changes into *changed (nullable);
 * re-zeroes the keys. */
int ancka_ivf_argmax_finish(unsigned long long* argmax_keys, int64_t m, int32_t* labels,
                            int32_t* changed, ancka_stream_t stream);
/* probes[r] = the nprobe largest of S[r, :nb] (knn.py:250, argpartition;
 * ties to the smaller column). */
int ancka_ivf_topsel(const float* S, int64_t lds, int64_t m, int32_t nb, int32_t nprobe,
                     int32_t* probes, ancka_stream_t stream);
/* Counting sort of count entries by key: ptr (nbuckets + 1) offsets, ent =
 * entry indices grouped by key; tiles (nullable) = per-bucket offsets of
 * ceil(size / tile) tiles.  Inverted lists (knn.py:200-203) and pair lists. */
size_t ancka_ivf_bucket_workspace_size(int32_t nbuckets);
int ancka_ivf_bucket(const int32_t* keys, int64_t count, int32_t nbuckets, int64_t* ptr,
                     int64_t* tiles, int32_t tile, int32_t* ent, void* workspace,
                     size_t workspace_bytes, ancka_stream_t stream);
/* Per (query, probe slot) pair: top-K2 f32 scores of the probed list's keys
 * (score desc, id asc; self excluded; scores <= -err dropped) into
 * part_s/part_i ((m * nprobe) x K2).  _ivf_search_all, knn.py:236-262.
 * qthr: m zeroed u32, the per-query threshold shared across pairs. */
int ancka_ivf_search(const float* xn, int64_t dp, const int32_t* perm, const int64_t* list_ptr,
                     const int64_t* pair_ptr, const int32_t* pair_ent, const int64_t* tile_ptr,
                     int32_t* counter, int32_t nlist, int32_t nprobe, int64_t q0, int32_t K2,
                     float err, float* part_s, int32_t* part_i, uint32_t* qthr,
                     ancka_stream_t stream);
/* Per query: merge the partial lists, re-rank in f64, top-K positive
 * (knn.py:257-260 with _ordered_top_k, knn.py:83-98); uncertified rows are
 * appended (global ids) to flagged / *nflag. */
int ancka_ivf_merge(const float* xn, int64_t dp, int64_t q0, int64_t m, int32_t nprobe, int32_t K2,
                    int32_t K, const float* part_s, const int32_t* part_i, float err, int32_t* ids,
                    double* scores, int32_t* flagged, int32_t* nflag, const float* lres,
                    const uint32_t* lmax_bits, ancka_stream_t stream);
/* The scan on the tensor cores: h = fp16(xn) (n x dh, dh = ceil16(d) <= 256,
 * entries below 2^-14 flushed) with per-row residual norms lres = ||xn - h||
 * and their maximum (u32 bits of a non-negative float); ancka_ivf_search_tc
 * scores each (list, pair tile) with mma.sync m16n8k16 (f32 accumulation),
 * floors and certificate at e_q = l_q + l_max + l_q l_max + acc_err (pass
 * lres / lmax_bits to ancka_ivf_merge; NULL there for the f32 scan). */
int ancka_ivf_half_prep(const float* xn, int64_t n, int64_t dp, void* h, int64_t dh, float* lres,
                        uint32_t* lmax_bits, ancka_stream_t stream);
/* Split of the probe slots for a two-phase scan: own = each query's own-list
 * slot (else -1), rest = the other slots (else -1); ancka_ivf_bucket skips
 * negative keys. */
int ancka_ivf_split_probes(const int32_t* probes, const int32_t* labels, int64_t q0, int64_t m,
                           int32_t nprobe, int32_t* own, int32_t* rest, ancka_stream_t stream);
int ancka_ivf_search_tc(const void* h, int64_t dh, const float* lres, const uint32_t* lmax_bits,
                        const int32_t* perm, const int64_t* list_ptr, const int64_t* pair_ptr,
                        const int32_t* pair_ent, const int64_t* tile_ptr, int32_t* counter,
                        int32_t nlist, int32_t nprobe, int64_t q0, int32_t K2, float acc_err,
                        float* part_s, int32_t* part_i, uint32_t* qthr, ancka_stream_t stream);
/* Exact top-K (f64 accumulation) for the listed rows against their probe
 * lists (probes != NULL) or all keys (the recall audit, _exact_rows_for,
 * knn.py:225-233).  compact: output row b instead of rows[b] - q0. */
int ancka_ivf_rows_exact(const float* xn, int64_t dp, int64_t n, const int32_t* rows,
                         int64_t nrows, const int32_t* probes, int32_t nprobe, int64_t q0,
                         const int32_t* perm, const int64_t* list_ptr, int32_t K, int32_t* ids,
                         double* scores, int32_t compact, ancka_stream_t stream);
/* One Lloyd update of the IVF centroids (_train_ivf, knn.py:143-153): cluster
 * sums in 64-bit fixed point (sums: nlist x d u64, counts: nlist, both
 * zeroed and left zeroed), C = mean (empty clusters keep their centre), bias
 * = -|C|^2/2 for the L2 assignment.  sums == NULL: bias only. */
int ancka_ivf_kmeans_update(const float* S, int64_t lds, const int32_t* arows, int64_t m,
                            const int32_t* labels, int32_t nlist, int64_t d,
                            unsigned long long* sums, int32_t* counts, float* C, int64_t ldc,
                            float* bias, ancka_stream_t stream);

/* Row-partitioned discretisation (engine.py:162-263 over a rank's rows
 * [row0, row0 + n_loc) of n_glob, 8 < k <= 192; dist.py drives it): the
 * device-driven rounds of the wide path with the caller's collectives in
 * between -- `tots` (k k + k u64 fixed-point cluster totals) is summed over
 * the ranks after each ANCKA_DW_ROUND_LOCAL (and ANCKA_DW_SNAP), `rvec`
 * (k f64) after each ANCKA_DW_PROTO_PICK, and `locbest` (3 f64: value,
 * global row, label) is all-gathered after each ANCKA_DW_PROTO_PASS /
 * ANCKA_DW_RESEED_CAND (the pass's into the buffer passed to PICK).  Labels (local rows) land in `labels`; `info` as ancka_discretize. */
enum {
  ANCKA_DW_START = 0,          /* a = run (0 identity, 1 prototype start) */
  ANCKA_DW_ROUND_LOCAL = 1,    /* a = run, b = first round: score, totals, snap into tots */
  ANCKA_DW_SNAP = 2,           /* the rank's current totals into tots */
  ANCKA_DW_CHECK_EMPTY = 3,    /* a = run: an empty global cluster sets the pause flag */
  ANCKA_DW_POLAR = 4,          /* a = run: rotation step from the global totals */
  ANCKA_DW_CLEAR_PAUSE = 5,
  ANCKA_DW_MARGINS = 6,        /* exact second-best scores of the local rows (reseed) */
  ANCKA_DW_MOVE_ROW = 7,       /* a = target cluster, b = local row */
  ANCKA_DW_PROTO_PASS = 8,     /* b = column j >= 1: running sums, local first minimum */
  ANCKA_DW_PROTO_PICK = 9,     /* a = world, b = forced global row or -1, ptr = gathered pairs */
  ANCKA_DW_PROTO_SETCOL = 10,  /* b = column j: R[:, j] = rvec */
  ANCKA_DW_FLAGS = 11,         /* ptr = device int32[6]: done0, done1, pause, empties0, empties1, it */
  ANCKA_DW_FINISH = 12,        /* winner's labels into `labels`; releases the host state */
  ANCKA_DW_RESEED_CAND = 13    /* ptr = device int64[k] global sizes: locbest = (margin, row, label) */
};
size_t ancka_discw_dist_workspace_size(int64_t n_loc, int32_t k);
int ancka_discw_dist_init(const float* Q, int64_t ldq, int64_t col0, int64_t n_loc, int64_t n_glob,
                          int64_t row0, int32_t k, int32_t max_iter, double tol, uint64_t* tots,
                          double* rvec, double* locbest, int32_t* labels, double* info, void* ws,
                          size_t workspace_bytes, ancka_stream_t stream);
int ancka_discw_dist_op(void* ws, int32_t op, int64_t a, int64_t b, const void* ptr,
                        ancka_stream_t stream);

/* Tensor-pipe peak microbenchmark (roofline denominators, no reference
 * counterpart): back-to-back tcgen05.mma M=128 N=256 on every SM, fmt 0 =
 * kind::f8f6f4 e4m3, 1 = kind::f16 bf16; returns the FLOP issued and the
 * event-timed milliseconds (synchronises `stream`); cycles: 148 per-CTA
 * clock64 spans (device memory). */
int ancka_tc_peak(int32_t fmt, int32_t iters, double* flop_out, double* ms_out,
                  long long* cycles, ancka_stream_t stream);
/* L2 read-bandwidth microbenchmark (the SpMM gather's denominator): `iters`
 * sweeps over a rows x row_floats f32 table that fits L2, rows read in order
 * (gather = 0) or hashed (gather = 1, the SpMM's row gathers). */
int ancka_l2_read(const float* table, int64_t rows, int32_t row_floats, int32_t iters,
                  int32_t gather, float* sink, double* bytes_out, double* ms_out,
                  ancka_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* ANCKA_B200_H */
