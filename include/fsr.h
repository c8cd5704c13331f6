/*
 * fsr.h -- C ABI of libfsr, the B200 (sm_100a) kernels behind the FSR hot path.
 *
 * The reference (specrank, pure Python) has no FFI; its "operator API" is the
 * module-level functions of spectral.py / ranking.py.  Each entry point below
 * replaces one numeric call site of those functions (cited file:line,
 * relative to /root/reference/pkg/src/specrank).  The Python host layer
 * (paper_1703_06935_b200.spectral / .ranking) keeps the reference signatures
 * and calls these through ctypes; a C/C++ host can bind them directly.
 *
 * Conventions
 *  - Plain C: no torch or CUDA types in the signatures.  `stream` arguments
 *    are cudaStream_t passed as void* (NULL = the context's stream).
 *  - Every matrix pointer is DEVICE memory, allocated by the caller.  Dense
 *    blocks are row-major with an explicit leading dimension (elements).
 *  - `dtype` selects the storage/arithmetic type: FSR_F32 or FSR_F64.  Small
 *    r_hat x r_hat matrices (Gram, projection, Cholesky factor, eigenvectors)
 *    are always float64.
 *  - CSR matrices: int64 row pointers, int32 column indices, values in dtype.
 *  - Return value: FSR_OK or an FSR_E* code; fsr_last_error(ctx) describes
 *    the most recent failure.  Calls are asynchronous on the context stream
 *    unless they return a host value (documented per function).
 *  - Deterministic: no floating-point atomics; for a fixed dtype, shapes and
 *    shard layout the results are bitwise reproducible.
 */
#ifndef FSR_H_
#define FSR_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSR_ABI_VERSION 1

enum fsr_status {
  FSR_OK = 0,
  FSR_EINVAL = 1,      /* contract violation (reference: ValueError)          */
  FSR_ENUMERICAL = 2,  /* non-finite / breakdown (reference: NumericalError)  */
  FSR_ECUDA = 3,
  FSR_ENOMEM = 4,
  FSR_ELIBRARY = 5,    /* cuBLAS / cuSOLVER failure                          */
  FSR_ENOTSPD = 6,     /* Cholesky breakdown: caller falls back to Householder */
  FSR_EIO = 7          /* file I/O or checksum failure (FSRX persistence)     */
};

enum fsr_dtype { FSR_F32 = 0, FSR_F64 = 1 };

typedef struct fsr_ctx fsr_ctx;

/* ---- context --------------------------------------------------------- */
int fsr_abi_version(void);
int fsr_ctx_create(int device, fsr_ctx** out);
void fsr_ctx_destroy(fsr_ctx* ctx);
int fsr_ctx_set_stream(fsr_ctx* ctx, void* stream);
const char* fsr_last_error(const fsr_ctx* ctx);
/* Number of libfsr kernels launched on this context so far (own kernels only;
 * cuBLAS/cuSOLVER calls are counted separately by fsr_library_calls). */
uint64_t fsr_launch_count(const fsr_ctx* ctx);
uint64_t fsr_library_calls(const fsr_ctx* ctx);
int fsr_synchronize(fsr_ctx* ctx);

/* Optional per-stage device timing: when enabled every entry point brackets
 * its device work with CUDA events on the context stream.  fsr_stage_time
 * synchronises, folds finished events into per-stage totals and returns the
 * accumulated milliseconds and launch count of one stage. */
enum fsr_stage {
  FSR_STAGE_GAUSSIAN = 0, FSR_STAGE_NORMALIZE = 1, FSR_STAGE_SPMM = 2, FSR_STAGE_GRAM = 3,
  FSR_STAGE_CHOLESKY = 4, FSR_STAGE_APPLY = 5, FSR_STAGE_EIGH = 6, FSR_STAGE_LIFT = 7,
  FSR_STAGE_SIGNS = 8, FSR_STAGE_HISTOGRAM = 9, FSR_STAGE_COMPACT = 10, FSR_STAGE_PROJECT = 11,
  FSR_STAGE_FILTER_SPMM = 12, FSR_STAGE_TRANSPOSE = 13 /* reserved */, FSR_STAGE_COPY_UNCOVERED = 14,
  FSR_STAGE_TOPK = 15, FSR_STAGE_HOUSEHOLDER = 16, FSR_NUM_STAGES = 17
};
int fsr_ctx_enable_timing(fsr_ctx* ctx, int on);

/* Context options.  FSR_OPT_DENSE_PATH: 0 = auto (F32 Gram / cross / apply /
 * lift on the tcgen05 int8 Ozaki kernels), 1 = cuBLAS/cuSOLVER (fp64-upcast
 * Gram, TRSM, SGEMM) -- kept for A/B checks.  FSR_OPT_SPMM_PANEL_BYTES: K2
 * schedule -- 0 = wide row panels, 32/64/128 = L2-resident column panels of
 * that many bytes per dense row (results identical; speed only).
 * FSR_OPT_TOPK_PRUNE: 1 (default) = fsr_filter_batch with top-k only (X ==
 * NULL), float32, sparse U, b >= 256 gathers Zs in fp16 and re-scores the
 * rows that can reach the top k exactly in fp32 (certified bound; the same
 * top-k indices and values as 0 = the unpruned fp32 path).
 * FSR_OPT_TOPK_SEGMENTS: segments a row is cut into by the exact top-k when
 * fewer rows than SMs are selected (0 = automatic; results identical). */
enum fsr_option {
  FSR_OPT_DENSE_PATH = 0, FSR_OPT_SPMM_PANEL_BYTES = 1, FSR_OPT_TOPK_PRUNE = 2, FSR_OPT_TOPK_SEGMENTS = 3
};
int fsr_ctx_set_option(fsr_ctx* ctx, int option, int64_t value);
int fsr_stage_time(fsr_ctx* ctx, int stage, double* ms, uint64_t* count);
int fsr_stage_reset(fsr_ctx* ctx);

/* ---- K0: start block  (spectral.py:55-65 gaussian_matrix) -------------
 * Rows [row_begin, row_end) of the (total_rows x cols) Box-Muller block drawn
 * from numpy's Philox4x64-10 stream with key (key0, key1) =
 * SeedSequence(seed).generate_state(2, uint64).  Uniforms are bit-identical to
 * numpy's; the transcendental step is fp64 (CUDA libm, <= 2 ulp).
 * out: (row_end-row_begin) x cols, ld = cols, dtype. */
int fsr_gaussian_block(fsr_ctx* ctx, int dtype, int64_t total_rows, int64_t cols,
                       int64_t row_begin, int64_t row_end, uint64_t key0, uint64_t key1,
                       void* out);

/* ---- K1: normalisation  (graph.py:118-139 degrees / normalize_adjacency) --
 * deg[i] = sum_j w_ij over the local rows (fp64). */
int fsr_csr_row_sums(fsr_ctx* ctx, int64_t n_rows, const int64_t* indptr, const double* data,
                     double* deg);
/* out[e] = (w_e * s_i) * s_j, s = 1/sqrt(deg) (0 where deg == 0).  `deg` is the
 * GLOBAL degree vector (indexed by column), local row i is global row
 * row_offset + i.  out has dtype `dtype_out`. */
int fsr_csr_normalize(fsr_ctx* ctx, int dtype_out, int64_t n_rows, int64_t row_offset,
                      const int64_t* indptr, const int32_t* indices, const double* data,
                      const double* deg, void* out);
/* Elementwise fp64 -> dtype conversion of n values (out may alias for F64). */
int fsr_convert_from_f64(fsr_ctx* ctx, int dtype, int64_t n, const double* in, void* out);

/* ---- K2: CSR SpMM  (spectral.py:170 -> sparsemat.py:63-64 -> csr_matvecs) --
 * Y[i, :ncols] = sum_e A_ie X[col_e, :ncols] for the n_rows local rows of A.
 * Accumulation follows CSR order per output element; in F64 the multiply and
 * add are rounded separately (no FMA), matching scipy's csr_matvecs bitwise. */
int fsr_csr_spmm(fsr_ctx* ctx, int dtype, int64_t n_rows, const int64_t* indptr,
                 const int32_t* indices, const void* values, int64_t ncols, const void* X,
                 int64_t ldx, void* Y, int64_t ldy);

/* ---- K3: orthonormalisation  (spectral.py:165-169 np.linalg.qr + check) ---
 * G (k x k, fp64, row-major, symmetric) = A^T A over n_rows rows
 * (accumulate != 0: G += A^T A). */
int fsr_gram(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t k, const void* A, int64_t lda,
             double* G, int accumulate);
/* F32 only: G (+)= A^T A on the tcgen05 int8 path with `levels` = 4 (four
 * 7-bit slices, 10 slice products: ~28-bit accurate, the default of fsr_gram)
 * or 1 (one slice, 1 product: ~7 bits -- enough for the first CholeskyQR pass,
 * whose R only needs to precondition; span(B R^-1) = span(B) for any R). */
int fsr_gram_levels(fsr_ctx* ctx, int64_t n_rows, int64_t k, const float* A, int64_t lda, double* G,
                    int accumulate, int levels);
/* In-place Cholesky G = R^T R (R upper).  Returns FSR_ENOTSPD on breakdown
 * (host-synchronous: reads the factorisation status). */
int fsr_cholesky(fsr_ctx* ctx, int64_t k, double* G);
/* A <- A R^-1 for the R produced by fsr_cholesky (row-major A, n_rows x k). */
int fsr_apply_rinv(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t k, const double* R, void* A,
                   int64_t lda);
/* F32 tcgen05 path: A <- A M' with M' = R^-1 kept to m_slices = 1 (7-bit) or
 * 4 (28-bit) slices; 1 is the first CholeskyQR pass (span(A M') = span(A)
 * for any invertible M'; 4 products instead of 10), used only when every
 * diagonal entry of R^-1 is >= 2^-4 of its column's maximum (else 4).  Other
 * dtypes / paths ignore m_slices. */
int fsr_apply_rinv_levels(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t k, const double* R, void* A,
                          int64_t lda, int m_slices);
/* Householder QR (single device): A <- Q, the reduced orthonormal factor.
 * Fallback for rank-deficient blocks, mirroring spectral.py:165. */
int fsr_householder_qr(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t k, void* A, int64_t lda);
/* max_ij |G_ij - delta_ij| written to *err_host (host-synchronous). */
int fsr_max_offdiag_error(fsr_ctx* ctx, int64_t k, const double* G, double* err_host);

/* ---- K4-K6: Rayleigh-Ritz  (spectral.py:174-198) ----------------------
 * C (k x k fp64) (+)= Q^T B over n_rows rows. */
int fsr_cross(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t k, const void* Q, int64_t ldq,
              const void* B, int64_t ldb, double* C, int accumulate);
/* Rayleigh-Ritz form: C = Q^T B where Q^T B is symmetric up to rounding
 * (B = A Q, A symmetric).  F32 tensor-core path computes the upper triangle
 * and mirrors it (half the work; the reference averages C and C^T, the two
 * differ at rounding level); other dtypes/paths compute the full product. */
int fsr_cross_sym(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t k, const void* Q, int64_t ldq,
                  const void* B, int64_t ldb, double* C, int accumulate);
/* C <- (C + C^T)/2; eigh; keep the r algebraically largest pairs in
 * argsort(-lambda, stable) order (spectral.py:141-144).  lam_host[r] gets the
 * eigenvalues (host-synchronous), V (k x r, fp64, row-major) the eigenvectors.
 * C is destroyed. */
int fsr_eigh_desc(fsr_ctx* ctx, int64_t k, double* C, int64_t r, double* lam_host, double* V);
/* Generalised form for a non-orthonormal basis Q~ (C = Q~^T A Q~, G = Q~^T Q~,
 * both destroyed): C v = lambda G v, top r by the same stable descending rule,
 * V (k x r fp64) G-orthonormal so U = Q~ V is orthonormal.  cuSOLVER sygvd. */
int fsr_eigh_gen_desc(fsr_ctx* ctx, int64_t k, double* C, double* G, int64_t r, double* lam_host, double* V);
/* U (n_rows x r, dtype) = Q (n_rows x k) V (k x r). */
int fsr_lift(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t k, int64_t r, const void* Q,
             int64_t ldq, const double* V, void* U, int64_t ldu);
/* Per column j: the first (lowest global row) entry of maximal |U_ij| over the
 * local rows; best_abs[j], best_row[j] (= row_offset + i) and best_val[j]
 * (signed).  (spectral.py:133-138 _fix_column_signs, first half.) */
int fsr_col_absmax(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t r, const void* U, int64_t ldu,
                   int64_t row_offset, double* best_abs, int64_t* best_row, double* best_val);
/* U[:, j] *= sign_j where sign_j = sign(best_val[j]) (0 -> +1), then
 * eta[i] = ||U_i,:|| (spectral.py:127-130, 133-138 second half). */
int fsr_apply_signs_rownorm(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t r, void* U,
                            int64_t ldu, const double* best_val, double* eta);
/* eta[i] = ||U_i,:|| without touching U. */
int fsr_row_norms(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t r, const void* U, int64_t ldu,
                  double* eta);

/* ---- K7: thresholding  (spectral.py:269-294 sparsify) ------------------
 * Entries are ordered by the key |u| (IEEE bits with the sign cleared:
 * 31-bit keys for F32, 63-bit for F64); exact zeros never count.
 * Histogram of digit ((key >> shift) & (2^bits-1)) over entries whose key
 * satisfies (key & ~(2^(shift+bits)-1)) == prefix.  hist (2^bits uint64) is
 * accumulated into (caller zeroes it).  bits <= 12. */
int fsr_abs_histogram(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t r, const void* U,
                      int64_t ldu, uint64_t prefix, int shift, int bits, uint64_t* hist);
/* Per row: gt[i] = #{key > T}, eq[i] = #{key == T}. */
int fsr_threshold_counts(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t r, const void* U,
                         int64_t ldu, uint64_t T, int64_t* gt, int64_t* eq);
/* Build the kept CSR rows: all entries with key > T plus the ties (key == T)
 * whose global (row, col) tie rank is < ties_to_take, where the local rows'
 * tie ranks start at tie_offset (ties held by lower-ranked shards).
 * indptr_out (n_rows+1) local, starting at 0; *nnz_host = kept count
 * (host-synchronous).  eta = row norms of the kept rows.  indices/values
 * must hold at least the kept count (<= sum(gt) + ties_to_take). */
int fsr_threshold_compact(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t r, const void* U,
                          int64_t ldu, uint64_t T, int64_t tie_offset, int64_t ties_to_take,
                          const int64_t* gt, const int64_t* eq, int64_t* indptr_out,
                          int32_t* indices_out, void* values_out, double* eta, int64_t* nnz_host);

/* ---- Operator level: the reference's offline functions as one call each ----
 * (the schedule spectral.py used to own, now in csrc/fsr_ops.cu).
 * Device arrays are row-major; temporaries are stream-ordered on the context
 * stream; calls that return host values synchronise it.
 * fsr_schedule_trace: ';'-separated orthonormalisation steps of the last
 * fsr_range_finder / fsr_orthonormalize call (e.g. "start;precond(dev=0.03);
 * precond+gram(dev=0.04)"), valid until the next such call on ctx. */
enum fsr_si_flags {
  FSR_SI_SPAN_ONLY = 1,         /* fp32: rounds 1..q-1 only precondition (span(Q) reaches the output) */
  FSR_SI_FUSED_RR = 2,          /* fp32: last round preconditioned, its exact Gram goes to Rayleigh-Ritz */
  FSR_SI_FAST_FIRST_APPLY = 4,  /* fp32: first CholeskyQR pass applies a 7-bit R^-1 */
  FSR_SI_DEFAULT = 7
};
/* numpy's Philox key for a seed: SeedSequence(seed).generate_state(2, uint64)
 * (the key fsr_gaussian_block takes; spectral.py:55-65).  Host only. */
void fsr_philox_key(uint64_t seed, uint64_t* key0, uint64_t* key1);
const char* fsr_schedule_trace(fsr_ctx* ctx);
/* Y (n x k, ld) <- an orthonormal basis of its span: CholeskyQR2, Householder
 * fallback (spectral.py:165-169 np.linalg.qr + the re-orthogonalisation check). */
int fsr_orthonormalize(fsr_ctx* ctx, int dtype, int64_t n, int64_t k, void* Y, int64_t ldy);
/* range_finder(A, r_hat, q, seed) (spectral.py:147-171) on the CSR A (n x n,
 * values in dtype).  Q, B: caller blocks n x r_hat (ld = r_hat); on return Q
 * is the last basis and B = A Q.  With FSR_SI_FUSED_RR (fp32) and gram_out
 * (r_hat x r_hat fp64, device) non-NULL the last basis is only well
 * conditioned and gram_out = Q^T Q; *gram_valid says whether that happened
 * (pass gram_out to fsr_rayleigh_ritz then).  EINVAL: r_hat outside [1, n],
 * q < 1 (spectral.py:158-161). */
int fsr_range_finder(fsr_ctx* ctx, int dtype, int64_t n, const int64_t* indptr, const int32_t* indices,
                     const void* values, int64_t r_hat, int q, uint64_t seed, int flags, void* Q, void* B,
                     double* gram_out, int* gram_valid);
/* approx_eigendecomposition (spectral.py:174-198): C = Q^T B, eigh (C v =
 * lambda G v when gram != NULL), top r descending (stable), U = Q V (n x r,
 * dtype), column signs (spectral.py:133-138), eta = row norms (device fp64).
 * lam_host[r].  EINVAL: r outside [1, r_hat]. */
int fsr_rayleigh_ritz(fsr_ctx* ctx, int dtype, int64_t n, int64_t r_hat, const void* Q, int64_t ldq,
                      const void* B, int64_t ldb, const double* gram, int64_t r, double* lam_host, void* U,
                      int64_t ldu, double* eta);
/* decompose(A, r, p, q, seed) (spectral.py:297-309): r_hat = min(r + p, n). */
int fsr_decompose(fsr_ctx* ctx, int dtype, int64_t n, const int64_t* indptr, const int32_t* indices,
                  const void* values, int64_t r, int64_t p, int q, uint64_t seed, int flags, double* lam_host,
                  void* U, int64_t ldu, double* eta);
/* sparsify(dec, tau) (spectral.py:269-294) on the dense U (n x r): exactly
 * keep = min(tau, nnz(U)) entries of largest |u|, ties in (row, col) order.
 * fsr_sparsify_select returns the threshold key, the ties taken and keep (to
 * size the outputs); fsr_sparsify writes the CSR (indptr n+1, indices and
 * values of >= keep capacity), eta of the kept rows and *nnz_host = keep.
 * EINVAL: tau < 1. */
int fsr_sparsify_select(fsr_ctx* ctx, int dtype, int64_t n, int64_t r, const void* U, int64_t ldu, int64_t tau,
                        uint64_t* T_out, int64_t* ties_out, int64_t* keep_out);
int fsr_sparsify(fsr_ctx* ctx, int dtype, int64_t n, int64_t r, const void* U, int64_t ldu, int64_t tau,
                 int64_t* indptr_out, int32_t* indices_out, void* values_out, int64_t capacity, double* eta,
                 int64_t* nnz_host);
/* The second half of fsr_sparsify for a threshold (T, ties) already chosen
 * by fsr_sparsify_select (outputs must hold its `keep` entries). */
int fsr_sparsify_apply(fsr_ctx* ctx, int dtype, int64_t n, int64_t r, const void* U, int64_t ldu, uint64_t T,
                       int64_t ties, int64_t* indptr_out, int32_t* indices_out, void* values_out, double* eta,
                       int64_t* nnz_host);

/* ---- K8/K9: online batch  (ranking.py:219-255 _project / filter) ------------
 * For b observation columns y_j (CSC: y_ptr[b+1], y_idx row ids, y_val in dtype):
 *   z_j = U[supp y_j]^T y_j            (K8, ranking.py:219-226)
 *   x_j = U (w .* z_j)                 (K9, ranking.py:246)
 *   x_j[i] = y_ij where eta_i == 0     (copy_uncovered, ranking.py:248-254)
 * U is CSR (u_indptr/u_indices/u_values, n x r; canonical: distinct sorted
 * column indices per row, as scipy/sparsify produce) when u_sparse, else dense
 * u_dense (n x r, ld ldu).  w: r weights h(lambda) (dtype).  eta: n fp64 (may
 * be NULL when copy_uncovered == 0).
 * Outputs: X (b x n, row j = x_j) when X != NULL; and/or the top `topk`
 * entries of every x_j ordered by (-x, index) (ranking.py:390-395) into
 * top_idx (b x topk int64) / top_val (b x topk dtype) when topk > 0.
 * workspace: device scratch of fsr_filter_workspace_bytes(...) bytes. */
int64_t fsr_filter_workspace_bytes(int dtype, int64_t n, int64_t r, int64_t b, int need_x);
int fsr_filter_batch(fsr_ctx* ctx, int dtype, int64_t n, int64_t r, int u_sparse,
                     const int64_t* u_indptr, const int32_t* u_indices, const void* u_values,
                     const void* u_dense, int64_t ldu, const void* w, const double* eta,
                     int64_t b, const int64_t* y_ptr, const int64_t* y_idx, const void* y_val,
                     int copy_uncovered, void* workspace, void* X, int64_t topk,
                     int64_t* top_idx, void* top_val);
/* The same with an optional 16-bit copy of U~'s column indices (r <= 65536,
 * built once by fsr_u16_columns): the single-query (b = 1) filter then
 * streams 6 instead of 8 bytes per entry, with bitwise the same sums. */
int fsr_u16_columns(fsr_ctx* ctx, int64_t nnz, const int32_t* indices, uint16_t* out);
int fsr_filter_batch_u16(fsr_ctx* ctx, int dtype, int64_t n, int64_t r, int u_sparse, const int64_t* u_indptr,
                         const int32_t* u_indices, const uint16_t* u_cols16, const void* u_values, const void* u_dense,
                         int64_t ldu, const void* w, const double* eta, int64_t b, const int64_t* y_ptr,
                         const int64_t* y_idx, const void* y_val, int copy_uncovered, void* workspace, void* X,
                         int64_t topk, int64_t* top_idx, void* top_val);
/* ---- K9e: the single-query filter on a sliced-ELL copy of U~ (csrc/k9e.cuh) ---
 * Replaces, for ONE float32 query on a sparse decomposition, the product
 * x = U~ (h(L) U~^T y) of specrank.ranking.filter (ranking.py:244-246) that
 * fsr_filter_batch computes from the CSR.  The layout (built once per
 * decomposition): rows sorted by length, descending (perm, lens), slices of
 * 32 rows stored column-major in pairs of entries (16-bit column, fp32 value;
 * slice_ptr; [j / 2][lane][j % 2]), rows
 * longer than long_len left to the CSR (sorted positions [0, n_long)).
 * fsr_sell_plan sorts and sizes (synchronises; *total_out = entries of the
 * cols / vals arrays to allocate, >= 1), fsr_sell_pack fills them.
 * fsr_filter_single_sell = fsr_filter_batch_u16 at b = 1 with the SpMV on
 * that layout; every x_i is the sequential CSR-order fmaf chain (bitwise the
 * b >= 256 kernels' sums).  r <= 16384.  fsr_filter_batch_sell: the same for
 * 1 <= b <= 64 queries (r <= 12800 when b >= 2), 2 or 4 queries per pass of
 * the layout.  The long rows' chains run through warp shuffles, so choose
 * long_len such that they hold a few percent of the entries at most. */
int64_t fsr_sell_plan_workspace_bytes(int64_t n);
int fsr_sell_plan(fsr_ctx* ctx, int64_t n, const int64_t* u_indptr, int64_t long_len, int32_t* perm, int32_t* lens,
                  int64_t* slice_ptr, void* workspace, int64_t* n_long_out, int64_t* total_out);
int fsr_sell_pack(fsr_ctx* ctx, int64_t n, const int64_t* u_indptr, const int32_t* u_indices, const float* u_values,
                  const int32_t* perm, const int64_t* slice_ptr, uint16_t* cols, float* vals);
int fsr_filter_single_sell(fsr_ctx* ctx, int64_t n, int64_t r, const int64_t* u_indptr, const int32_t* u_indices,
                           const uint16_t* u_cols16, const float* u_values, const int32_t* sell_perm,
                           const int32_t* sell_lens, const int64_t* sell_slice_ptr, const uint16_t* sell_cols,
                           const float* sell_vals, int64_t n_long, const float* w, const double* eta,
                           const int64_t* y_ptr, const int64_t* y_idx, const float* y_val, int copy_uncovered,
                           void* workspace, float* X, int64_t topk, int64_t* top_idx, float* top_val);
int fsr_filter_batch_sell(fsr_ctx* ctx, int64_t n, int64_t r, const int64_t* u_indptr, const int32_t* u_indices,
                          const uint16_t* u_cols16, const float* u_values, const int32_t* sell_perm,
                          const int32_t* sell_lens, const int64_t* sell_slice_ptr, const uint16_t* sell_cols,
                          const float* sell_vals, int64_t n_long, const float* w, const double* eta, int64_t b,
                          const int64_t* y_ptr, const int64_t* y_idx, const float* y_val, int copy_uncovered,
                          void* workspace, float* X, int64_t topk, int64_t* top_idx, float* top_val);
/* ---- K9t: the ranked-query step on tensor cores (csrc/k9t.cu) ----------------
 * Replaces, for a float32 sparse decomposition and top-k-only output, the
 * per-query loop of ranking.py:229-255 (filter) + ranking.py:390-395 (rank)[:topk]
 * for a whole batch: the same top_idx / top_val as fsr_filter_batch's unpruned
 * fp32 path, bit for bit (certified bound + exact fp32 re-score).
 * dense_u: a layout of fsr_dense_u_bytes(n, r) bytes (256-aligned) built once
 * per U~ by fsr_dense_u_build (fp16 copy of U~, n x round_up(r, 8), zeros off
 * the support, and the per-row bound factors).  workspace:
 * fsr_filter_tc_workspace_bytes(n, r, b) bytes (256-aligned); its first int is
 * the number of queries the call answered through the exact fallback
 * (fsr_filter_tc_fallback_count).  Shapes: fsr_filter_tc_applicable. */
int64_t fsr_dense_u_bytes(int64_t n, int64_t r);
int fsr_dense_u_build(fsr_ctx* ctx, int64_t n, int64_t r, const int64_t* u_indptr,
                      const int32_t* u_indices, const float* u_values, void* dense_u);
int64_t fsr_filter_tc_workspace_bytes(int64_t n, int64_t r, int64_t b);
int fsr_filter_tc_applicable(int64_t n, int64_t r, int64_t b, int64_t topk);
int fsr_filter_topk_tc(fsr_ctx* ctx, int64_t n, int64_t r, const int64_t* u_indptr,
                       const int32_t* u_indices, const float* u_values, const void* dense_u,
                       const float* w, const double* eta, int64_t b, const int64_t* y_ptr,
                       const int64_t* y_idx, const float* y_val, int copy_uncovered,
                       void* workspace, int64_t topk, int64_t* top_idx, float* top_val);
int fsr_filter_tc_fallback_count(fsr_ctx* ctx, const void* workspace, int* out);
/* Diagnostics of the last call: per query (candidate rows, rows re-scored
 * exactly), b int32 pairs to host memory (zeros for queries not finished by
 * the certified selection). */
int fsr_filter_tc_stats(fsr_ctx* ctx, int64_t n, int64_t r, int64_t b, const void* workspace, int32_t* out);

/* K9s: the same certified top-k for small batches (the tensor-core step needs
 * b >= 128 queries to amortise streaming the dense U~).  Replaces, like
 * fsr_filter_topk_tc, ranking.filter + rank (ranking.py:229-255, 390-395)
 * for a batch; the same top_idx / top_val as the unpruned sequential-order
 * fp32 path bit for bit.  stream_u: fsr_stream_u_bytes(n, r, nnz) bytes
 * (256-aligned) built once per U~ by fsr_stream_u_build (4-byte packed
 * entries fp16 value << 16 | column, r <= 65536, per-row bound factors, chunk
 * table).  workspace: fsr_filter_stream_workspace_bytes(n, r, b) bytes; its
 * first int is the fallback count (fsr_filter_tc_fallback_count) and
 * fsr_filter_tc_stats reads its diagnostics.  Shapes:
 * fsr_filter_stream_applicable. */
int64_t fsr_stream_u_bytes(int64_t n, int64_t r, int64_t nnz);
int fsr_stream_u_build(fsr_ctx* ctx, int64_t n, int64_t r, int64_t nnz, const int64_t* u_indptr,
                       const int32_t* u_indices, const float* u_values, void* stream_u);
int fsr_filter_stream_applicable(int64_t n, int64_t r, int64_t nnz, int64_t b, int64_t topk);
int64_t fsr_filter_stream_workspace_bytes(int64_t n, int64_t r, int64_t b);
int fsr_filter_topk_stream(fsr_ctx* ctx, int64_t n, int64_t r, int64_t nnz, const int64_t* u_indptr,
                           const int32_t* u_indices, const float* u_values, const void* stream_u,
                           const float* w, const double* eta, int64_t b, const int64_t* y_ptr,
                           const int64_t* y_idx, const float* y_val, int copy_uncovered,
                           void* workspace, int64_t topk, int64_t* top_idx, float* top_val);

/* Top-k of every row of X (b x n): indices/values ordered by (-x, index). */
int fsr_topk_rows(fsr_ctx* ctx, int dtype, int64_t b, int64_t n, const void* X, int64_t ldx,
                  int64_t topk, int64_t* top_idx, void* top_val);
/* K8 alone: Zt (b x r, ld r) row j = w .* U[supp y_j]^T y_j (ranking.py:219-226
 * _project; w may be NULL for no scaling).  Used by filter_pooled and the
 * embedding (ranking.py:337-387). */
int fsr_project_batch(fsr_ctx* ctx, int dtype, int64_t n, int64_t r, int u_sparse,
                      const int64_t* u_indptr, const int32_t* u_indices, const void* u_values,
                      const void* u_dense, int64_t ldu, const void* w, int64_t b,
                      const int64_t* y_ptr, const int64_t* y_idx, const void* y_val, void* Zt);

/* ---- K11: connected components  (graph.py:215-250) ----------------------
 * root[i] = the smallest vertex index of i's connected component, every
 * stored entry counting as an edge.  Host-synchronous (iterates to a fixed
 * point); *rounds_host (may be NULL) = hook/jump rounds used. */
int fsr_connected_components(fsr_ctx* ctx, int64_t n, const int64_t* indptr, const int32_t* indices,
                             int64_t* root, int64_t* rounds_host);

/* ---- K10: epilogues --------------------------------
 * FSRw (ranking.py:256-274): X[j, :] += (1 - eta) .* (V Qsum[j, :]^T) for b
 * score rows; V (n x d, ld ldv) the dataset vectors, Qsum (b x d, ld ldq) the
 * per-query sums of region vectors, eta fp64 (n). */
int fsr_fsrw_correct(fsr_ctx* ctx, int dtype, int64_t b, int64_t n, int64_t d, const void* V,
                     int64_t ldv, const void* Qsum, int64_t ldq, const double* eta, void* X,
                     int64_t ldx);
/* pooled_basis (ranking.py:329-334): U_bar (N x r, ld ldb) = P U with P the
 * (N x n) pooling CSR (values in dtype) and U dense or CSR as in
 * fsr_filter_batch.  Accumulation in CSR order (scipy's). */
int fsr_pool_rows(fsr_ctx* ctx, int dtype, int64_t N, const int64_t* p_indptr,
                  const int32_t* p_indices, const void* p_values, int64_t n, int64_t r,
                  int u_sparse, const int64_t* u_indptr, const int32_t* u_indices,
                  const void* u_values, const void* u_dense, int64_t ldu, void* Ubar, int64_t ldb);
/* pool (ranking.py:322-326) for b score rows: Xp (b x N, ld ldp) = X P^T. */
int fsr_pool_scores(fsr_ctx* ctx, int dtype, int64_t b, int64_t N, const int64_t* p_indptr,
                    const int32_t* p_indices, const void* p_values, const void* X, int64_t ldx,
                    void* Xp, int64_t ldp);
/* filter_pooled (ranking.py:337-353): Out (b x N, ld ldo) = Z A^T with A =
 * U_bar (N x k, ld lda) and Z the scaled projections (b x k, ld ldz). */
int fsr_dense_scores(fsr_ctx* ctx, int dtype, int64_t N, int64_t k, const void* A, int64_t lda,
                     int64_t b, const void* Z, int64_t ldz, void* Out, int64_t ldo);

/* ---- FSRX decomposition files ---------
 * Host buffers only.  variant: 0 exact, 1 rank_r, 2 approx, 3 sparse;
 * storage: 0 dense U (n x r float32, row-major), 1 CSR (n+1 u64 offsets, nnz
 * u32 columns, nnz float32 values).  A CRC-32 trailer covers every byte;
 * fsr_fsrx_read returns FSR_EIO on a truncated file or checksum mismatch. */
typedef struct fsr_fsrx_header {
  uint64_t n;
  uint32_t r;
  uint8_t variant;
  uint8_t storage;
  uint64_t seed;
  double alpha_hint;
  uint64_t nnz;
  uint64_t components;
} fsr_fsrx_header;
int fsr_fsrx_write(fsr_ctx* ctx, const char* path, const fsr_fsrx_header* h, const double* eigenvalues,
                   const float* U_dense, const uint64_t* indptr, const uint32_t* indices,
                   const float* values, const float* eta, const uint64_t* sizes,
                   const uint64_t* permutation);
/* Header only (sizes for the caller's buffers); no checksum verification. */
int fsr_fsrx_read_header(fsr_ctx* ctx, const char* path, fsr_fsrx_header* h);
int fsr_fsrx_read(fsr_ctx* ctx, const char* path, fsr_fsrx_header* h, double* eigenvalues,
                  float* U_dense, uint64_t* indptr, uint32_t* indices, float* values, float* eta,
                  uint64_t* sizes, uint64_t* permutation);

#ifdef __cplusplus
}
#endif

#endif /* FSR_H_ */
