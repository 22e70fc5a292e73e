/*
 * slra_cuda.h — C-ABI of the B200 (sm_100a) hot path of the `slra` library
 * (Pan–Luan–Svadlenka–Zhao, arXiv:1611.01391).
 *
 * Plain pointers and sizes only. Matrices are column-major FP64 with an
 * explicit leading dimension (the reference's Eigen::MatrixXd layout,
 * /root/reference/proj/include/slra/matrix.hpp:10); index sets are int64
 * (Eigen::Index, matrix.hpp:14). Every pointer named d_* is DEVICE memory;
 * h_* is host memory. All calls are asynchronous on the context's stream
 * unless they return data to the host (documented per call).
 *
 * Each entry point replaces one reference interface on the hot path
 * (SURVEY.md §8a); the reference file:line is cited per function. The C++
 * host layer (the headers under paper_1611_01391_b200/include/slra) keeps the reference
 * signatures and calls these; INTEGRATION.md shows the reference-side
 * dispatch a maintainer would add. There is no CPU fallback: without a CUDA
 * device every call returns SLRA_ERR_NO_DEVICE.
 */
#ifndef SLRA_CUDA_H_
#define SLRA_CUDA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes map 1:1 onto the reference's typed failures
 * (/root/reference/proj/include/slra/errors.hpp:11-33). */
enum slra_status {
  SLRA_OK = 0,
  SLRA_ERR_INVALID_ARGUMENT = 1,      /* std::invalid_argument            */
  SLRA_ERR_RANGE_FAILURE = 2,         /* RangeFailure        (lra.cpp:21) */
  SLRA_ERR_SKETCH_RANK_FAILURE = 3,   /* SketchRankFailure   (lsr.cpp:55) */
  SLRA_ERR_SELECTION_FAILURE = 4,     /* SelectionFailure    (cur.cpp:106)*/
  SLRA_ERR_GENERATOR_RANK_FAILURE = 5,/* GeneratorRankFailure(cur.cpp:157)*/
  SLRA_ERR_CUDA = 6,                  /* CUDA runtime error               */
  SLRA_ERR_NO_DEVICE = 7,             /* no CUDA device / wrong arch      */
  SLRA_ERR_UNSUPPORTED = 8,           /* shape outside the device kernels */
  SLRA_ERR_PREMULT_RANK_FAILURE = 9   /* PremultRankFailure  (lra.cpp:47) */
};

typedef struct slra_context* slra_ctx;

/* ------------------------------------------------------------ runtime */
const char* slra_status_string(int status);
/* Last CUDA error text recorded by this thread (for SLRA_ERR_CUDA). */
const char* slra_last_error(void);
/* Create a context on `device`; `stream` is a cudaStream_t (NULL = a new
 * non-blocking stream owned by the context). */
int slra_ctx_create(int device, void* stream, slra_ctx* out);
int slra_ctx_destroy(slra_ctx ctx);
int slra_ctx_synchronize(slra_ctx ctx);
void* slra_ctx_stream(slra_ctx ctx);
/* Number of kernels this context launched since creation (bench evidence). */
int64_t slra_ctx_launch_count(slra_ctx ctx);
/* Per-kernel-family device timing (CUDA events on the context stream around
 * every launch). set_timing clears the records; the report is
 * "family=ms,launches;..." summed since then. */
int slra_ctx_set_timing(slra_ctx ctx, int on);
int slra_ctx_timing_report(slra_ctx ctx, char* buf, int64_t len);
/* Stream-ordered device memory (cudaMallocAsync / cudaFreeAsync on the
 * context stream, pooled): a buffer may be freed right after the calls that
 * use it are issued on the context stream; other streams must synchronise
 * with slra_ctx_stream first. */
int slra_device_alloc(slra_ctx ctx, int64_t bytes, void** d_out);
int slra_device_free(slra_ctx ctx, void* d_ptr);
int slra_memcpy_h2d(slra_ctx ctx, void* d_dst, const void* h_src, int64_t bytes);
int slra_memcpy_d2h(slra_ctx ctx, void* h_dst, const void* d_src, int64_t bytes); /* syncs */
int slra_memcpy_d2d(slra_ctx ctx, void* d_dst, const void* d_src, int64_t bytes);
/* Page-locked host memory (cudaHostAlloc / cudaFreeHost) for results that
 * cross the bus on every call: a D2H copy into it runs at the link's rate
 * instead of through the driver's pageable staging. */
int slra_host_alloc(int64_t bytes, void** h_out);
int slra_host_free(void* h_ptr);

/* ------------------------------------------------------------ a2/a14 gathers
 * EntryOracle::rows_of / cols_of / block (testgen.cpp:11-30) and
 * select_rows / select_cols / select_block (linalg.cpp:35-52). Bit-exact. */
int slra_gather_rows(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t n,
                     const int64_t* d_I, int64_t k, double* d_R, int64_t ldr);
int slra_gather_cols(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t n,
                     const int64_t* d_J, int64_t l, double* d_C, int64_t ldc);
int slra_gather_block(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t n,
                      const int64_t* d_I, int64_t k, const int64_t* d_J, int64_t l,
                      double* d_G, int64_t ldg);

/* ------------------------------------------------------------ a3 sketches
 * A compiled sketch plan: output unit t (a column for the right-side
 * product M*H, a row for the left-side product F*W) is a signed combination
 * of `width` source columns/rows, src[t*width + s] with coefficient
 * coef[t*width + s] (exact +-1 for the in-scope kinds), evaluated in the
 * reference's order:
 *   tree = SLRA_TREE_LIST: ((c0 x0 + c1 x1) + c2 x2) + ...  — SparseCirculantOp
 *          nz-list order (sketch.cpp:250-255, 269-273); width 1 = SubIdentity.
 *   tree = SLRA_TREE_FWHT: in-place radix-2 butterfly over the width = 2^d
 *          leaves (ah_recurse, sketch.cpp:98-107), output leaf q[t].
 * The host layer compiles ColumnSlice(Product{P,D,AH}) / ColumnSlice(Z_f) /
 * Product{SubIdentity, Z_f, D} / SubIdentity into plans (only the l kept
 * outputs are computed, the sublinear form of sketch.cpp:558-567).
 * Results are bit-identical to the reference's full application. */
enum slra_tree { SLRA_TREE_LIST = 0, SLRA_TREE_FWHT = 1 };
/* out(:, t) = combine_s coef * A(:, src)  — apply(H, M, Side::Right), sketch.cpp:679-682 */
int slra_sketch_cols(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t n,
                     const int64_t* d_src, const double* d_coef, const int32_t* d_q,
                     int64_t width, int tree, int64_t l, double* d_out, int64_t ldo);
/* out(t, :) = combine_s coef * W(src, :)  — F.apply(W), sketch.cpp:520-523 */
int slra_sketch_rows(slra_ctx ctx, const double* d_W, int64_t ldw, int64_t m, int64_t ncols,
                     const int64_t* d_src, const double* d_coef, const int32_t* d_q,
                     int64_t width, int tree, int64_t k, double* d_out, int64_t ldo);
/* Row-sharded LIST-order sketch / gather:
 * d_W holds rows [row0, row0 + m_local) of the full W (ld ldw); src holds
 * GLOBAL row indices. Terms from rows held elsewhere are skipped, so the sum
 * over ranks (NCCL allreduce) equals slra_sketch_rows on the full W —
 * bit-exactly for width <= 2. transpose = 1 writes the ncols x k transpose
 * (the n x k strip A(I,:)^T that select_rows_spanning factorises). */
int slra_sketch_rows_shard(slra_ctx ctx, const double* d_W, int64_t ldw, int64_t row0,
                           int64_t m_local, int64_t ncols, const int64_t* d_src,
                           const double* d_coef, int64_t width, int64_t k, double* d_out,
                           int64_t ldo, int transpose);

/* ------------------------------------------------------------ a4/a8 small dense
 * thin_qr (linalg.cpp:67-79): Householder QR, R(i,i) >= 0, explicit thin Q.
 * Any m >= c, c <= 64 (TSQR over 256-row leaves). */
int slra_thin_qr(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t c,
                 double* d_Q, int64_t ldq, double* d_R, int64_t ldr);
/* svd (linalg.cpp:81-98): compact SVD, sigma nonincreasing, largest-|.|
 * entry of each left vector >= 0. S is m x p, T is n x p, p = min(m, n).
 * min(m,n) <= 64: one CTA (QR pre-reduction for tall inputs); larger: a
 * multi-CTA one-sided Jacobi in HBM (p <= 16384). Blocks only on arena growth. */
int slra_svd(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t n,
             double* d_S, int64_t lds, double* d_sigma, double* d_T, int64_t ldt);

/* ------------------------------------------------------------ a5/a6 pivoting
 * maxvol_rows (cur.cpp:88-116) on a tall A (m x r): ColPivHouseholderQR(A^T)
 * init + <= max_swaps+1 swap rounds. max_swaps = 0 means 4r. r <= 64; A that
 * does not fit one SM runs the grid-wide cooperative kernel. */
int slra_maxvol_rows(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t r,
                     double h, int64_t max_swaps, int64_t* d_idx);
/* select_rows_spanning (cur.cpp:118-135): thin_qr + maxvol (+ the padding
 * rows when count > c, strips up to 256 rows); optionally |det Q[idx,:]|
 * (cur.cpp:192-197). Taller strips (count == c <= 64): TSQR + grid-wide
 * maxvol. */
int slra_select_rows_spanning(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m,
                              int64_t c, int64_t count, double h, int64_t* d_idx,
                              double* d_volume);

/* ------------------------------------------------------------ a7/a8 CUR
 * primitive_cur (cur.cpp:137-162): nucleus U = T_r diag(1/sigma_r) S_r^T
 * (l x k) of the generator G = A(I,J). r <= 0 selects the adaptive rank
 * numerical_rank(G, 1e-10, Relative) (linalg.cpp:123-132; configs 3 and 5).
 * Optional factor outputs d_Tsig (l x r = T_r diag(1/sigma_r)) and d_Sr
 * (k x r) let the residual run with inner dimension r. h_r_out receives r. */
int slra_primitive_cur(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t n,
                       const int64_t* d_I, int64_t k, const int64_t* d_J, int64_t l, int64_t r,
                       double* d_nucleus, int64_t ldu, double* d_Tsig, double* d_Sr,
                       int64_t* h_r_out);
/* cross_approx (cur.cpp:201-255), stop_tol unset. init_rows (k indices)
 * must be given (the host draws them with Rng::distinct_indices exactly as
 * cur.cpp:207-209). Outputs: I (k), J (l), nucleus (l x k), the trace
 * (2*loops steps: rows k, cols l, volume proxy), adaptive r. k, l <= 64.
 * Strips that fit one SM run the whole loop in one CTA-resident kernel;
 * taller ones (config 3) use TSQR + the grid-wide cooperative maxvol per
 * half-sweep (k == l there). d_Tsig / d_Sr (nullable) receive the factored
 * nucleus as in slra_primitive_cur. Blocks until done (status is
 * host-visible). */
int slra_cross_approx(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t n,
                      int64_t r, int64_t k, int64_t l, const int64_t* d_init_rows, int loops,
                      double h, int64_t* d_I, int64_t* d_J, double* d_nucleus,
                      int64_t* d_trace_rows, int64_t* d_trace_cols, double* d_trace_volume,
                      double* d_Tsig, double* d_Sr, int64_t* h_r_out);
/* Batched cross_approx + per-block Frobenius residual: nblocks independent
 * m x n blocks at d_A + b*block_stride (ld = lda); one CTA per block (the
 * per-block ca_factors -> cross_approx -> cur_evaluate pattern of
 * hss.cpp:47-55 and cur.cpp:80-82). Per-block outputs: I (k), J (l),
 * nucleus (l x k), r, status (slra_status), resid_sq = ||B - C U R||_F^2,
 * norm_sq = ||B||_F^2. Strips must fit on one SM: m, n <= 256, k, l <= 64.
 * With k, l <= 32 and m, n multiples of 8 the residual is computed inside
 * the C-A kernel (one more pass over each block, no factors written). */
int slra_cross_approx_batched(slra_ctx ctx, const double* d_A, int64_t lda, int64_t block_stride,
                              int64_t nblocks, int64_t m, int64_t n, int64_t r, int64_t k,
                              int64_t l, const int64_t* d_init_rows, int loops, double h,
                              int64_t* d_I, int64_t* d_J, double* d_nucleus, int64_t* d_r,
                              int32_t* d_status, double* d_resid_sq, double* d_norm_sq);

/* The same over blocks in HOST memory (h_A, block b at h_A + b*block_stride),
 * the end-to-end form a host caller uses: the blocks are streamed to the
 * device in chunks on a copy stream, each chunk's C-A kernel overlapping the
 * next chunk's host-to-device copy, and the per-block results are copied
 * back into the h_* arrays (same layouts as above). Page-locked h_A makes
 * the copies asynchronous. Blocks until every result is on the host. */
int slra_cross_approx_batched_host(slra_ctx ctx, const double* h_A, int64_t lda, int64_t block_stride,
                                   int64_t nblocks, int64_t m, int64_t n, int64_t r, int64_t k,
                                   int64_t l, const int64_t* h_init_rows, int loops, double h,
                                   int64_t* h_I, int64_t* h_J, double* h_nucleus, int64_t* h_r,
                                   int32_t* h_status, double* h_resid_sq, double* h_norm_sq);
/* cross_approx (cur.cpp:201-255) over the Cauchy FunctionOracle A_ij =
 * 1/(x_i - y_j) (config 3's FMM-style block, oracle.hpp:43-54): the same
 * selections and nucleus as slra_cross_approx on the materialised matrix
 * (bit for bit), with the strips and the generator evaluated from the
 * points x (m), y (n) — device pointers — instead of gathered from HBM.
 * k == l <= 64 when m or n > 256. */
int slra_cross_approx_cauchy(slra_ctx ctx, const double* d_x, const double* d_y, int64_t m, int64_t n, int64_t r,
                             int64_t k, int64_t l, const int64_t* d_init_rows, int loops, double h, int64_t* d_I,
                             int64_t* d_J, double* d_nucleus, int64_t* d_trace_rows, int64_t* d_trace_cols,
                             double* d_trace_vol, double* d_Tsig, double* d_Sr, int64_t* h_r_out);
/* cur_evaluate(M, c, Frobenius) (cur.cpp:76-82) for the Cauchy oracle with
 * the factored nucleus: C, R evaluated, the full pass over A evaluates its
 * tiles (cauchy_residual_stream_kernel). d_out[0..1] = resid_sq, norm_sq. */
int slra_cur_residual_factored_cauchy(slra_ctx ctx, const double* d_x, const double* d_y, int64_t m, int64_t n,
                                      const int64_t* d_I, int64_t k, const int64_t* d_J, int64_t l,
                                      const double* d_Tsig, const double* d_Sr, int64_t r, double* d_out);
/* cross_approx_batched over log-kernel blocks given by their points
 * (FunctionOracle, oracle.hpp:43-54; the config-5 recipe K_ij =
 * 0.5 log((p_i - q_j)^2), hss.cpp:47-55 pattern): the same C-A per block as
 * slra_cross_approx_batched, every entry the algorithm reads evaluated on
 * the fly (the strips, the generator, the residual's full pass) instead of
 * read from a materialised block — bit-identical entries to
 * slra_gen_log_kernel_blocks, hence identical results. Points per block:
 * px, py (nblocks x m), qx, qy (nblocks x n), device. k, l <= 32 and
 * m, n multiples of 8 (the residual is fused), else SLRA_ERR_UNSUPPORTED. */
int slra_cross_approx_batched_logkernel(slra_ctx ctx, const double* d_px, const double* d_py, const double* d_qx,
                                        const double* d_qy, int64_t nblocks, int64_t m, int64_t n, int64_t r,
                                        int64_t k, int64_t l, const int64_t* d_init_rows, int loops, double h,
                                        int64_t* d_I, int64_t* d_J, double* d_nucleus, int64_t* d_r,
                                        int32_t* d_status, double* d_resid_sq, double* d_norm_sq);
/* The same from host buffers (pinned for overlap): the points stream to the
 * device in eight chunks on a copy stream while the previous chunk is
 * factorised; results come back as in slra_cross_approx_batched_host. */
int slra_cross_approx_batched_logkernel_host(slra_ctx ctx, const double* h_px, const double* h_py,
                                             const double* h_qx, const double* h_qy, int64_t nblocks, int64_t m,
                                             int64_t n, int64_t r, int64_t k, int64_t l, const int64_t* h_init_rows,
                                             int loops, double h, int64_t* h_I, int64_t* h_J, double* h_nucleus,
                                             int64_t* h_r, int32_t* h_status, double* h_resid_sq,
                                             double* h_norm_sq);

/* ------------------------------------------------------------ a13 input generator
 * Config-5 log-kernel blocks (testgen: K_ij = log|p_i - q_j| =
 * 0.5 log(dx^2 + dy^2), FunctionOracle recipe oracle.hpp:43-54) materialised
 * on the device from per-block points drawn on the host: block b reads
 * d_px/d_py[b*m + i], d_qx/d_qy[b*n + j] and writes d_A + b*block_stride
 * (column-major, ld = lda). Untimed setup, not the hot path. */
int slra_gen_log_kernel_blocks(slra_ctx ctx, const double* d_px, const double* d_py, const double* d_qx,
                               const double* d_qy, int64_t nblocks, int64_t m, int64_t n, double* d_A,
                               int64_t lda, int64_t block_stride);

/* ------------------------------------------------------------ a9 residual
 * ||A - P Q||_F^2 and ||A||_F^2 in one pass over A (FP64 DMMA tiles fused
 * with subtract-square-reduce, deterministic two-stage reduction).
 * P is m x inner (ldp), Q is inner x n (ldq). Results land in DEVICE
 * doubles d_out[0] = resid_sq, d_out[1] = norm_sq. */
int slra_lowrank_residual(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t n,
                          const double* d_P, int64_t ldp, const double* d_Q, int64_t ldq,
                          int64_t inner, double* d_out);
/* cur_evaluate(M, c, Frobenius) (cur.cpp:80-82): ||A - A(:,J) U A(I,:)||_F.
 * Returns resid_sq and norm_sq to the host (blocks). */
int slra_cur_residual(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t n,
                      const int64_t* d_I, int64_t k, const int64_t* d_J, int64_t l,
                      const double* d_nucleus, int64_t ldu, double* h_resid_sq,
                      double* h_norm_sq);
/* The same residual with the nucleus in its factored form U = Tsig Sr^T
 * (Tsig l x r, Sr k x r, as returned by slra_primitive_cur): the pass over A
 * runs at inner dimension r instead of k. d_out[0..1] = resid_sq, norm_sq. */
int slra_cur_residual_factored(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t n,
                               const int64_t* d_I, int64_t k, const int64_t* d_J, int64_t l,
                               const double* d_Tsig, const double* d_Sr, int64_t r,
                               double* d_out);

/* ------------------------------------------------------------ GEMM
 * C = alpha op(A) op(B) + beta C, FP64 DMMA (mma.sync m8n8k4). trans = 0/1. */
int slra_gemm(slra_ctx ctx, int transA, int transB, int64_t m, int64_t n, int64_t k, double alpha,
              const double* d_A, int64_t lda, const double* d_B, int64_t ldb, double beta,
              double* d_C, int64_t ldc);

/* ------------------------------------------------------------ a10 range finder
 * range_finder (lra.cpp:31-39) with the sketch H given as a compiled
 * right-side plan (see slra_sketch_cols). variant 0 = BasisQr (U = Q of MH,
 * m x l; V = U^T M), 1 = TruncatedRankR (U = S_r Sigma_r, m x r; V = U^+ M).
 * Also returns the residual ||M - U V||_F^2 and ||M||_F^2 (d_out[0..1]),
 * and the sketch singular values (l). Blocks (rank check is host-visible);
 * SLRA_ERR_RANGE_FAILURE when numerical_rank(MH, 1e-10, Relative) < r. */
int slra_range_finder(slra_ctx ctx, const double* d_M, int64_t ldm, int64_t m, int64_t n,
                      const int64_t* d_src, const double* d_coef, const int32_t* d_q,
                      int64_t width, int tree, int64_t l, int64_t r, int variant, double* d_U,
                      int64_t ldu, double* d_V, int64_t ldv, double* d_out,
                      double* d_sigma);
/* The same for nsk sketches of one M in one call (their factorisations run
 * concurrently, one CTA per sketch). h_* are HOST arrays of nsk entries
 * (device pointers / sizes); d_out holds 2*nsk doubles, d_sigma nsk*l. With
 * h_status non-null a rank failure is reported per sketch (SLRA_OK or
 * SLRA_ERR_RANGE_FAILURE) and the call returns SLRA_OK. For variant 1 the
 * singular values below the rank cut are upper bounds (Jacobi deflation). */
int slra_range_finder_batched(slra_ctx ctx, const double* d_M, int64_t ldm, int64_t m, int64_t n,
                              int nsk, const int64_t* const* h_src, const double* const* h_coef,
                              const int32_t* const* h_q, const int64_t* h_width, const int* h_tree,
                              int64_t l, int64_t r, int variant, double* const* h_U, int64_t ldu,
                              double* const* h_V, int64_t ldv, double* d_out, double* d_sigma,
                              int32_t* h_status);

/* ------------------------------------------------------------ §8f range-finder variants
 * pseudo_inverse (linalg.cpp:111-121): P = A^+ (n x m) through the SVD,
 * sigma below rank_tol * sigma_0 dropped; *h_rank = the kept count (so with
 * rank_tol = tol it is numerical_rank(A, tol, Relative)). Shapes as slra_svd. */
int slra_pinv(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t n, double rank_tol,
              double* d_P, int64_t ldp, int64_t* h_rank);
/* primitive_cur's qr_nucleus branch (cur.cpp:146-152): P = G^+ (l x k) of a
 * k x l generator through Eigen's CompleteOrthogonalDecomposition (ColPivQR,
 * RZ step at the default rank, setThreshold(threshold) before rank() and
 * pseudoInverse()); *h_rank = cod.rank() at `threshold` (the caller throws
 * GeneratorRankFailure when it is below r). k, l <= 4096. Blocks when
 * h_rank is set. */
int slra_cod_pinv(slra_ctx ctx, const double* d_G, int64_t ldg, int64_t k, int64_t l, double threshold,
                  double* d_P, int64_t ldp, int64_t* h_rank);
/* lra_premult (lra.cpp:41-52): U = range_basis(M, H, r, variant) as in
 * slra_range_finder (H: right plan, l outputs), then V = (F U)^+ (F M) with F
 * a compiled LEFT plan of s rows (see slra_sketch_rows). U is m x l (variant
 * 0) or m x r (variant 1); V is that many rows x n. d_out (optional) gets
 * ||M - U V||_F^2 and ||M||_F^2. SLRA_ERR_RANGE_FAILURE as range_finder;
 * SLRA_ERR_PREMULT_RANK_FAILURE when numerical_rank(F U, 1e-10, Relative) < r.
 * min(s, cols of U) <= 64. Blocks. */
int slra_lra_premult(slra_ctx ctx, const double* d_M, int64_t ldm, int64_t m, int64_t n,
                     const int64_t* d_hsrc, const double* d_hcoef, const int32_t* d_hq,
                     int64_t h_width, int h_tree, int64_t l, const int64_t* d_fsrc,
                     const double* d_fcoef, const int32_t* d_fq, int64_t f_width, int f_tree,
                     int64_t s, int64_t r, int variant, double* d_U, int64_t ldu, double* d_V,
                     int64_t ldv, double* d_out);
/* two_stage_truncate (lra.cpp:54-63): Q R = thin_qr(U) (U m x l), core =
 * svd(R V) (V l x n), U' = Q S_r diag(sigma_r) (m x r), V' = T_r^T (r x n).
 * 1 <= r <= min(l, n), l <= min(m, 64). */
int slra_two_stage_truncate(slra_ctx ctx, const double* d_U, int64_t ldu, int64_t m, int64_t l,
                            const double* d_V, int64_t ldv, int64_t n, int64_t r, double* d_Uo,
                            int64_t lduo, double* d_Vo, int64_t ldvo);

/* ------------------------------------------------------------ §8f HSS (hss.cpp)
 * Packed, level-major HSS representation of an n x n matrix at depth L
 * (n divisible by 2^L, leaf = n / 2^L >= r): at level l the 2^(l+1)
 * off-diagonal blocks (node t: upper block b = 2t, rows [t s, t s + s/2) x
 * cols [t s + s/2, (t+1) s); lower b = 2t + 1, the transposed position;
 * s = n / 2^l) have disjoint row ranges tiling [0, n) and disjoint column
 * ranges, so
 *   d_F  + l n r : F_l  (n x r, ld n), F_l(row0_b + i, a) = F_b(i, a)
 *   d_HT + l n r : HT_l (n x r, ld n), HT_l(col0_b + j, a) = H_b(a, j)
 *   d_D          : n x leaf (ld n), D(i, j) = M(i, leaf0(i) + j)
 *   rank[g]      : g = 2^(l+1) - 2 + b (level-major), rank_b <= r.
 * The reference's block order (hss.cpp:151-160, preorder: upper, lower,
 * left subtree, right subtree) is a permutation of g.
 *
 * build_hss(M, L, r, tol, Svd) (hss.cpp:69-96, 143-185): every block's SVD
 * (one-CTA Jacobi for s/2 <= 64, multi-CTA otherwise), the smallest rank
 * <= min(r, s/2) whose discarded tail is <= tol ||sigma||, overflow flags
 * (h_overflow[g]) where rank r misses tol. h_rank/h_overflow are HOST arrays
 * of 2^(L+1) - 2 entries. Blocks (one host read of the singular values). */
int slra_hss_build_svd(slra_ctx ctx, const double* d_M, int64_t ldm, int64_t n, int L, int64_t r,
                       double tol, double* d_D, double* d_F, double* d_HT, int64_t* h_rank,
                       int32_t* h_overflow);
/* The dense diagonal leaves only (hss.cpp:145-148), as d_D above. */
int slra_hss_leaves(slra_ctx ctx, const double* d_M, int64_t ldm, int64_t n, int L, double* d_D);
/* hss_matvec (hss.cpp:193-212): y = HSS x; d_rank is the DEVICE copy of the
 * rank array. Two kernels: the 2^(L+1)-2 projections H_b x_b, then one
 * thread per row adds its leaf product and its L generator terms in the
 * reference's order (leaf first, then by level). */
int slra_hss_matvec(slra_ctx ctx, int64_t n, int L, int64_t r, const double* d_D, const double* d_F,
                    const double* d_HT, const int64_t* d_rank, const double* d_x, double* d_y);
/* hss_reconstruct (hss.cpp:214-221) into d_out (n x n, ld ldo); with d_M
 * non-null writes M - reconstruction instead (hss_error's operand). */
int slra_hss_reconstruct(slra_ctx ctx, int64_t n, int L, int64_t r, const double* d_D, const double* d_F,
                         const double* d_HT, const int64_t* d_rank, const double* d_M, int64_t ldm,
                         double* d_out, int64_t ldo);
/* matrix_norm (linalg.cpp:134-151): kind 0 spectral (largest singular
 * value), 1 Frobenius, 2 Chebyshev (max |a_ij|). Blocks; *h_out on the host. */
int slra_matrix_norm(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t n, int kind,
                     double* h_out);

/* ------------------------------------------------------------ §8f leverage-score CUR
 * (leverage.cpp:12-149) elementwise passes; the SVDs are slra_svd, the
 * gathers slra_gather_*, the sampling itself draws from the host Rng.
 * out[i] = sum_j A(i,j)^2 / divisor (svd_leverage_scores: divisor = r). */
int slra_row_sqnorms(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t n, double divisor,
                     double* d_out);
/* B = diag(dr) A diag(dc), evaluated (dr_i A_ij) dc_j; null dr/dc = identity.
 * B may alias A when ldb == lda. */
int slra_scale_rows_cols(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t n,
                         const double* d_dr, const double* d_dc, double* d_B, int64_t ldb);
/* InverseBidiagonalOp (sketch.cpp:286-331) on the c columns of X (n rows):
 * forward y_0 = x_0, y_i = x_i + b[i-1] y_{i-1}; backward y_{n-1} = x_{n-1},
 * y_i = x_i + b[i] y_{i+1}. Sequential per column in the reference's order
 * (bit-exact for b = +-1); Y may alias X. */
/* AbridgedFourierOp (sketch.cpp:137-211) on a complex n x c operand held as
 * real / imaginary planes (ld, ldo): d butterfly levels (transpose = 0:
 * af_recurse, 1: af_recurse_transpose). d_twr / d_twi hold the twiddles
 * exp(i 2 pi k / L) level after level (L = n >> s, k < L / 2), as the
 * reference computes them on the host. 2^d must divide n. */
int slra_af_apply(slra_ctx ctx, const double* d_re, const double* d_im, int64_t ld, int64_t n, int64_t c,
                  int d, const double* d_twr, const double* d_twi, int transpose, double* d_ore,
                  double* d_oim, int64_t ldo);
int slra_bidiag_scan(slra_ctx ctx, const double* d_X, int64_t ldx, int64_t n, int64_t c,
                     const double* d_b, int forward, double* d_Y, int64_t ldy);
/* Y = alpha X + beta Y, one rounding per entry (SumOp accumulation,
 * sketch.cpp:469-475). beta = 0 ignores Y's previous contents. */
int slra_axpby(slra_ctx ctx, double alpha, const double* d_X, int64_t ldx, double beta, double* d_Y,
               int64_t ldy, int64_t m, int64_t n);
/* B = A^T (n x m, ld ldb), 32 x 32 shared-memory tiles. */
int slra_transpose(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t n, double* d_B,
                   int64_t ldb);

/* ------------------------------------------------------------ a11/a12 LSR
 * sketch_solve (lsr.cpp:37-67): FW = F (A|b) through a compiled left-side
 * plan (k rows), then min ||FA x - Fb||: a Gram/Cholesky solve with one
 * refinement step when FA is well conditioned (every Cholesky pivot above
 * 1e-6 of its column's squared norm), otherwise the reference's own
 * column-pivoted Householder QR of FA (threshold 1e-10;
 * SLRA_ERR_SKETCH_RANK_FAILURE exactly when its rank() < d) and its solve.
 * h_sketched_residual = ||FA x_hat - Fb||. d <= 768. Blocks (one host
 * synchronisation, at the end). */
int slra_sketch_solve(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t d,
                      const double* d_b, const int64_t* d_src, const double* d_coef,
                      const int32_t* d_q, int64_t width, int tree, int64_t k, double* d_x_hat,
                      double* h_sketched_residual);
/* The solve half of sketch_solve (lsr.cpp:52-60) for an already sketched
 * system FW = (FA | Fb), k x (d+1), ld k — the row-sharded path (config 4)
 * all-reduces the per-rank sketch contributions and then calls this. */
/* sketch_solve (lsr.cpp:37-67) for nsk <= 4 sketches F_s of the same (A, b)
 * — config 4's two samplers: the per-sketch gathers and Grams, then one
 * launch of each cluster kernel solves all of them side by side (a cluster
 * per sketch) with one host synchronisation; results identical to nsk
 * separate slra_sketch_solve calls. Host arrays of device pointers (src,
 * coef, q, x_hat) and of sizes; h_sketched_residual[s] (host, nullable). */
int slra_sketch_solve_batched(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t d,
                              const double* d_b, int nsk, const int64_t* const* d_src,
                              const double* const* d_coef, const int32_t* const* d_q, const int64_t* width,
                              const int* tree, int64_t k, double* const* d_x_hat, double* h_sketched_residual);
int slra_lsr_solve_sketched(slra_ctx ctx, const double* d_FW, int64_t ldfw, int64_t k, int64_t d,
                            double* d_x_hat, double* h_sketched_residual);
/* solve_exact (lsr.cpp:21-24): x = pinv(A) b, the minimum-norm least-squares
 * solution with the pseudo-inverse's cut sigma_i > 1e-10 sigma_1
 * (linalg.cpp:111-121). Well-conditioned A: the normal-equation solve (one
 * refinement step); otherwise the column-pivoted Householder QR A P = Q R and
 * pinv(R) (sigma(R) = sigma(A)). Never reports a rank failure; *h_rank = the
 * kept singular values (d on the fast path). d <= 768. Blocks. */
int slra_lsq_exact(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t d, const double* d_b,
                   double* d_x, int64_t* h_rank);
/* residual_norm (lsr.cpp:26-28): ||A x - b||^2 into d_out[0] (device). */
int slra_lsr_residual(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t d,
                      const double* d_b, const double* d_x, double* d_out);
/* residual_norm (lsr.cpp:26-28) for nx <= 4 candidate solutions at once
 * (the columns of d_X, ld d): d_out[s] = ||A x_s - b||^2, A read ONCE — the
 * two samplers of config 4 certified in one pass over the 2^20 x 256 A. */
int slra_lsr_residual_multi(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t d,
                            const double* d_b, const double* d_X, int64_t nx, double* d_out);

/* ------------------------------------------------------------ §8b/§8e multi-GPU
 * NCCL collectives (NVLink / NVSwitch on one box) on the context's stream
 * for the row-sharded configurations: config 4's single all-reduce of the
 * k x (d+1) sketched rows (lsr.cpp:44-50 sharded by rows), config 3's
 * per-half-sweep strip exchange (cur.cpp:215-236) and the residual partials.
 * One process per GPU; rank 0 makes the id and hands it to the others out of
 * band (e.g. over the launcher's store). NCCL is loaded at first use
 * (dlopen libnccl.so.2); without it these return SLRA_ERR_UNSUPPORTED.
 * Collectives order with the kernels on the same stream (no host sync). */
typedef struct slra_comm_s* slra_comm;
#define SLRA_COMM_ID_BYTES 128
int slra_comm_available(void);
int slra_comm_unique_id(void* h_id); /* SLRA_COMM_ID_BYTES bytes */
int slra_comm_init(slra_ctx ctx, int nranks, int rank, const void* h_id, slra_comm* out);
int slra_comm_destroy(slra_comm comm);
int slra_comm_size(slra_comm comm);
int slra_comm_rank(slra_comm comm);
int slra_comm_allreduce_sum(slra_comm comm, const double* d_send, double* d_recv, int64_t count);
int slra_comm_allreduce_max(slra_comm comm, const double* d_send, double* d_recv, int64_t count);
/* d_recv = the ranks' d_send blocks (count_per_rank each) in rank order */
int slra_comm_allgather(slra_comm comm, const double* d_send, double* d_recv, int64_t count_per_rank);
int slra_comm_broadcast(slra_comm comm, double* d_buf, int64_t count, int root);

#ifdef __cplusplus
}
#endif
#endif /* SLRA_CUDA_H_ */
