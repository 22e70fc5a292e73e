// Range-finder variants of §8f: pseudo_inverse (linalg.cpp:111-121),
// lra_premult (lra.cpp:41-52) and two_stage_truncate (lra.cpp:54-63), composed
// from the device kernels of the range finder (sketch plans, CholeskyQR3/TSQR,
// one-CTA Jacobi SVD, DMMA GEMM). Operands stay in HBM; the only host reads
// are the singular values that decide ranks (the reference's own branch
// points).
#include <vector>

#include "common.cuh"

namespace slra_dev {

int range_finder_core(Context* cx, const double* M, int64_t ldm, int64_t m, int64_t n, int nsk,
                      const int64_t* const* h_src, const double* const* h_coef, const int32_t* const* h_q,
                      const int64_t* h_width, const int* h_tree, int64_t l, int64_t r, int variant,
                      double* const* h_U, int64_t ldu, double* const* h_V, int64_t ldv, double* d_out,
                      double* d_sigma, int32_t* h_status, bool want_v);
int launch_sketch_rows(Context* c, const double* Wm, int64_t ldw, int64_t ncols, const int64_t* src,
                       const double* coef, const int32_t* q, int64_t width, int tree, int64_t k, double* out,
                       int64_t ldo);
int launch_svd(Context* cx, const double* A, int64_t lda, int64_t m, int64_t n, double* S, int64_t lds,
               double* sigma, double* T, int64_t ldt);
int launch_gemm_fam(Context* c, const char* fam, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha,
                    const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* Cm, int64_t ldc);
int launch_transpose(Context* cx, const double* A, int64_t lda, int64_t m, int64_t n, double* B, int64_t ldb);
int launch_lowrank_residual(Context* c, const double* A, int64_t lda, int64_t m, int64_t n, const double* P,
                            int64_t ldp, const double* Q, int64_t ldq, int64_t inner, double* d_out);

namespace {

// Y(:, j) = X(:, j) * f_j with f_j = s[j] or 1 / s[j] (Eigen's cwiseInverse,
// then the diagonal product: one multiply by the reciprocal).
__global__ void scale_cols_kernel1(const double* __restrict__ X, int64_t ldx, int64_t m, int64_t cols,
                                   const double* __restrict__ s, int inv, double* __restrict__ Y, int64_t ldy) {
  const int64_t total = m * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    const double f = inv ? 1.0 / s[j] : s[j];
    Y[i + j * ldy] = X[i + j * ldx] * f;
  }
}

int launch_scale_cols(Context* cx, const double* X, int64_t ldx, int64_t m, int64_t cols, const double* s, int inv,
                      double* Y, int64_t ldy) {
  if (m * cols == 0) return SLRA_OK;
  int64_t g = ceil_div(m * cols, 256);
  if (g > cx->num_sms * 4) g = cx->num_sms * 4;
  SLRA_TIMED(cx, "scale", scale_cols_kernel1<<<(unsigned)g, 256, 0, cx->stream>>>(X, ldx, m, cols, s, inv, Y, ldy);)
  SLRA_CHECK_LAUNCH(cx);
  return SLRA_OK;
}

// Count of sigma above rel_tol * sigma_0 (numerical_rank, Relative mode;
// also pseudo_inverse's rho): one small read-back.
int read_rank(Context* cx, const double* sig, int64_t p, double rel_tol, int64_t* rank) {
  std::vector<double> h((size_t)p);
  SLRA_CUDA(cudaMemcpyAsync(h.data(), sig, 8 * p, cudaMemcpyDeviceToHost, cx->stream));
  SLRA_CUDA(cudaStreamSynchronize(cx->stream));
  int64_t c = 0;
  if (p > 0 && h[0] != 0.0)
    for (int64_t i = 0; i < p; ++i) c += h[(size_t)i] > rel_tol * h[0] ? 1 : 0;
  *rank = c;
  return SLRA_OK;
}

}  // namespace

// P = A^+ (n x m) = T_rho diag(1/sigma_rho) S_rho^T; ws holds
// S (m x p), sigma (p), T (n x p), TS (n x p).
int launch_pinv(Context* cx, const double* A, int64_t lda, int64_t m, int64_t n, double rank_tol, double* P,
                int64_t ldp, double* ws, int64_t* rho_out) {
  const int64_t p = m < n ? m : n;
  double* S = ws;
  double* sig = S + m * p;
  double* T = sig + p;
  double* TS = T + n * p;
  SLRA_TRY(launch_svd(cx, A, lda, m, n, S, m, sig, T, n));
  int64_t rho = 0;
  SLRA_TRY(read_rank(cx, sig, p, rank_tol, &rho));
  if (rho_out) *rho_out = rho;
  if (rho == 0) {  // zero matrix (linalg.cpp:113-118)
    SLRA_CUDA(cudaMemset2DAsync(P, 8 * ldp, 0, 8 * n, m, cx->stream));
    return SLRA_OK;
  }
  SLRA_TRY(launch_scale_cols(cx, T, n, n, rho, sig, 1, TS, n));
  return launch_gemm_fam(cx, "gemm_pinv", 0, 1, n, m, rho, 1.0, TS, n, S, m, 0.0, P, ldp);
}

size_t pinv_workspace_doubles(int64_t m, int64_t n) {
  const int64_t p = m < n ? m : n;
  return (size_t)(m * p + p + 2 * n * p);
}

}  // namespace slra_dev

using namespace slra_dev;

extern "C" {

int slra_pinv(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t n, double rank_tol, double* P,
              int64_t ldp, int64_t* h_rank) {
  if (!ctx || m < 1 || n < 1 || lda < m || ldp < n || !(rank_tol >= 0.0)) return SLRA_ERR_INVALID_ARGUMENT;
  Context* cx = C(ctx);
  double* ws = static_cast<double*>(arena(cx, 8, sizeof(double) * pinv_workspace_doubles(m, n)));
  if (!ws) return SLRA_ERR_CUDA;
  return launch_pinv(cx, A, lda, m, n, rank_tol, P, ldp, ws, h_rank);
}

int slra_lra_premult(slra_ctx ctx, const double* M, int64_t ldm, int64_t m, int64_t n, const int64_t* h_src,
                     const double* h_coef, const int32_t* h_q, int64_t h_width, int h_tree, int64_t l,
                     const int64_t* f_src, const double* f_coef, const int32_t* f_q, int64_t f_width, int f_tree,
                     int64_t s, int64_t r, int variant, double* U, int64_t ldu, double* V, int64_t ldv,
                     double* d_out) {
  if (!ctx || s < 1 || f_width < 1) return SLRA_ERR_INVALID_ARGUMENT;
  Context* cx = C(ctx);
  const int64_t uc = variant == 1 ? r : l;
  if (ldv < uc || ldu < m) return SLRA_ERR_INVALID_ARGUMENT;
  // U = range_basis(M, H, r, variant) (lra.cpp:45), RangeFailure included
  SLRA_TRY(range_finder_core(cx, M, ldm, m, n, 1, &h_src, &h_coef, &h_q, &h_width, &h_tree, l, r, variant, &U, ldu,
                             &V, ldv, nullptr, nullptr, nullptr, false));
  const int64_t p = s < uc ? s : uc;
  if (p > 64) return SLRA_ERR_UNSUPPORTED;
  const size_t need = (size_t)(s * uc + s * n + uc * s);
  double* buf = static_cast<double*>(arena(cx, 9, sizeof(double) * need));
  double* pw = static_cast<double*>(arena(cx, 8, sizeof(double) * pinv_workspace_doubles(s, uc)));
  if (!buf || !pw) return SLRA_ERR_CUDA;
  double* FU = buf;            // s x uc
  double* FM = FU + s * uc;    // s x n
  double* Pf = FM + s * n;     // uc x s = (F U)^+
  SLRA_TRY(launch_sketch_rows(cx, U, ldu, uc, f_src, f_coef, f_q, f_width, f_tree, s, FU, s));
  // numerical_rank(FU, 1e-10, Relative) < r -> PremultRankFailure (lra.cpp:47-48);
  // pseudo_inverse's default cut is the same 1e-10 * sigma_0, so one SVD serves both
  int64_t rank = 0;
  SLRA_TRY(launch_pinv(cx, FU, s, s, uc, 1e-10, Pf, uc, pw, &rank));
  if (rank < r) return SLRA_ERR_PREMULT_RANK_FAILURE;
  SLRA_TRY(launch_sketch_rows(cx, M, ldm, n, f_src, f_coef, f_q, f_width, f_tree, s, FM, s));
  SLRA_TRY(launch_gemm_fam(cx, "gemm_v", 0, 0, uc, n, s, 1.0, Pf, uc, FM, s, 0.0, V, ldv));
  if (d_out) SLRA_TRY(launch_lowrank_residual(cx, M, ldm, m, n, U, ldu, V, ldv, uc, d_out));
  return SLRA_OK;
}

int slra_two_stage_truncate(slra_ctx ctx, const double* U, int64_t ldu, int64_t m, int64_t l, const double* V,
                            int64_t ldv, int64_t n, int64_t r, double* Uo, int64_t lduo, double* Vo, int64_t ldvo) {
  if (!ctx || r < 1 || r > l || l > m || r > n || ldu < m || ldv < l || lduo < m || ldvo < r)
    return SLRA_ERR_INVALID_ARGUMENT;
  if (l > 64) return SLRA_ERR_UNSUPPORTED;
  Context* cx = C(ctx);
  const int64_t p = l < n ? l : n;
  const size_t need = (size_t)(m * l + l * l + l * n + l * p + p + n * p);
  double* buf = static_cast<double*>(arena(cx, 9, sizeof(double) * need));
  if (!buf) return SLRA_ERR_CUDA;
  double* Q = buf;         // m x l
  double* R = Q + m * l;   // l x l
  double* RV = R + l * l;  // l x n
  double* S = RV + l * n;  // l x p
  double* sig = S + l * p;
  double* T = sig + p;     // n x p
  // Q, R = thin_qr(U); core = svd(R V) (lra.cpp:56-57)
  SLRA_TRY(slra_thin_qr(ctx, U, ldu, m, l, Q, m, R, l));
  SLRA_TRY(launch_gemm_fam(cx, "gemm_core", 0, 0, l, n, l, 1.0, R, l, V, ldv, 0.0, RV, l));
  SLRA_TRY(launch_svd(cx, RV, l, l, n, S, l, sig, T, n));
  // U' = (Q S_r) diag(sigma_r); V' = T_r^T (lra.cpp:59-60)
  SLRA_TRY(launch_gemm_fam(cx, "gemm_u", 0, 0, m, r, l, 1.0, Q, m, S, l, 0.0, Uo, lduo));
  SLRA_TRY(launch_scale_cols(cx, Uo, lduo, m, r, sig, 0, Uo, lduo));
  return launch_transpose(cx, T, n, n, r, Vo, ldvo);
}

}  // extern "C"
