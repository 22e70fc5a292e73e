// Orchestration of the multi-kernel entry points: cur_evaluate(Frobenius)
// (cur.cpp:76-82) and range_finder (lra.cpp:14-39). Everything stays on the
// device; only rank/status decisions are read back.
#include "common.cuh"

namespace slra_dev {

int launch_gather_cols(Context* c, const double* A, int64_t lda, int64_t m, const int64_t* J, int64_t l, double* Cm,
                       int64_t ldc);
int launch_gather_rows(Context* c, const double* A, int64_t lda, int64_t n, const int64_t* I, int64_t k, double* R,
                       int64_t ldr);
int launch_sketch_cols(Context* c, const double* A, int64_t lda, int64_t m, const int64_t* src, const double* coef,
                       const int32_t* q, int64_t width, int tree, int64_t l, double* out, int64_t ldo);
int launch_gemm_fam(Context* c, const char* fam, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha,
                    const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* Cm, int64_t ldc);
int launch_gemm(Context* c, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
                int64_t lda, const double* B, int64_t ldb, double beta, double* Cm, int64_t ldc);
int launch_lowrank_residual(Context* c, const double* A, int64_t lda, int64_t m, int64_t n, const double* P,
                            int64_t ldp, const double* Q, int64_t ldq, int64_t inner, double* d_out);
int launch_thin_qr(Context* cx, const double* A, int64_t lda, int64_t m, int c, double* Q, int64_t ldq, double* R,
                   int64_t ldr);
int launch_svd_small(Context* cx, const double* A, int64_t lda, int m, int n, double* S, int64_t lds, double* sigma,
                     double* T, int64_t ldt, double deflate);
int launch_colsign(Context* cx, double* S, int64_t lds, int64_t m, double* T, int64_t ldt, int64_t n, int64_t cols);

// Scale columns: X(:, j) *= s[j] (or 1/s[j] when inv).
__global__ void scale_cols_kernel(double* __restrict__ X, int64_t ldx, int64_t m, int64_t cols,
                                  const double* __restrict__ s, int inv, double* __restrict__ Y, int64_t ldy) {
  const int64_t total = m * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    const double f = inv ? 1.0 / s[j] : s[j];
    Y[i + j * ldy] = X[i + j * ldx] * f;
  }
}

int launch_scale_cols(Context* c, double* X, int64_t ldx, int64_t m, int64_t cols, const double* s, int inv,
                      double* Y, int64_t ldy) {
  int g = ceil_div(m * cols, 256);
  if (g > c->num_sms * 8) g = c->num_sms * 8;
  if (g < 1) g = 1;
  SLRA_TIMED(c, "scale", scale_cols_kernel<<<g, 256, 0, c->stream>>>(X, ldx, m, cols, s, inv, Y, ldy);)
  SLRA_CHECK_LAUNCH(c);
  return SLRA_OK;
}

}  // namespace slra_dev

using namespace slra_dev;

extern "C" {

int slra_cur_residual(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t n, const int64_t* I, int64_t k,
                      const int64_t* J, int64_t l, const double* U, int64_t ldu, double* h_resid_sq,
                      double* h_norm_sq) {
  if (!ctx || lda < m || ldu < l || k < 1 || l < 1) return SLRA_ERR_INVALID_ARGUMENT;
  Context* cx = C(ctx);
  // ws: C (m x l) | R (k x n) | CU (m x k) | out (2)
  const size_t need = (size_t)m * l + (size_t)k * n + (size_t)m * k + 8;
  double* ws = static_cast<double*>(arena(cx, 1, sizeof(double) * need));
  if (!ws) return SLRA_ERR_CUDA;
  double* Cm = ws;
  double* Rm = Cm + (size_t)m * l;
  double* CU = Rm + (size_t)k * n;
  double* out = CU + (size_t)m * k;
  int st = launch_gather_cols(cx, A, lda, m, J, l, Cm, m);
  if (st == SLRA_OK) st = launch_gather_rows(cx, A, lda, n, I, k, Rm, k);
  // (C U) R, Eigen's left-to-right evaluation (cur.cpp:76-78)
  if (st == SLRA_OK) st = launch_gemm(cx, 0, 0, m, k, l, 1.0, Cm, m, U, ldu, 0.0, CU, m);
  if (st == SLRA_OK) st = launch_lowrank_residual(cx, A, lda, m, n, CU, m, Rm, k, k, out);
  double* hs = static_cast<double*>(cx->hsmall);
  if (st == SLRA_OK) cudaMemcpyAsync(hs, out, 16, cudaMemcpyDeviceToHost, cx->stream);
  SLRA_CUDA(cudaStreamSynchronize(cx->stream));
  if (st != SLRA_OK) return st;
  if (h_resid_sq) *h_resid_sq = hs[0];
  if (h_norm_sq) *h_norm_sq = hs[1];
  return SLRA_OK;
}

// range_finder: MH (sketch plan) -> Q R (thin QR / TSQR) -> SVD(R) -> rank
// check -> U, V -> residual. Workspace is allocated once per shape.
int slra_range_finder(slra_ctx ctx, const double* M, int64_t ldm, int64_t m, int64_t n, const int64_t* src,
                      const double* coef, const int32_t* q, int64_t width, int tree, int64_t l, int64_t r,
                      int variant, double* U, int64_t ldu, double* V, int64_t ldv, double* d_out,
                      double* d_sigma) {
  if (!ctx || ldm < m || l < 1 || r < 1 || r > l || l > m || l > 64) return SLRA_ERR_INVALID_ARGUMENT;
  Context* cx = C(ctx);
  const int64_t ucols = variant == 1 ? r : l;
  if (ldu < m || ldv < ucols) return SLRA_ERR_INVALID_ARGUMENT;
  const size_t need = 2 * (size_t)m * l + 3 * (size_t)l * l + 2 * (size_t)l + 64;
  double* buf = static_cast<double*>(arena(cx, 0, sizeof(double) * need));
  if (!buf) return SLRA_ERR_CUDA;
  double* MH = buf;                       // m x l
  double* Qm = MH + (size_t)m * l;        // m x l
  double* Rm = Qm + (size_t)m * l;        // l x l
  double* UR = Rm + (size_t)l * l;        // l x l
  double* VR = UR + (size_t)l * l;        // l x l
  double* sig = VR + (size_t)l * l;       // l
  SLRA_TRY(launch_sketch_cols(cx, M, ldm, m, src, coef, q, width, tree, l, MH, m));
  SLRA_TRY(launch_thin_qr(cx, MH, m, m, (int)l, Qm, m, Rm, l));
  SLRA_TRY(launch_svd_small(cx, Rm, l, (int)l, (int)l, UR, l, sig, VR, l, 1e-10 / sqrt((double)l)));
  if (d_sigma) SLRA_CUDA(cudaMemcpyAsync(d_sigma, sig, 8 * l, cudaMemcpyDeviceToDevice, cx->stream));
  // rank check: numerical_rank(MH, 1e-10, Relative) < r -> RangeFailure
  double* hs = static_cast<double*>(cx->hsmall);
  SLRA_CUDA(cudaMemcpyAsync(hs, sig, 8 * l, cudaMemcpyDeviceToHost, cx->stream));
  SLRA_CUDA(cudaStreamSynchronize(cx->stream));
  int64_t rank = 0;
  for (int64_t i = 0; i < l; ++i) rank += (hs[i] > 1e-10 * hs[0]) ? 1 : 0;
  if (rank < r) return SLRA_ERR_RANGE_FAILURE;
  if (variant == 0) {
    // BasisQr: U = Q (thin_qr sign rule already applied), V = U^T M
    SLRA_CUDA(cudaMemcpy2DAsync(U, 8 * ldu, Qm, 8 * m, 8 * m, l, cudaMemcpyDeviceToDevice, cx->stream));
    SLRA_TRY(launch_gemm_fam(cx, "gemm_v", 1, 0, l, n, m, 1.0, U, ldu, M, ldm, 0.0, V, ldv));
  } else {
    // TruncatedRankR: S = Q U_R with the svd sign rule on S; U = S_r Sigma_r;
    // V = U^+ M = Sigma_r^-1 S_r^T M (U's SVD is S_r, Sigma_r, I).
    double* S = MH;  // reuse: m x l
    SLRA_TRY(launch_gemm(cx, 0, 0, m, l, l, 1.0, Qm, m, UR, l, 0.0, S, m));
    SLRA_TRY(launch_colsign(cx, S, m, m, VR, l, l, l));
    SLRA_TRY(launch_scale_cols(cx, S, m, m, r, sig, 0, U, ldu));    // U = S_r Sigma_r
    SLRA_TRY(launch_scale_cols(cx, S, m, m, r, sig, 1, Qm, m));     // Qm := S_r Sigma_r^-1
    SLRA_TRY(launch_gemm_fam(cx, "gemm_v", 1, 0, r, n, m, 1.0, Qm, m, M, ldm, 0.0, V, ldv));
  }
  if (d_out) SLRA_TRY(launch_lowrank_residual(cx, M, ldm, m, n, U, ldu, V, ldv, ucols, d_out));
  return SLRA_OK;
}

}  // extern "C"
