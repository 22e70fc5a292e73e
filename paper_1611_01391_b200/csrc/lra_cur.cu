// Orchestration of the multi-kernel entry points: cur_evaluate(Frobenius)
// (cur.cpp:76-82) and range_finder (lra.cpp:14-39), the latter batched over
// several sketches of the same matrix so their latency-bound factorisations
// overlap (one kernel launch covers all sketches, one CTA per sketch).
// Everything stays on the device; only rank/status decisions are read back.
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
size_t tsqr_workspace_doubles(int64_t m, int c);
size_t cholqr3_workspace_doubles(int64_t m, int n);
int launch_cholqr3_batched(Context* cx, const double* Y, int64_t ldy, int64_t sY, int64_t m, int n, double* Q,
                           int64_t ldq, int64_t sQ, double* R, int64_t ldr, int64_t sR, int nb, double* ws,
                           int32_t* status);
int launch_thin_qr_batched(Context* cx, const double* A, int64_t lda, int64_t sA, int64_t m, int c, double* Q,
                           int64_t ldq, int64_t sQ, double* R, int64_t ldr, int64_t sR, int nb, double* ws);
int launch_svd_small_batched(Context* cx, const double* A, int64_t lda, int64_t sA, int m, int n, double* S,
                             int64_t lds, int64_t sS, double* sigma, int64_t sSig, double* T, int64_t ldt, int64_t sT,
                             int nb, double deflate);
int launch_colsign_batched(Context* cx, double* S, int64_t lds, int64_t sS, int64_t m, double* T, int64_t ldt,
                           int64_t sT, int64_t n, int64_t cols, int nb);

// Y_b(:, j) = X_b(:, j) * s_b[j] (or / s_b[j] when inv), batched over problems.
__global__ void scale_cols_kernel(const double* __restrict__ X, int64_t ldx, int64_t sX, int64_t m, int64_t cols,
                                  const double* __restrict__ s, int64_t sS, int inv, double* const* __restrict__ Yp,
                                  int64_t ldy) {
  const int64_t total = m * cols;
  const int pb = blockIdx.y;
  X += pb * sX;
  s += pb * sS;
  double* Y = Yp[pb];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    const double f = inv ? 1.0 / s[j] : s[j];
    Y[i + j * ldy] = X[i + j * ldx] * f;
  }
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
  SLRA_TRY(launch_gather_cols(cx, A, lda, m, J, l, Cm, m));
  SLRA_TRY(launch_gather_rows(cx, A, lda, n, I, k, Rm, k));
  // (C U) R, Eigen's left-to-right evaluation (cur.cpp:76-78)
  SLRA_TRY(launch_gemm(cx, 0, 0, m, k, l, 1.0, Cm, m, U, ldu, 0.0, CU, m));
  SLRA_TRY(launch_lowrank_residual(cx, A, lda, m, n, CU, m, Rm, k, k, out));
  double* hs = static_cast<double*>(cx->hsmall);
  SLRA_CUDA(cudaMemcpyAsync(hs, out, 16, cudaMemcpyDeviceToHost, cx->stream));
  SLRA_CUDA(cudaStreamSynchronize(cx->stream));
  if (h_resid_sq) *h_resid_sq = hs[0];
  if (h_norm_sq) *h_norm_sq = hs[1];
  return SLRA_OK;
}

// ||A - C U R||_F with the nucleus in factored form U = Tsig Sr^T (rank r):
// P = C Tsig (m x r), Q = Sr^T R (r x n), one pass over A at inner dimension r.
int slra_cur_residual_factored(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t n, const int64_t* I,
                               int64_t k, const int64_t* J, int64_t l, const double* Tsig, const double* Sr, int64_t r,
                               double* d_out) {
  if (!ctx || lda < m || k < 1 || l < 1 || r < 1 || r > k || r > l) return SLRA_ERR_INVALID_ARGUMENT;
  Context* cx = C(ctx);
  const int64_t ldq = (r + 1) & ~1;  // even ld keeps the streaming kernel's 16-byte staging
  const size_t need = (size_t)m * l + (size_t)k * n + (size_t)m * r + (size_t)ldq * n + 16;
  double* ws = static_cast<double*>(arena(cx, 5, sizeof(double) * need));
  if (!ws) return SLRA_ERR_CUDA;
  double* Cm = ws;
  double* Rm = Cm + (size_t)m * l;
  double* P = Rm + (size_t)k * n;
  double* Q = P + (size_t)m * r;
  SLRA_TRY(launch_gather_cols(cx, A, lda, m, J, l, Cm, m));
  SLRA_TRY(launch_gather_rows(cx, A, lda, n, I, k, Rm, k));
  SLRA_TRY(launch_gemm(cx, 0, 0, m, r, l, 1.0, Cm, m, Tsig, l, 0.0, P, m));
  SLRA_TRY(launch_gemm(cx, 1, 0, r, n, k, 1.0, Sr, k, Rm, k, 0.0, Q, ldq));
  return launch_lowrank_residual(cx, A, lda, m, n, P, m, Q, ldq, r, d_out);
}

// range_finder over nsk sketches H_s of one M: MH_s (plans) -> Q_s R_s (batched
// thin QR / TSQR) -> SVD(R_s) (batched, one CTA each) -> one rank check for
// all -> U_s, V_s -> residuals. Host-array arguments (h_*) hold per-sketch
// device pointers / sizes.
}  // extern "C"

namespace slra_dev {
// want_v = false: the basis only (range_basis, lra.cpp:14-28) for lra_premult.
int range_finder_core(Context* cx, const double* M, int64_t ldm, int64_t m, int64_t n, int nsk,
                      const int64_t* const* h_src, const double* const* h_coef, const int32_t* const* h_q,
                      const int64_t* h_width, const int* h_tree, int64_t l, int64_t r, int variant,
                      double* const* h_U, int64_t ldu, double* const* h_V, int64_t ldv, double* d_out,
                      double* d_sigma, int32_t* h_status, bool want_v) {
  if (ldm < m || l < 1 || r < 1 || r > l || l > m || l > 64 || nsk < 1 || nsk > 64)
    return SLRA_ERR_INVALID_ARGUMENT;
  const int64_t ucols = variant == 1 ? r : l;
  if (ldu < m || ldv < ucols) return SLRA_ERR_INVALID_ARGUMENT;
  const size_t tw = tsqr_workspace_doubles(m, (int)l);
  const size_t cw = cholqr3_workspace_doubles(m, (int)l);
  const size_t per = 2 * (size_t)m * l + 3 * (size_t)l * l + (size_t)l + tw + cw;
  double* buf = static_cast<double*>(arena(cx, 0, sizeof(double) * (per * nsk + 64)));
  if (!buf) return SLRA_ERR_CUDA;
  const int64_t sMH = m * l, sLL = l * l;
  double* MH = buf;                     // nsk x (m x l)
  double* Qm = MH + (size_t)nsk * sMH;  // nsk x (m x l)
  double* Rm = Qm + (size_t)nsk * sMH;  // nsk x (l x l)
  double* UR = Rm + (size_t)nsk * sLL;
  double* VR = UR + (size_t)nsk * sLL;
  double* sig = VR + (size_t)nsk * sLL;  // nsk x l
  double* tws = sig + (size_t)nsk * l;   // TSQR workspace (nsk problems)
  double* cws = tws + (size_t)nsk * tw;  // CholeskyQR3 workspace (nsk problems)
  double** dptr = reinterpret_cast<double**>(static_cast<char*>(cx->dsmall) + 2048);  // 2*nsk pointers
  int32_t* cq_status = reinterpret_cast<int32_t*>(static_cast<char*>(cx->dsmall) + 3584);  // nsk flags
  for (int s = 0; s < nsk; ++s)
    SLRA_TRY(launch_sketch_cols(cx, M, ldm, m, h_src[s], h_coef[s], h_q[s], h_width[s], h_tree[s], l,
                                MH + s * sMH, m));
  // Q R of the sketch: shifted CholeskyQR3 (cholqr.cu); a breakdown falls
  // back to the Householder TSQR below, after the one host sync
  SLRA_TRY(launch_cholqr3_batched(cx, MH, m, sMH, m, (int)l, Qm, m, sMH, Rm, l, sLL, nsk, cws, cq_status));
  // TruncatedRankR only needs the top r triplets and the count of sigma above
  // the cut: Jacobi skips pairs of columns below cut / sqrt(l) (dense_cta.cuh)
  const double deflate = variant == 1 ? 1e-10 / sqrt((double)l) : 0.0;
  SLRA_TRY(launch_svd_small_batched(cx, Rm, l, sLL, (int)l, (int)l, UR, l, sLL, sig, l, VR, l, sLL, nsk, deflate));
  // rank check: numerical_rank(MH, 1e-10, Relative) < r -> RangeFailure
  std::vector<double> hsv((size_t)nsk * l);
  std::vector<int32_t> hq((size_t)nsk);
  double* hs = hsv.data();
  SLRA_CUDA(cudaMemcpyAsync(hq.data(), cq_status, 4 * nsk, cudaMemcpyDeviceToHost, cx->stream));
  SLRA_CUDA(cudaMemcpyAsync(hs, sig, 8 * l * nsk, cudaMemcpyDeviceToHost, cx->stream));
  SLRA_CUDA(cudaStreamSynchronize(cx->stream));
  bool redo = false;
  for (int s = 0; s < nsk; ++s)
    if (hq[s]) {
      redo = true;
      SLRA_TRY(launch_thin_qr_batched(cx, MH + s * sMH, m, sMH, m, (int)l, Qm + s * sMH, m, sMH, Rm + s * sLL, l, sLL,
                                      1, tw ? tws : nullptr));
      SLRA_TRY(launch_svd_small_batched(cx, Rm + s * sLL, l, sLL, (int)l, (int)l, UR + s * sLL, l, sLL, sig + s * l,
                                        l, VR + s * sLL, l, sLL, 1, deflate));
    }
  if (redo) {
    SLRA_CUDA(cudaMemcpyAsync(hs, sig, 8 * l * nsk, cudaMemcpyDeviceToHost, cx->stream));
    SLRA_CUDA(cudaStreamSynchronize(cx->stream));
  }
  if (d_sigma) SLRA_CUDA(cudaMemcpyAsync(d_sigma, sig, 8 * l * nsk, cudaMemcpyDeviceToDevice, cx->stream));
  int first_fail = -1;
  std::vector<int> ok(nsk, 1);
  for (int s = 0; s < nsk; ++s) {
    int64_t rank = 0;
    for (int64_t i = 0; i < l; ++i) rank += (hs[s * l + i] > 1e-10 * hs[s * l]) ? 1 : 0;
    const int st = rank < r ? SLRA_ERR_RANGE_FAILURE : SLRA_OK;
    ok[s] = st == SLRA_OK;
    if (h_status) h_status[s] = st;
    if (st != SLRA_OK && first_fail < 0) first_fail = s;
  }
  if (first_fail >= 0 && !h_status) return SLRA_ERR_RANGE_FAILURE;
  if (variant == 1) {
    // TruncatedRankR: S = Q U_R with the svd sign rule on S; U = S_r Sigma_r;
    // V = U^+ M = Sigma_r^-1 S_r^T M (U's SVD is S_r, Sigma_r, I).
    double* S = MH;  // reuse: nsk x (m x l)
    for (int s = 0; s < nsk; ++s)
      SLRA_TRY(launch_gemm(cx, 0, 0, m, l, l, 1.0, Qm + s * sMH, m, UR + s * sLL, l, 0.0, S + s * sMH, m));
    SLRA_TRY(launch_colsign_batched(cx, S, m, sMH, m, VR, l, sLL, l, l, nsk));
    std::vector<double*> hp(2 * nsk);
    for (int s = 0; s < nsk; ++s) {
      hp[s] = h_U[s];
      hp[nsk + s] = Qm + s * sMH;
    }
    SLRA_CUDA(cudaMemcpyAsync(dptr, hp.data(), sizeof(double*) * 2 * nsk, cudaMemcpyHostToDevice, cx->stream));
    int g = ceil_div(m * r, 256);
    if (g > cx->num_sms * 4) g = cx->num_sms * 4;
    // U = S_r Sigma_r ; Qm := S_r Sigma_r^-1
    SLRA_TIMED(cx, "scale", scale_cols_kernel<<<dim3(g, nsk), 256, 0, cx->stream>>>(S, m, sMH, m, r, sig, l, 0, dptr,
                                                                                    ldu);)
    SLRA_CHECK_LAUNCH(cx);
    SLRA_TIMED(cx, "scale", scale_cols_kernel<<<dim3(g, nsk), 256, 0, cx->stream>>>(S, m, sMH, m, r, sig, l, 1,
                                                                                    dptr + nsk, m);)
    SLRA_CHECK_LAUNCH(cx);
    for (int s = 0; s < nsk; ++s)
      if (ok[s] && want_v)
        SLRA_TRY(launch_gemm_fam(cx, "gemm_v", 1, 0, r, n, m, 1.0, Qm + s * sMH, m, M, ldm, 0.0, h_V[s], ldv));
  } else {
    // BasisQr: U = Q (thin_qr sign rule already applied), V = U^T M
    for (int s = 0; s < nsk; ++s) {
      SLRA_CUDA(cudaMemcpy2DAsync(h_U[s], 8 * ldu, Qm + s * sMH, 8 * m, 8 * m, l, cudaMemcpyDeviceToDevice,
                                  cx->stream));
      if (ok[s] && want_v)
        SLRA_TRY(launch_gemm_fam(cx, "gemm_v", 1, 0, l, n, m, 1.0, h_U[s], ldu, M, ldm, 0.0, h_V[s], ldv));
    }
  }
  if (d_out && want_v)
    for (int s = 0; s < nsk; ++s)
      if (ok[s]) SLRA_TRY(launch_lowrank_residual(cx, M, ldm, m, n, h_U[s], ldu, h_V[s], ldv, ucols, d_out + 2 * s));
  return SLRA_OK;
}
}  // namespace slra_dev

extern "C" {

int slra_range_finder_batched(slra_ctx ctx, const double* M, int64_t ldm, int64_t m, int64_t n, int nsk,
                              const int64_t* const* h_src, const double* const* h_coef, const int32_t* const* h_q,
                              const int64_t* h_width, const int* h_tree, int64_t l, int64_t r, int variant,
                              double* const* h_U, int64_t ldu, double* const* h_V, int64_t ldv, double* d_out,
                              double* d_sigma, int32_t* h_status) {
  if (!ctx) return SLRA_ERR_INVALID_ARGUMENT;
  return range_finder_core(C(ctx), M, ldm, m, n, nsk, h_src, h_coef, h_q, h_width, h_tree, l, r, variant, h_U, ldu,
                           h_V, ldv, d_out, d_sigma, h_status, true);
}

int slra_range_finder(slra_ctx ctx, const double* M, int64_t ldm, int64_t m, int64_t n, const int64_t* src,
                      const double* coef, const int32_t* q, int64_t width, int tree, int64_t l, int64_t r,
                      int variant, double* U, int64_t ldu, double* V, int64_t ldv, double* d_out,
                      double* d_sigma) {
  return slra_range_finder_batched(ctx, M, ldm, m, n, 1, &src, &coef, &q, &width, &tree, l, r, variant, &U, ldu, &V,
                                   ldv, d_out, d_sigma, nullptr);
}

}  // extern "C"
