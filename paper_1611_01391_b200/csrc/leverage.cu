// Elementwise helpers of the leverage-score CUR path (leverage.cpp:12-149):
// row squared norms (the scores p_i = ||t_i||^2 / r), diagonal rescaling
// diag(dr) A diag(dc) in Eigen's evaluation order, and an out-of-place
// transpose. All bandwidth-bound single passes.
#include "common.cuh"

namespace slra_dev {

int launch_transpose(Context* cx, const double* A, int64_t lda, int64_t m, int64_t n, double* B, int64_t ldb);

namespace {

// out[i] = (sum_j A(i, j)^2) / divisor, j ascending (one thread per row:
// consecutive threads read consecutive rows of each column -> coalesced).
__global__ void row_sqnorms_kernel(const double* __restrict__ A, int64_t lda, int64_t m, int64_t n, double divisor,
                                   double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      const double x = A[i + j * lda];
      s = fma(x, x, s);
    }
    out[i] = s / divisor;
  }
}

// B(i, j) = (dr[i] * A(i, j)) * dc[j]; a null scale vector is the identity.
__global__ void scale_rows_cols_kernel(const double* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                                       const double* __restrict__ dr, const double* __restrict__ dc,
                                       double* __restrict__ B, int64_t ldb) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    double v = A[i + j * lda];
    if (dr) v = dr[i] * v;
    if (dc) v = v * dc[j];
    B[i + j * ldb] = v;
  }
}

}  // namespace
}  // namespace slra_dev

using namespace slra_dev;

extern "C" {

int slra_row_sqnorms(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t n, double divisor, double* out) {
  if (!ctx || m < 0 || n < 0 || lda < m || !(divisor > 0.0)) return SLRA_ERR_INVALID_ARGUMENT;
  if (m == 0) return SLRA_OK;
  Context* cx = C(ctx);
  int64_t g = ceil_div(m, 256);
  if (g > cx->num_sms * 8) g = cx->num_sms * 8;
  SLRA_TIMED(cx, "leverage", row_sqnorms_kernel<<<(unsigned)g, 256, 0, cx->stream>>>(A, lda, m, n, divisor, out);)
  SLRA_CHECK_LAUNCH(cx);
  return SLRA_OK;
}

int slra_scale_rows_cols(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t n, const double* dr,
                         const double* dc, double* B, int64_t ldb) {
  if (!ctx || m < 0 || n < 0 || lda < m || ldb < m) return SLRA_ERR_INVALID_ARGUMENT;
  if (m == 0 || n == 0) return SLRA_OK;
  Context* cx = C(ctx);
  int64_t g = ceil_div(m * n, 256);
  if (g > cx->num_sms * 8) g = cx->num_sms * 8;
  SLRA_TIMED(cx, "leverage", scale_rows_cols_kernel<<<(unsigned)g, 256, 0, cx->stream>>>(A, lda, m, n, dr, dc, B,
                                                                                          ldb);)
  SLRA_CHECK_LAUNCH(cx);
  return SLRA_OK;
}

int slra_transpose(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t n, double* B, int64_t ldb) {
  if (!ctx || m < 0 || n < 0 || lda < m || ldb < n) return SLRA_ERR_INVALID_ARGUMENT;
  if (m == 0 || n == 0) return SLRA_OK;
  return launch_transpose(C(ctx), A, lda, m, n, B, ldb);
}

}  // extern "C"
