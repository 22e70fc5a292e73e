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

// ---------------------------------------------------------------- inverse bidiagonal
// InverseBidiagonalOp (sketch.cpp:286-331): per column the recurrence
// y_i = x_i + b_{i-1} y_{i-1} (forward) or y_i = x_i + b_i y_{i+1}
// (backward), in the reference's sequential order (bit-exact for b = +-1).
// One warp owns 32 columns: 32 x 32 tiles are staged through shared memory
// so global loads/stores are row-contiguous (coalesced), and each lane then
// walks its column through the tile carrying y across tiles.
namespace slra_dev {
namespace {
__global__ void bidiag_scan_kernel(const double* __restrict__ X, int64_t ldx, int64_t n, int64_t c,
                                   const double* __restrict__ b, int forward, double* __restrict__ Y, int64_t ldy) {
  __shared__ double tile[4][32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c0 = ((int64_t)blockIdx.x * 4 + w) * 32;
  if (c0 >= c) return;
  double (*t)[33] = tile[w];
  const int64_t col = c0 + lane;
  const int ncol = (int)((c - c0) < 32 ? (c - c0) : 32);
  double y = 0.0;
  const int64_t ntiles = (n + 31) / 32;
  for (int64_t tt = 0; tt < ntiles; ++tt) {
    const int64_t tile_idx = forward ? tt : ntiles - 1 - tt;
    const int64_t r0 = tile_idx * 32;
    const int nr = (int)((n - r0) < 32 ? (n - r0) : 32);
    for (int j = 0; j < ncol; ++j)
      if (lane < nr) t[lane][j] = X[r0 + lane + (c0 + j) * ldx];
    __syncwarp();
    if (lane < ncol) {
      if (forward) {
        for (int i = 0; i < nr; ++i) {
          const int64_t gi = r0 + i;
          const double v = t[i][lane];
          y = gi == 0 ? v : v + b[gi - 1] * y;
          t[i][lane] = y;
        }
      } else {
        for (int i = nr - 1; i >= 0; --i) {
          const int64_t gi = r0 + i;
          const double v = t[i][lane];
          y = gi == n - 1 ? v : v + b[gi] * y;
          t[i][lane] = y;
        }
      }
    }
    __syncwarp();
    for (int j = 0; j < ncol; ++j)
      if (lane < nr) Y[r0 + lane + (c0 + j) * ldy] = t[lane][j];
    __syncwarp();
  }
  (void)col;
}
}  // namespace
}  // namespace slra_dev

extern "C" int slra_bidiag_scan(slra_ctx ctx, const double* X, int64_t ldx, int64_t n, int64_t c, const double* b,
                                int forward, double* Y, int64_t ldy) {
  if (!ctx || n < 1 || c < 0 || ldx < n || ldy < n) return SLRA_ERR_INVALID_ARGUMENT;
  if (c == 0) return SLRA_OK;
  slra_dev::Context* cx = slra_dev::C(ctx);
  const unsigned g = (unsigned)slra_dev::ceil_div(c, 128);
  SLRA_TIMED(cx, "sketch", slra_dev::bidiag_scan_kernel<<<g, 128, 0, cx->stream>>>(X, ldx, n, c, b, forward, Y, ldy);)
  SLRA_CHECK_LAUNCH(cx);
  return SLRA_OK;
}

// Y = alpha X + beta Y (one rounding per entry: fma(alpha, x, beta y)); the
// signed accumulation of SumOp (sketch.cpp:469-475) with alpha = +-1, beta = 1.
namespace slra_dev {
namespace {
__global__ void axpby_kernel(double alpha, const double* __restrict__ X, int64_t ldx, double beta,
                             double* __restrict__ Y, int64_t ldy, int64_t m, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    const double y = beta == 0.0 ? 0.0 : beta * Y[i + j * ldy];
    Y[i + j * ldy] = fma(alpha, X[i + j * ldx], y);
  }
}
}  // namespace
}  // namespace slra_dev

extern "C" int slra_axpby(slra_ctx ctx, double alpha, const double* X, int64_t ldx, double beta, double* Y,
                          int64_t ldy, int64_t m, int64_t n) {
  if (!ctx || m < 0 || n < 0 || ldx < m || ldy < m) return SLRA_ERR_INVALID_ARGUMENT;
  if (m == 0 || n == 0) return SLRA_OK;
  slra_dev::Context* cx = slra_dev::C(ctx);
  int64_t g = slra_dev::ceil_div(m * n, 256);
  if (g > cx->num_sms * 8) g = cx->num_sms * 8;
  SLRA_TIMED(cx, "sketch", slra_dev::axpby_kernel<<<(unsigned)g, 256, 0, cx->stream>>>(alpha, X, ldx, beta, Y, ldy, m, n);)
  SLRA_CHECK_LAUNCH(cx);
  return SLRA_OK;
}
