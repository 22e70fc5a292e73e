// K-d: sketched least squares (sketch_solve, lsr.cpp:37-67) and the residual
// pass (residual_norm, lsr.cpp:26-28).
//
// Device formulation: FW = F (A|b) through a compiled left plan (one pass,
// only the k sampled/sketched rows are touched), the Gram matrix
// [FA Fb]^T [FA Fb] on the DMMA GEMM (split-K, deterministic), a blocked
// Cholesky of FA^T FA in one CTA (left-looking, 32-column panels), two
// triangular solves, one step of iterative refinement, and the sketched
// residual ||FA x - Fb|| by a direct pass (never from the Gram identity).
// Rank test: a Cholesky pivot that is non-positive or below
// (1e-10 * max_i ||FA(:,i)||)^2 reports SketchRankFailure — the analogue of
// ColPivHouseholderQR's rank() < d with threshold 1e-10 (lsr.cpp:52-55).
#include "common.cuh"

namespace slra_dev {

int launch_sketch_rows(Context* c, const double* Wm, int64_t ldw, int64_t ncols, const int64_t* src,
                       const double* coef, const int32_t* q, int64_t width, int tree, int64_t k, double* out,
                       int64_t ldo);
int launch_gemm(Context* c, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
                int64_t lda, const double* B, int64_t ldb, double beta, double* Cm, int64_t ldc);

constexpr int kLT = 512;
constexpr int kPW = 32;  // Cholesky panel width

// In-place lower Cholesky of G (d x d, ld d, global/L2), one CTA.
// status[0] = 0 ok, 1 rank failure.
__global__ void __launch_bounds__(kLT) cholesky_kernel(double* __restrict__ G, int d, double tol2,
                                                       int32_t* __restrict__ status) {
  extern __shared__ __align__(16) double P[];  // d x kPW panel (ld d)
  __shared__ int fail;
  const int tid = threadIdx.x;
  if (tid == 0) fail = 0;
  for (int p0 = 0; p0 < d; p0 += kPW) {
    const int pw = (d - p0) < kPW ? (d - p0) : kPW;
    const int rows = d - p0;
    // load panel G[p0:d, p0:p0+pw] and subtract L[p0:d, 0:p0] L[p0:p0+pw, 0:p0]^T
    for (int e = tid; e < rows * pw; e += kLT) {
      const int i = e % rows, c = e / rows;
      if (i < c) {
        P[i + c * d] = 0.0;
        continue;
      }
      const double* Li = G + (p0 + i);
      const double* Lc = G + (p0 + c);
      double acc = G[(p0 + i) + (int64_t)(p0 + c) * d];
      for (int t = 0; t < p0; ++t) acc -= Li[(int64_t)t * d] * Lc[(int64_t)t * d];
      P[i + c * d] = acc;
    }
    __syncthreads();
    // unblocked factorisation of the panel
    for (int j = 0; j < pw; ++j) {
      const double piv = P[j + j * d];
      if (!(piv > tol2)) {
        if (tid == 0) fail = 1;
        __syncthreads();
        break;
      }
      const double ljj = sqrt(piv);
      __syncthreads();
      for (int i = j + tid; i < rows; i += kLT) P[i + j * d] = (i == j) ? ljj : P[i + j * d] / ljj;
      __syncthreads();
      for (int e = tid; e < rows * (pw - j - 1); e += kLT) {
        const int i = e % rows, c = j + 1 + e / rows;
        if (i >= c) P[i + c * d] -= P[i + j * d] * P[c + j * d];
      }
      __syncthreads();
    }
    if (fail) break;
    for (int e = tid; e < rows * pw; e += kLT) {
      const int i = e % rows, c = e / rows;
      G[(p0 + i) + (int64_t)(p0 + c) * d] = P[i + c * d];
    }
    __syncthreads();
  }
  if (tid == 0) *status = fail;
}

// x = (L L^T)^{-1} rhs (lower L in G, ld d), one warp; rhs/x may alias.
__device__ void warp_chol_solve(const double* G, int d, const double* rhs, double* x, double* y) {
  const int lane = threadIdx.x & 31;
  for (int i = 0; i < d; ++i) {  // L y = rhs
    double s = 0.0;
    for (int j = lane; j < i; j += 32) s += G[i + (int64_t)j * d] * y[j];
    s = warp_sum(s);
    if (lane == 0) y[i] = (rhs[i] - s) / G[i + (int64_t)i * d];
    __syncwarp();
  }
  for (int i = d - 1; i >= 0; --i) {  // L^T x = y
    double s = 0.0;
    for (int j = i + 1 + lane; j < d; j += 32) s += G[j + (int64_t)i * d] * x[j];
    s = warp_sum(s);
    if (lane == 0) x[i] = (y[i] - s) / G[i + (int64_t)i * d];
    __syncwarp();
  }
}

__global__ void chol_solve_kernel(const double* __restrict__ L, int d, const double* __restrict__ rhs,
                                  double* __restrict__ x, double* __restrict__ y, const int32_t* __restrict__ status,
                                  int accumulate) {
  if (*status) return;
  if (threadIdx.x >= 32) return;
  // solve into y2 = scratch at y + d, then x (+)= solution
  double* sol = y + d;
  warp_chol_solve(L, d, rhs, sol, y);
  for (int i = threadIdx.x; i < d; i += 32) x[i] = accumulate ? x[i] + sol[i] : sol[i];
}

// r = Fb - FA x (k rows); also writes the squared norm partials.
__global__ void lsq_residual_kernel(const double* __restrict__ FW, int64_t k, int d, const double* __restrict__ x,
                                    double* __restrict__ r, double* __restrict__ part) {
  __shared__ double red[40];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < d; ++j) acc += FW[i + j * k] * x[j];
    const double e = FW[i + (int64_t)d * k] - acc;
    r[i] = e;
    s += e * e;
  }
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void sum_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double red[40];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) out[0] = s;
}

// ||A x - b||^2 over a tall column-major A (m x d): each thread owns rows,
// walks the d columns (coalesced across the warp), deterministic partials.
__global__ void __launch_bounds__(256) lsr_residual_kernel(const double* __restrict__ A, int64_t lda, int64_t m,
                                                           int d, const double* __restrict__ b,
                                                           const double* __restrict__ x, double* __restrict__ part) {
  extern __shared__ double xs[];
  __shared__ double red[40];
  for (int j = threadIdx.x; j < d; j += blockDim.x) xs[j] = x[j];
  __syncthreads();
  double s = 0.0;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x * 2; i0 < m; i0 += (int64_t)gridDim.x * blockDim.x * 2) {
    const int64_t i = i0 + 2 * threadIdx.x;
    if (i + 1 < m && (lda % 2 == 0) && (((uintptr_t)A) % 16 == 0)) {
      double a0 = 0.0, a1 = 0.0;
      const double2* col = reinterpret_cast<const double2*>(A + i);
#pragma unroll 8
      for (int j = 0; j < d; ++j) {
        const double2 v = __ldg(col + (int64_t)j * (lda / 2));
        a0 += v.x * xs[j];
        a1 += v.y * xs[j];
      }
      const double e0 = a0 - b[i], e1 = a1 - b[i + 1];
      s += e0 * e0 + e1 * e1;
    } else {
      for (int64_t ii = i; ii < i + 2 && ii < m; ++ii) {
        double a0 = 0.0;
        for (int j = 0; j < d; ++j) a0 += A[ii + (int64_t)j * lda] * xs[j];
        const double e0 = a0 - b[ii];
        s += e0 * e0;
      }
    }
  }
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

int launch_lsr_residual(Context* c, const double* A, int64_t lda, int64_t m, int64_t d, const double* b,
                        const double* x, double* d_out) {
  int grid = c->num_sms * 4;
  const int64_t need = (m + 511) / 512;
  if (need < grid) grid = (int)(need > 0 ? need : 1);
  double* part = partials(c, grid);
  if (!part) return SLRA_ERR_CUDA;
  SLRA_TIMED(c, "lsr_residual", lsr_residual_kernel<<<grid, 256, sizeof(double) * d, c->stream>>>(A, lda, m, (int)d, b, x, part);)
  SLRA_CHECK_LAUNCH(c);
  SLRA_TIMED(c, "reduce", sum_kernel<<<1, 256, 0, c->stream>>>(part, grid, d_out);)
  SLRA_CHECK_LAUNCH(c);
  return SLRA_OK;
}

}  // namespace slra_dev

using namespace slra_dev;

extern "C" {

int slra_lsr_residual(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t d, const double* b,
                      const double* x, double* d_out) {
  if (!ctx || lda < m || d < 1 || d > 4096) return SLRA_ERR_INVALID_ARGUMENT;
  return launch_lsr_residual(C(ctx), A, lda, m, d, b, x, d_out);
}

int slra_sketch_solve(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t d, const double* b,
                      const int64_t* src, const double* coef, const int32_t* q, int64_t width, int tree, int64_t k,
                      double* x_hat, double* h_sketched_residual) {
  if (!ctx || lda < m || m <= d || d < 1 || k <= d) return SLRA_ERR_INVALID_ARGUMENT;
  if (d > 768) return SLRA_ERR_UNSUPPORTED;
  Context* cx = C(ctx);
  const int64_t dc = d + 1;
  int rgrid = cx->num_sms * 2;
  if ((k + 255) / 256 < rgrid) rgrid = (int)((k + 255) / 256);
  // arena 2: FW (k x dc) | Gw (dc x dc) | G (d x d) | g (d) | r (k) | c (d) | y (2d) | part | out
  const size_t need = (size_t)k * dc + (size_t)dc * dc + (size_t)d * d + 4 * (size_t)d + (size_t)k + rgrid + 16;
  double* ws = static_cast<double*>(arena(cx, 2, sizeof(double) * need));
  if (!ws) return SLRA_ERR_CUDA;
  double* FW = ws;
  double* Gw = FW + (size_t)k * dc;
  double* G = Gw + (size_t)dc * dc;
  double* g = G + (size_t)d * d;
  double* cvec = g + d;
  double* y = cvec + d;
  double* r = y + 2 * d;
  double* part = r + k;
  double* out = part + rgrid;
  int32_t* d_status = static_cast<int32_t*>(cx->dsmall);
  cudaStream_t st = cx->stream;
  // FW = F (A | b): one pass over the k sketched rows
  SLRA_TRY(launch_sketch_rows(cx, A, lda, d, src, coef, q, width, tree, k, FW, k));
  SLRA_TRY(launch_sketch_rows(cx, b, m, 1, src, coef, q, width, tree, k, FW + (size_t)k * d, k));
  // Gram [FA Fb]^T [FA Fb] (dc x dc); G = leading d x d block, g = FA^T Fb
  SLRA_TRY(launch_gemm(cx, 1, 0, dc, dc, k, 1.0, FW, k, FW, k, 0.0, Gw, dc));
  SLRA_CUDA(cudaMemcpy2DAsync(G, 8 * d, Gw, 8 * dc, 8 * d, d, cudaMemcpyDeviceToDevice, st));
  SLRA_CUDA(cudaMemcpyAsync(g, Gw + (size_t)d * dc, 8 * d, cudaMemcpyDeviceToDevice, st));
  // rank tolerance from the largest column norm of FA
  double* hs = static_cast<double*>(cx->hsmall);
  SLRA_CUDA(cudaMemcpy2DAsync(hs, 8, Gw, 8 * (dc + 1), 8, (d < 500 ? d : 500), cudaMemcpyDeviceToHost, st));
  SLRA_CUDA(cudaStreamSynchronize(st));
  double dmax = 0.0;
  for (int64_t i = 0; i < (d < 500 ? d : 500); ++i) dmax = hs[i] > dmax ? hs[i] : dmax;
  const double tol2 = 1e-20 * dmax;
  const size_t smem = sizeof(double) * (size_t)d * kPW;
  SLRA_CUDA(cudaFuncSetAttribute(cholesky_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SLRA_TIMED(cx, "lsr_solve", cholesky_kernel<<<1, kLT, smem, st>>>(G, (int)d, tol2, d_status);)
  SLRA_CHECK_LAUNCH(cx);
  // x = G^{-1} g, then one refinement step x += G^{-1} FA^T (Fb - FA x)
  SLRA_TIMED(cx, "lsr_solve", chol_solve_kernel<<<1, 32, 0, st>>>(G, (int)d, g, x_hat, y, d_status, 0);)
  SLRA_CHECK_LAUNCH(cx);
  SLRA_TIMED(cx, "lsr_solve", lsq_residual_kernel<<<rgrid, 256, 0, st>>>(FW, k, (int)d, x_hat, r, part);)
  SLRA_CHECK_LAUNCH(cx);
  SLRA_TRY(launch_gemm(cx, 1, 0, d, 1, k, 1.0, FW, k, r, k, 0.0, cvec, d));
  SLRA_TIMED(cx, "lsr_solve", chol_solve_kernel<<<1, 32, 0, st>>>(G, (int)d, cvec, x_hat, y, d_status, 1);)
  SLRA_CHECK_LAUNCH(cx);
  // sketched residual ||FA x - Fb|| by a direct pass
  SLRA_TIMED(cx, "lsr_solve", lsq_residual_kernel<<<rgrid, 256, 0, st>>>(FW, k, (int)d, x_hat, r, part);)
  SLRA_CHECK_LAUNCH(cx);
  SLRA_TIMED(cx, "reduce", sum_kernel<<<1, 256, 0, st>>>(part, rgrid, out);)
  SLRA_CHECK_LAUNCH(cx);
  SLRA_CUDA(cudaMemcpyAsync(hs, out, 8, cudaMemcpyDeviceToHost, st));
  SLRA_CUDA(cudaMemcpyAsync(hs + 1, d_status, 4, cudaMemcpyDeviceToHost, st));
  SLRA_CUDA(cudaStreamSynchronize(st));
  if (*reinterpret_cast<int32_t*>(hs + 1)) return SLRA_ERR_SKETCH_RANK_FAILURE;
  if (h_sketched_residual) *h_sketched_residual = sqrt(hs[0]);
  return SLRA_OK;
}

}  // extern "C"
