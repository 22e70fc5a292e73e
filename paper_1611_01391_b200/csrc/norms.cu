// matrix_norm (linalg.cpp:134-151) on the device: spectral = sigma_0 of the
// SVD (one-CTA or multi-CTA Jacobi), Frobenius = one streaming pass,
// Chebyshev = max |a_ij| (one pass, per-CTA maxima then one CTA).
#include "common.cuh"

namespace slra_dev {

int launch_svd(Context* cx, const double* A, int64_t lda, int64_t m, int64_t n, double* S, int64_t lds,
               double* sigma, double* T, int64_t ldt);
int launch_lowrank_residual(Context* c, const double* A, int64_t lda, int64_t m, int64_t n, const double* P,
                            int64_t ldp, const double* Q, int64_t ldq, int64_t inner, double* d_out);

namespace {

__global__ void maxabs_kernel(const double* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                              double* __restrict__ part) {
  __shared__ double red[33];
  double mx = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * n; e += (int64_t)gridDim.x * blockDim.x)
    mx = fmax(mx, fabs(A[e % m + (e / m) * lda]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, red[w]);
    part[blockIdx.x] = t;
  }
}

__global__ void max_reduce_kernel(const double* __restrict__ part, int np, double* __restrict__ out) {
  __shared__ double red[33];
  double mx = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) mx = fmax(mx, part[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, red[w]);
    *out = t;
  }
}

}  // namespace
}  // namespace slra_dev

using namespace slra_dev;

extern "C" {

int slra_matrix_norm(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t n, int kind, double* h_out) {
  if (!ctx || !h_out || m < 0 || n < 0 || lda < m || kind < 0 || kind > 2) return SLRA_ERR_INVALID_ARGUMENT;
  Context* cx = C(ctx);
  if (m == 0 || n == 0) {
    *h_out = 0.0;
    return SLRA_OK;
  }
  double* res = static_cast<double*>(cx->dsmall);
  if (kind == 0) {  // spectral_norm (linalg.cpp:134-137): largest singular value
    const int64_t p = m < n ? m : n;
    double* ws = static_cast<double*>(workspace(cx, sizeof(double) * ((size_t)m * p + (size_t)n * p + p)));
    if (!ws) return SLRA_ERR_CUDA;
    SLRA_TRY(launch_svd(cx, A, lda, m, n, ws, m, ws + m * p + n * p, ws + m * p, n));
    SLRA_CUDA(cudaMemcpyAsync(h_out, ws + m * p + n * p, sizeof(double), cudaMemcpyDeviceToHost, cx->stream));
  } else if (kind == 1) {  // frobenius_norm (linalg.cpp:139)
    SLRA_TRY(launch_lowrank_residual(cx, A, lda, m, n, nullptr, 1, nullptr, 1, 0, res));
    double two[2];
    SLRA_CUDA(cudaMemcpyAsync(two, res, sizeof(two), cudaMemcpyDeviceToHost, cx->stream));
    SLRA_CUDA(cudaStreamSynchronize(cx->stream));
    *h_out = sqrt(two[1]);
    return SLRA_OK;
  } else {  // chebyshev_norm (linalg.cpp:141-143)
    int g = (int)ceil_div(m * n, 256);
    if (g > cx->num_sms * 4) g = cx->num_sms * 4;
    double* part = partials(cx, g);
    if (!part) return SLRA_ERR_CUDA;
    SLRA_TIMED(cx, "norm", maxabs_kernel<<<g, 256, 0, cx->stream>>>(A, lda, m, n, part);)
    SLRA_CHECK_LAUNCH(cx);
    SLRA_TIMED(cx, "norm", max_reduce_kernel<<<1, 256, 0, cx->stream>>>(part, g, res);)
    SLRA_CHECK_LAUNCH(cx);
    SLRA_CUDA(cudaMemcpyAsync(h_out, res, sizeof(double), cudaMemcpyDeviceToHost, cx->stream));
  }
  SLRA_CUDA(cudaStreamSynchronize(cx->stream));
  return SLRA_OK;
}

}  // extern "C"
