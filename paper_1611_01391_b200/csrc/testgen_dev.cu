// a13 input generator on the device: the config-5 log-kernel blocks
// K_ij = 0.5 log(dx^2 + dy^2) (testgen gen_log_kernel_block; FunctionOracle
// recipe, oracle.hpp:43-54) from per-block points drawn on the host by the
// reference Rng. Setup only (untimed); the products and the sum are rounded
// separately as on the host (no FMA contraction), the log is CUDA's (within
// an ulp of the host's).
#include "common.cuh"

namespace slra_dev {

__global__ void log_kernel_blocks_kernel(const double* __restrict__ px, const double* __restrict__ py,
                                         const double* __restrict__ qx, const double* __restrict__ qy, int64_t nb,
                                         int m, int n, double* __restrict__ A, int64_t lda, int64_t stride) {
  const int64_t b = blockIdx.y;
  const double* pxb = px + b * m;
  const double* pyb = py + b * m;
  double* Ab = A + b * stride;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)m * n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % m), j = (int)(e / m);
    const double dx = __dsub_rn(pxb[i], qx[b * n + j]);
    const double dy = __dsub_rn(pyb[i], qy[b * n + j]);
    Ab[i + j * lda] = 0.5 * log(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
  }
}

}  // namespace slra_dev

using namespace slra_dev;

extern "C" int slra_gen_log_kernel_blocks(slra_ctx ctx, const double* px, const double* py, const double* qx,
                                          const double* qy, int64_t nblocks, int64_t m, int64_t n, double* A,
                                          int64_t lda, int64_t stride) {
  if (!ctx || m < 1 || n < 1 || lda < m || nblocks < 0 || stride < lda * n) return SLRA_ERR_INVALID_ARGUMENT;
  if (nblocks == 0) return SLRA_OK;
  Context* c = C(ctx);
  for (int64_t b0 = 0; b0 < nblocks; b0 += 65535) {  // grid.y limit
    const int64_t nb = nblocks - b0 < 65535 ? nblocks - b0 : 65535;
    const dim3 grid((unsigned)std::min<int64_t>(((int64_t)m * n + 255) / 256, 64), (unsigned)nb);
    log_kernel_blocks_kernel<<<grid, 256, 0, c->stream>>>(px + b0 * m, py + b0 * m, qx + b0 * n, qy + b0 * n, nb,
                                                          (int)m, (int)n, A + b0 * stride, lda, stride);
    SLRA_CHECK_LAUNCH(c);
  }
  return SLRA_OK;
}
