// Abridged Fourier operator (sketch.cpp:137-211) on the device: d radix-2
// decimation-in-frequency butterfly levels over the rows of a complex n x c
// operand held as real / imaginary planes, then the reference's per-level
// interleave as ONE gather (output row j 2^d + rev_d(q) <- leaf q, offset j).
// Twiddles are the reference's exp(i theta k) values computed on the host
// (glibc, as the reference computes them) and uploaded; complex products are
// evaluated as (ac - bd, ad + bc) with separately rounded products, as
// std::complex / Eigen do, so the device matches the reference's arithmetic.
#include <vector>

#include "common.cuh"

namespace slra_dev {
namespace {

__device__ __forceinline__ void cmul(double a, double b, double c, double d, double& re, double& im) {
  re = __dsub_rn(__dmul_rn(a, c), __dmul_rn(b, d));
  im = __dadd_rn(__dmul_rn(a, d), __dmul_rn(b, c));
}

// one level on segments of length L (half = L / 2), in place; thread per
// (pair, column). forward: u = x0 + x1, w = (x0 - x1) t; transpose:
// w = x1 t, x0' = x0 + w, x1' = x0 - w.
__global__ void af_level_kernel(double* __restrict__ re, double* __restrict__ im, int64_t ld, int64_t n, int64_t c,
                                int64_t L, const double* __restrict__ twr, const double* __restrict__ twi,
                                int transpose) {
  const int64_t half = L / 2, pairs = n / 2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < pairs * c; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e % pairs, j = e / pairs;
    const int64_t g = p / half, o = p % half;
    const int64_t r0 = g * L + o + j * ld, r1 = r0 + half;
    const double ar = re[r0], ai = im[r0], br = re[r1], bi = im[r1];
    const double tr = twr[o], ti = twi[o];
    if (!transpose) {
      double wr, wi;
      cmul(__dsub_rn(ar, br), __dsub_rn(ai, bi), tr, ti, wr, wi);
      re[r0] = __dadd_rn(ar, br);
      im[r0] = __dadd_rn(ai, bi);
      re[r1] = wr;
      im[r1] = wi;
    } else {
      double wr, wi;
      cmul(br, bi, tr, ti, wr, wi);
      re[r0] = __dadd_rn(ar, wr);
      im[r0] = __dadd_rn(ai, wi);
      re[r1] = __dsub_rn(ar, wr);
      im[r1] = __dsub_rn(ai, wi);
    }
  }
}

__device__ __forceinline__ int64_t rev_bits(int64_t q, int d) {
  int64_t r = 0;
  for (int k = 0; k < d; ++k) r |= ((q >> k) & 1) << (d - 1 - k);
  return r;
}

// gather between the level-major layout (row q B + j) and the reference's
// interleaved output (row j 2^d + rev_d(q)); to_output selects the direction
__global__ void af_permute_kernel(const double* __restrict__ sr, const double* __restrict__ si, int64_t lds,
                                  double* __restrict__ dr, double* __restrict__ di, int64_t ldd, int64_t n, int64_t c,
                                  int d, int to_output) {
  const int64_t B = n >> d, mask = ((int64_t)1 << d) - 1;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * c; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e % n, col = e / n;
    int64_t from;
    if (to_output) {  // dst row = j 2^d + rev(q)  <-  src row q B + j
      const int64_t q = rev_bits(row & mask, d), j = row >> d;
      from = q * B + j;
    } else {          // dst row = q B + j  <-  src row j 2^d + rev(q)
      const int64_t q = row / B, j = row % B;
      from = (j << d) + rev_bits(q, d);
    }
    dr[row + col * ldd] = sr[from + col * lds];
    di[row + col * ldd] = si[from + col * lds];
  }
}

}  // namespace
}  // namespace slra_dev

using namespace slra_dev;

extern "C" int slra_af_apply(slra_ctx ctx, const double* re, const double* im, int64_t ld, int64_t n, int64_t c,
                             int d, const double* twr, const double* twi, int transpose, double* ore, double* oim,
                             int64_t ldo) {
  if (!ctx || n < 2 || c < 0 || d < 1 || d > 62 || ld < n || ldo < n || (n % ((int64_t)1 << d)) != 0)
    return SLRA_ERR_INVALID_ARGUMENT;
  if (c == 0) return SLRA_OK;
  Context* cx = C(ctx);
  double* ws = static_cast<double*>(workspace(cx, sizeof(double) * 2 * (size_t)n * c));
  if (!ws) return SLRA_ERR_CUDA;
  double* wr = ws;
  double* wi = ws + n * c;
  int64_t g = ceil_div(n * c, 256);
  if (g > cx->num_sms * 8) g = cx->num_sms * 8;
  int64_t gp = ceil_div(n / 2 * c, 256);
  if (gp > cx->num_sms * 8) gp = cx->num_sms * 8;
  if (!transpose) {
    // levels top-down on a copy (unit permutation = copy), then the interleave
    SLRA_CUDA(cudaMemcpy2DAsync(wr, 8 * n, re, 8 * ld, 8 * n, c, cudaMemcpyDeviceToDevice, cx->stream));
    SLRA_CUDA(cudaMemcpy2DAsync(wi, 8 * n, im, 8 * ld, 8 * n, c, cudaMemcpyDeviceToDevice, cx->stream));
    int64_t off = 0;
    for (int s = 0; s < d; ++s) {
      const int64_t L = n >> s;
      SLRA_TIMED(cx, "sketch", af_level_kernel<<<(unsigned)gp, 256, 0, cx->stream>>>(wr, wi, n, n, c, L, twr + off,
                                                                                     twi + off, 0);)
      SLRA_CHECK_LAUNCH(cx);
      off += L / 2;
    }
    SLRA_TIMED(cx, "sketch", af_permute_kernel<<<(unsigned)g, 256, 0, cx->stream>>>(wr, wi, n, ore, oim, ldo, n, c, d,
                                                                                    1);)
    SLRA_CHECK_LAUNCH(cx);
  } else {
    // de-interleave, then the levels bottom-up
    SLRA_TIMED(cx, "sketch", af_permute_kernel<<<(unsigned)g, 256, 0, cx->stream>>>(re, im, ld, wr, wi, n, n, c, d,
                                                                                    0);)
    SLRA_CHECK_LAUNCH(cx);
    std::vector<int64_t> offs(d);
    int64_t off = 0;
    for (int s = 0; s < d; ++s) {
      offs[s] = off;
      off += (n >> s) / 2;
    }
    for (int s = d - 1; s >= 0; --s) {
      const int64_t L = n >> s;
      SLRA_TIMED(cx, "sketch", af_level_kernel<<<(unsigned)gp, 256, 0, cx->stream>>>(wr, wi, n, n, c, L,
                                                                                     twr + offs[s], twi + offs[s], 1);)
      SLRA_CHECK_LAUNCH(cx);
    }
    SLRA_CUDA(cudaMemcpy2DAsync(ore, 8 * ldo, wr, 8 * n, 8 * n, c, cudaMemcpyDeviceToDevice, cx->stream));
    SLRA_CUDA(cudaMemcpy2DAsync(oim, 8 * ldo, wi, 8 * n, 8 * n, c, cudaMemcpyDeviceToDevice, cx->stream));
  }
  return SLRA_OK;
}
