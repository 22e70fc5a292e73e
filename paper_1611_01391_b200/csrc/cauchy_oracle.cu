// Config 3's matrix as a FunctionOracle (oracle.hpp:43-54): the FMM-style
// off-diagonal kernel block A_ij = 1/(x_i - y_j) given by its points. The
// C-A of cross_approx (cur.cpp:201-255) reads A only through its strips and
// the generator, and cur_evaluate (cur.cpp:76-82) through one full pass:
// here every such read evaluates the entry (one IEEE division, the same value
// the materialised matrix holds) instead of loading it, so the 2 GiB matrix
// never exists and only the 2 x 128 KiB of points cross the host link.
//
//   cauchy_strip_kernel     A(I, :)^T (rows = true) or A(:, J): the strips
//   cauchy_block_kernel     G = A(I, J): the generator
//   (stream_dmma.cu)        cauchy_residual_stream_kernel: ||A - P Q||_F
//
// The selection and nucleus machinery is the dense path's (TSQR, grid-wide
// maxvol, the CTA-resident primitive_cur on the gathered generator), so the
// results are the dense path's bit for bit (tests/test_gpu_parity.py).
#include "common.cuh"

namespace slra_dev {

size_t tsqr_workspace_doubles(int64_t m, int c);
int launch_thin_qr_batched(Context* cx, const double* A, int64_t lda, int64_t sA, int64_t m, int c, double* Q,
                           int64_t ldq, int64_t sQ, double* R, int64_t ldr, int64_t sR, int nb, double* ws);
size_t maxvol_large_scratch_doubles(int num_sms, int64_t m);
int launch_maxvol_large(Context* cx, const double* Q, int64_t ldq, int64_t m, int r, double h, int max_swaps,
                        int64_t* d_idx, double* d_vol, double* scratch);
int launch_gemm(Context* c, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
                int64_t lda, const double* B, int64_t ldb, double beta, double* Cm, int64_t ldc);
int launch_residual_stream_cauchy(Context* c, const double* x, const double* y, int64_t m, int64_t n,
                                  const double* P, int64_t ldp, const double* Q, int64_t ldq, int64_t inner,
                                  double* d_out);

__device__ __forceinline__ double cauchy_entry(double xi, double yj) { return __ddiv_rn(1.0, __dsub_rn(xi, yj)); }

// rows: S(j, t) = A(idx[t], j) (len = n, the transposed row strip);
// else  S(i, t) = A(i, idx[t]) (len = m). A thread per strip row, the
// strip's own coordinate loaded once.
__global__ void __launch_bounds__(256) cauchy_strip_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                                           int64_t len, const int64_t* __restrict__ idx, int64_t c,
                                                           int rows, double* __restrict__ S, int64_t lds) {
  const int64_t i = blockIdx.x * 256LL + threadIdx.x;
  if (i >= len) return;
  const int64_t t0 = blockIdx.y * 8LL;
  const double own = rows ? __ldg(y + i) : __ldg(x + i);
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int64_t t = t0 + u;
    if (t < c) {
      const double o = rows ? __ldg(x + idx[t]) : __ldg(y + idx[t]);
      S[i + t * lds] = rows ? cauchy_entry(o, own) : cauchy_entry(own, o);
    }
  }
}

__global__ void cauchy_block_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                    const int64_t* __restrict__ I, int64_t k, const int64_t* __restrict__ J,
                                    int64_t l, double* __restrict__ G, int64_t ldg) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < k * l; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = e % k, b = e / k;
    G[a + b * ldg] = cauchy_entry(__ldg(x + (I ? I[a] : a)), __ldg(y + (J ? J[b] : b)));
  }
}

__global__ void iota_kernel(int64_t* v, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) v[e] = e;
}

static int launch_cauchy_strip(Context* c, const double* x, const double* y, int64_t len, const int64_t* idx,
                               int64_t cnt, bool rows, double* S, int64_t lds) {
  const dim3 grid((unsigned)((len + 255) / 256), (unsigned)((cnt + 7) / 8));
  SLRA_TIMED(c, "gather", cauchy_strip_kernel<<<grid, 256, 0, c->stream>>>(x, y, len, idx, cnt, rows ? 1 : 0, S, lds);)
  SLRA_CHECK_LAUNCH(c);
  return SLRA_OK;
}

}  // namespace slra_dev

using namespace slra_dev;

extern "C" {

int slra_cross_approx(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t n, int64_t r, int64_t k,
                      int64_t l, const int64_t* init_rows, int loops, double h, int64_t* I_out, int64_t* J_out,
                      double* nucleus, int64_t* trace_rows, int64_t* trace_cols, double* trace_vol,
                      double* Tsig, double* Sr, int64_t* h_r_out);
int slra_primitive_cur(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t n, const int64_t* I, int64_t k,
                       const int64_t* J, int64_t l, int64_t r, double* nucleus, int64_t ldu, double* Tsig,
                       double* Sr, int64_t* h_r_out);

int slra_cross_approx_cauchy(slra_ctx ctx, const double* x, const double* y, int64_t m, int64_t n, int64_t r,
                             int64_t k, int64_t l, const int64_t* init_rows, int loops, double h, int64_t* I_out,
                             int64_t* J_out, double* nucleus, int64_t* trace_rows, int64_t* trace_cols,
                             double* trace_vol, double* Tsig, double* Sr, int64_t* h_r_out) {
  if (!ctx || !x || !y || loops < 1 || k < 1 || l < 1 || (r > 0 && (k < r || l < r)) || k > m || l > n)
    return SLRA_ERR_INVALID_ARGUMENT;
  Context* cx = C(ctx);
  if (m <= 256 && n <= 256) {
    // a block that fits one SM: evaluate it once (<= 512 KiB) and take the
    // CTA-resident kernel
    double* Aw = static_cast<double*>(workspace(cx, sizeof(double) * (size_t)m * n));
    if (!Aw) return SLRA_ERR_CUDA;
    cauchy_block_kernel<<<64, 256, 0, cx->stream>>>(x, y, nullptr, m, nullptr, n, Aw, m);
    SLRA_CHECK_LAUNCH(cx);
    return slra_cross_approx(ctx, Aw, m, m, n, r, k, l, init_rows, loops, h, I_out, J_out, nucleus, trace_rows,
                             trace_cols, trace_vol, Tsig, Sr, h_r_out);
  }
  if (k > 64 || l > 64 || l > k || k > l) return SLRA_ERR_UNSUPPORTED;  // as the dense large path (k == l <= 64)
  const int64_t c = k, mm = m > n ? m : n;
  const size_t tw = tsqr_workspace_doubles(mm, (int)c);
  const size_t mvs = maxvol_large_scratch_doubles(cx->num_sms, mm);
  const size_t need = 2 * (size_t)mm * c + (size_t)c * c + tw + mvs + 4 * (size_t)c + 64;
  // arena 4 as the dense large path (the two are never live at once)
  double* buf = static_cast<double*>(arena(cx, 4, sizeof(double) * need));
  if (!buf) return SLRA_ERR_CUDA;
  double* S = buf;
  double* Q = S + (size_t)mm * c;
  double* R = Q + (size_t)mm * c;
  double* tws = R + (size_t)c * c;
  double* mvw = tws + tw;
  int64_t* dI = reinterpret_cast<int64_t*>(mvw + mvs);
  int64_t* dJ = dI + c;
  int64_t* iota = dJ + c;
  SLRA_CUDA(cudaMemcpyAsync(dI, init_rows, 8 * k, cudaMemcpyDeviceToDevice, cx->stream));
  for (int loop = 0; loop < loops; ++loop) {
    SLRA_TRY(launch_cauchy_strip(cx, x, y, n, dI, k, true, S, n));
    SLRA_TRY(launch_thin_qr_batched(cx, S, n, 0, n, (int)k, Q, n, 0, R, k, 0, 1, tw ? tws : nullptr));
    SLRA_TRY(launch_maxvol_large(cx, Q, n, n, (int)l, h, 4 * (int)l, dJ, trace_vol ? trace_vol + 2 * loop : nullptr,
                                 mvw));
    {
      int32_t st = 0;
      SLRA_CUDA(cudaMemcpyAsync(&st, cx->dsmall, 4, cudaMemcpyDeviceToHost, cx->stream));
      SLRA_CUDA(cudaStreamSynchronize(cx->stream));
      if (st != SLRA_OK) return st;
    }
    if (trace_rows) {
      SLRA_CUDA(cudaMemcpyAsync(trace_rows + (2 * loop) * k, dI, 8 * k, cudaMemcpyDeviceToDevice, cx->stream));
      SLRA_CUDA(cudaMemcpyAsync(trace_cols + (2 * loop) * l, dJ, 8 * l, cudaMemcpyDeviceToDevice, cx->stream));
    }
    SLRA_TRY(launch_cauchy_strip(cx, x, y, m, dJ, l, false, S, m));
    SLRA_TRY(launch_thin_qr_batched(cx, S, m, 0, m, (int)l, Q, m, 0, R, l, 0, 1, tw ? tws : nullptr));
    SLRA_TRY(launch_maxvol_large(cx, Q, m, m, (int)k, h, 4 * (int)k, dI,
                                 trace_vol ? trace_vol + 2 * loop + 1 : nullptr, mvw));
    if (trace_rows) {
      SLRA_CUDA(cudaMemcpyAsync(trace_rows + (2 * loop + 1) * k, dI, 8 * k, cudaMemcpyDeviceToDevice, cx->stream));
      SLRA_CUDA(cudaMemcpyAsync(trace_cols + (2 * loop + 1) * l, dJ, 8 * l, cudaMemcpyDeviceToDevice, cx->stream));
    }
    int32_t st = 0;
    SLRA_CUDA(cudaMemcpyAsync(&st, cx->dsmall, 4, cudaMemcpyDeviceToHost, cx->stream));
    SLRA_CUDA(cudaStreamSynchronize(cx->stream));
    if (st != SLRA_OK) return st;
  }
  SLRA_CUDA(cudaMemcpyAsync(I_out, dI, 8 * k, cudaMemcpyDeviceToDevice, cx->stream));
  SLRA_CUDA(cudaMemcpyAsync(J_out, dJ, 8 * l, cudaMemcpyDeviceToDevice, cx->stream));
  // primitive_cur on the evaluated generator G = A(I, J) (k x l) with
  // identity index sets: the nucleus depends on G alone (cur.cpp:137-162)
  double* G = S;
  cauchy_block_kernel<<<16, 256, 0, cx->stream>>>(x, y, dI, k, dJ, l, G, k);
  SLRA_CHECK_LAUNCH(cx);
  iota_kernel<<<1, 256, 0, cx->stream>>>(iota, c);
  SLRA_CHECK_LAUNCH(cx);
  return slra_primitive_cur(ctx, G, k, k, l, iota, k, iota, l, r, nucleus, l, Tsig, Sr, h_r_out);
}

int slra_cur_residual_factored_cauchy(slra_ctx ctx, const double* x, const double* y, int64_t m, int64_t n,
                                      const int64_t* I, int64_t k, const int64_t* J, int64_t l, const double* Tsig,
                                      const double* Sr, int64_t r, double* d_out) {
  if (!ctx || !x || !y || k < 1 || l < 1 || r < 1 || r > k || r > l) return SLRA_ERR_INVALID_ARGUMENT;
  Context* cx = C(ctx);
  const int64_t ldq = (r + 1) & ~1;
  const size_t need = (size_t)m * l + (size_t)k * n + (size_t)m * r + (size_t)ldq * n + 16;
  double* ws = static_cast<double*>(arena(cx, 5, sizeof(double) * need));
  if (!ws) return SLRA_ERR_CUDA;
  // the dense entry's layouts and products (slra_cur_residual_factored):
  // identical values in the same order, hence the same residual bits
  double* Cm = ws;                       // A(:, J): m x l
  double* Rm = Cm + (size_t)m * l;       // A(I, :): k x n
  double* P = Rm + (size_t)k * n;
  double* Qf = P + (size_t)m * r;
  SLRA_TRY(launch_cauchy_strip(cx, x, y, m, J, l, false, Cm, m));
  SLRA_TIMED(cx, "gather", cauchy_block_kernel<<<4 * cx->num_sms, 256, 0, cx->stream>>>(x, y, I, k, nullptr, n, Rm, k);)
  SLRA_CHECK_LAUNCH(cx);
  SLRA_TRY(launch_gemm(cx, 0, 0, m, r, l, 1.0, Cm, m, Tsig, l, 0.0, P, m));      // P = C Tsig
  SLRA_TRY(launch_gemm(cx, 1, 0, r, n, k, 1.0, Sr, k, Rm, k, 0.0, Qf, ldq));     // Q = Sr^T R
  return launch_residual_stream_cauchy(cx, x, y, m, n, P, m, Qf, ldq, r, d_out);
}

}  // extern "C"
