// Shifted CholeskyQR3 (Fukaya, Kannan, Nakatsukasa, Yamamoto, Yanagisawa,
// "Shifted Cholesky QR for computing the QR factorization of ill-conditioned
// matrices", SISC 2020) for the tall-skinny sketch Y = M H of the range
// finder (lra.cpp:14-39, thin_qr linalg.cpp:67-79).
//
// Why here: Householder QR of a 4096 x 48 strip is a chain of 48 dependent
// column steps per tree level (latency-bound on one SM per leaf); CholeskyQR
// is three rounds of {Gram, an n x n Cholesky, a row-parallel triangular
// solve}. Pass 1 adds the shift s = 11 (m n + n (n + 1)) u ||Y||_F^2 so the
// Cholesky succeeds for cond(Y) up to ~1/u; passes 2-3 restore orthogonality
// to O(u). R = R3 R2 R1 has a positive diagonal — thin_qr's R(i,i) >= 0
// convention. Q spans the same space as Householder's Q; the range finder
// consumes only the top-r singular subspace of R, which is well conditioned
// here, so the result matches the oracle within tolerance. A Cholesky
// breakdown (cond(Y) beyond ~1/u, e.g. an exactly rank-deficient sketch) sets
// status[b] = 1 and the caller falls back to the Householder TSQR.
//
// Kernels per pass (templated on NP = n rounded up to a multiple of 8, so
// every loop bound is a compile-time constant — FP64 dependent latency is
// ~24 cycles here and index/predicate arithmetic was most of the issue
// slots): gram_partial_kernel (row chunks -> partial NP x NP Grams, no
// atomics), chol_small_kernel (sums the partials in a fixed order, shift,
// Cholesky padded with the identity beyond n, 1/R(i,i)), trsm_rows_kernel
// (Q = Y R^-1, a thread per row, right-looking in registers).
#include "common.cuh"

namespace slra_dev {

constexpr int kCQ = 256;
constexpr int kCQMax = 64;
constexpr int kGR = 128;  // rows per Gram chunk

// P_{b,k} = Y_b(chunk k, :)^T Y_b(chunk k, :) for chunk k = blockIdx.x
// (upper triangle, NP x NP with zero columns beyond n).
template <int NP>
__global__ void __launch_bounds__(kCQ) gram_partial_kernel(const double* __restrict__ Y, int64_t ldy, int64_t sY,
                                                           int64_t m, int n, double* __restrict__ P, int64_t sP,
                                                           const int32_t* __restrict__ status) {
  extern __shared__ __align__(16) double T[];  // chunk rows, ld kGR + 1 per column (odd: conflict-free)
  constexpr int ldt = kGR + 1;
  const int b = blockIdx.y, k = blockIdx.x, tid = threadIdx.x;
  if (status[b]) return;
  Y += b * sY;
  const int64_t r0 = (int64_t)k * kGR;
  const int rows = (int)((m - r0) < kGR ? (m - r0) : kGR);
#pragma unroll 4
  for (int e = tid; e < kGR * NP; e += kCQ) {
    const int i = e % kGR, c = e / kGR;
    T[i + c * ldt] = load_sel(Y, (r0 + i) + (int64_t)c * ldy, i < rows && c < n);
  }
  __syncthreads();
  double* out = P + b * sP + (int64_t)k * NP * NP;
  constexpr int NB = NP / 2;  // 2 x 2 output blocks: four independent FMA chains per thread
  for (int e = tid; e < NB * NB; e += kCQ) {
    const int bi = e % NB, bc = e / NB;
    if (bi > bc) continue;
    const int i0 = 2 * bi, c0 = 2 * bc;
    const double* a0 = T + i0 * ldt;
    const double* d0 = T + c0 * ldt;
    double s00 = 0.0, s01 = 0.0, s10 = 0.0, s11 = 0.0;
#pragma unroll 8
    for (int t = 0; t < kGR; ++t) {
      const double x0 = a0[t], x1 = a0[t + ldt], y0 = d0[t], y1 = d0[t + ldt];
      s00 = fma(x0, y0, s00);
      s01 = fma(x0, y1, s01);
      s10 = fma(x1, y0, s10);
      s11 = fma(x1, y1, s11);
    }
    out[i0 + c0 * NP] = s00;
    out[i0 + (c0 + 1) * NP] = s01;
    out[(i0 + 1) + c0 * NP] = s10;  // below the diagonal when bi == bc: unused
    out[(i0 + 1) + (c0 + 1) * NP] = s11;
  }
}

// Upper Cholesky factor R of G + shift*I (first n entries) padded with the
// identity beyond n, where G = the sum of the nchunk partial Grams (chunk
// order fixed); shift = shift_coef * trace(G). Thread (row ti, phase tc)
// owns L(ti, c) for c = tc, tc + 4, ...: each column step stages column j in
// registers, then writes (two barriers per step). Writes R (n x n, ld n),
// and 1/R(i,i) for all NP entries. A breakdown sets status[b] = 1.
template <int NP>
__global__ void __launch_bounds__(kCQ) chol_small_kernel(const double* __restrict__ P, int64_t sP, int nchunk, int n,
                                                         double shift_coef, double* __restrict__ R, int64_t sR,
                                                         double* __restrict__ rinv, int64_t sRi,
                                                         int32_t* __restrict__ status) {
  constexpr int ld = NP + 1;
  __shared__ double L[NP * ld];  // L(i, c) at i + c * ld, lower triangle
  __shared__ double red[40];
  __shared__ int fail;
  const int b = blockIdx.x, tid = threadIdx.x;
  if (status[b]) return;
  P += b * sP;
  R += b * sR;
  rinv += b * sRi;
  constexpr int NN = NP * NP;
  // upper-triangle entries only, every chunk's partial of an entry in flight
  // at once (the partials are L2 reads: this sum, not the factorisation, was
  // most of the kernel), added in chunk order
  constexpr int NU = NP * (NP + 1) / 2;
  for (int u = tid; u < NU; u += kCQ) {
    int c = (int)((sqrt(8.0 * u + 1.0) - 1.0) * 0.5);  // u = c (c + 1) / 2 + i, i <= c
    while ((c + 1) * (c + 2) / 2 <= u) ++c;
    while (c * (c + 1) / 2 > u) --c;
    const int i = u - c * (c + 1) / 2;
    const int e = i + c * NP;
    double s = 0.0;
    int k = 0;
    for (; k + 16 <= nchunk; k += 16) {
      double v[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) v[t] = P[(k + t) * NN + e];
#pragma unroll
      for (int t = 0; t < 16; ++t) s += v[t];
    }
    for (; k < nchunk; ++k) s += P[k * NN + e];
    L[c + i * ld] = s;  // lower: L(c, i) = G(i, c), c >= i
  }
  __syncthreads();
  double tr = 0.0;
  for (int i = tid; i < n; i += kCQ) tr += L[i + i * ld];
  tr = block_sum<kCQ>(tr, red);
  for (int i = tid; i < NP; i += kCQ) L[i + i * ld] = i < n ? L[i + i * ld] + shift_coef * tr : 1.0;
  if (tid == 0) fail = 0;
  __syncthreads();
  // Column-publishing right-looking factorisation (one barrier per column):
  // thread (i = tid % 64, g = tid / 64) holds A(i, g + 4 v) in registers;
  // column j, once final, sits in L(:, j) (published by its owner group at
  // the end of step j - 1) and every thread applies A(i, c) -= A(i, j) A(c, j)
  // / A(j, j) to all of its entries unconditionally — entries of published
  // columns and above the diagonal take garbage that is never read (the
  // owner of column j + 1 republishes only its unpublished columns). At the
  // end L(i, c) = A(i, c) / sqrt(A(c, c)).
  constexpr int kV = NP / 4;
  __shared__ double piv_s[NP];
  const int ti = tid & 63, tg = tid >> 6;
  double a[kV];
#pragma unroll
  for (int v = 0; v < kV; ++v) {
    const int c = tg + 4 * v;
    a[v] = (ti < NP && ti >= c) ? L[ti + c * ld] : 0.0;
  }
  for (int j = 0; j < NP; ++j) {
    const double* cj = L + j * ld;
    const double piv = cj[j];
    if (!(piv > 0.0)) {  // uniform: every thread read the same pivot
      if (tid == 0) fail = 1;
      break;
    }
    const double rp = piv >= DBL_MIN ? fast_rcp(piv) : 1.0 / piv;
    const double f = (ti > j && ti < NP) ? -cj[ti] * rp : 0.0;
#pragma unroll
    for (int v = 0; v < kV; ++v) a[v] = fma(f, cj[tg + 4 * v], a[v]);
    const int jn = j + 1;
    if (tg == (jn & 3) && ti < NP && jn < NP) {
      const int vv = jn >> 2;
#pragma unroll
      for (int v = 0; v < kV; ++v)
        if (v >= vv) L[ti + (tg + 4 * v) * ld] = a[v];
    }
    if (tid == 0) piv_s[j] = piv;
    __syncthreads();
  }
  if (fail) {
    if (tid == 0) status[b] = 1;
    return;
  }
  // R(i, c) = L(c, i) = A(c, i) / sqrt(A(i, i)) for i < c, sqrt(A(i, i)) on the diagonal
  for (int e = tid; e < n * n; e += kCQ) {
    const int i = e % n, c = e / n;
    const double pi = piv_s[i];
    const double r = fast_rsqrt(pi);
    R[e] = (i < c) ? L[c + i * ld] * r : (i == c ? pi * r : 0.0);
  }
  for (int i = tid; i < NP; i += kCQ) rinv[i] = fast_rsqrt(piv_s[i]);
}

// Q(i, :) = Y(i, :) R^-1 for every row i, one thread per row; problem
// blockIdx.y. R (n x n, ld n) is padded to NP x NP with the identity in
// shared memory; the row lives in registers and the substitution is
// right-looking (each final z(c) updates the later entries), so the
// dependent chain is one multiply + one FMA per column.
template <int NP>
__global__ void __launch_bounds__(128) trsm_rows_kernel(const double* __restrict__ Y, int64_t ldy, int64_t sY,
                                                        int64_t m, int n, const double* __restrict__ R, int64_t sR,
                                                        const double* __restrict__ rinv, int64_t sRi,
                                                        double* __restrict__ Q, int64_t ldq, int64_t sQ,
                                                        const int32_t* __restrict__ status) {
  __shared__ double Rs[NP * NP];
  __shared__ double ri[NP];
  const int b = blockIdx.y, tid = threadIdx.x;
  if (status[b]) return;
  Y += b * sY;
  Q += b * sQ;
  R += b * sR;
  rinv += b * sRi;
  for (int e = tid; e < NP * NP; e += 128) {
    const int r = e % NP, c = e / NP;
    Rs[e] = (r < n && c < n) ? R[r + c * n] : (r == c ? 1.0 : 0.0);
  }
  for (int c = tid; c < NP; c += 128) ri[c] = rinv[c];
  __syncthreads();
  const int64_t i = blockIdx.x * 128LL + tid;
  if (i >= m) return;
  double zr[NP];
#pragma unroll
  for (int c = 0; c < NP; ++c) zr[c] = load_sel(Y + i, (int64_t)c * ldy, c < n);
#pragma unroll
  for (int c = 0; c < NP; ++c) {
    const double z = zr[c] * ri[c];
    zr[c] = z;
#pragma unroll
    for (int c2 = c + 1; c2 < NP; ++c2) zr[c2] = fma(-z, Rs[c + c2 * NP], zr[c2]);
  }
#pragma unroll
  for (int c = 0; c < NP; ++c)
    if (c < n) Q[i + (int64_t)c * ldq] = zr[c];
}

// R = (R3 R2) R1 for upper-triangular n x n factors (ld n), problem
// blockIdx.x, operands staged in shared memory.
__global__ void __launch_bounds__(kCQ) trmm3_upper_kernel(const double* __restrict__ R1, const double* __restrict__ R2,
                                                          const double* __restrict__ R3, int64_t sIn, int n,
                                                          double* __restrict__ Rout, int64_t sOut, int64_t ldo,
                                                          const int32_t* __restrict__ status) {
  extern __shared__ __align__(16) double tm[];
  const int b = blockIdx.x, tid = threadIdx.x;
  if (status[b]) return;
  const int nn = n * n;
  double* A = tm;
  double* B = tm + nn;
  for (int e = tid; e < nn; e += kCQ) {
    A[e] = R3[b * sIn + e];
    B[e] = R2[b * sIn + e];
  }
  __syncthreads();
  constexpr int kPer = (kCQMax * kCQMax + kCQ - 1) / kCQ;
  double t3[kPer];
#pragma unroll
  for (int q = 0; q < kPer; ++q) {  // T = R3 R2 (upper)
    const int e = tid + q * kCQ;
    double acc = 0.0;
    if (e < nn) {
      const int i = e % n, c = e / n;
      for (int t = i; t <= c; ++t) acc = fma(A[i + t * n], B[t + c * n], acc);
    }
    t3[q] = acc;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int e = tid + q * kCQ;
    if (e < nn) {
      A[e] = t3[q];
      B[e] = R1[b * sIn + e];
    }
  }
  __syncthreads();
  for (int e = tid; e < nn; e += kCQ) {  // R = T R1
    const int i = e % n, c = e / n;
    double acc = 0.0;
    for (int t = i; t <= c; ++t) acc = fma(A[i + t * n], B[t + c * n], acc);
    Rout[b * sOut + i + (int64_t)c * ldo] = i <= c ? acc : 0.0;
  }
}

static int64_t gram_chunks(int64_t m) { return (m + kGR - 1) / kGR; }

size_t cholqr3_workspace_doubles(int64_t m, int n) {
  return (size_t)m * n + (size_t)gram_chunks(m) * kCQMax * kCQMax + 3 * (size_t)n * n + kCQMax + 8;
}

template <int NP>
static int cholqr3_passes(Context* cx, const double* Y, int64_t ldy, int64_t sY, int64_t m, int n, double* Q,
                          int64_t ldq, int64_t sQ, double* R, int64_t ldr, int64_t sR, int nb, double* ws,
                          int32_t* status) {
  const int64_t per = (int64_t)cholqr3_workspace_doubles(m, n);
  const int64_t nn = (int64_t)n * n, nch = gram_chunks(m);
  // per problem: T (m x n) | partial Grams (nch x NP x NP) | R1 | R2 | R3 | rinv (NP)
  double* T = ws;
  double* P = ws + m * n;
  double* R1 = P + nch * kCQMax * kCQMax;
  double* rinv = R1 + 3 * nn;
  const double shift_coef = 11.0 * ((double)m * n + (double)n * (n + 1)) * (2.220446049250313e-16 / 2);  // u = eps/2
  const size_t gsm_bytes = sizeof(double) * (size_t)(kGR + 1) * NP;
  SLRA_CUDA(cudaFuncSetAttribute(gram_partial_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)gsm_bytes));
  SLRA_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t) * nb, cx->stream));
  const double* src[3] = {Y, Q, T};
  const int64_t lds[3] = {ldy, ldq, m}, ss[3] = {sY, sQ, per};
  double* dst[3] = {Q, T, Q};
  const int64_t ldd[3] = {ldq, m, ldq}, sd[3] = {sQ, per, sQ};
  const dim3 gg((unsigned)nch, (unsigned)nb), tg((unsigned)((m + 127) / 128), (unsigned)nb);
  for (int pass = 0; pass < 3; ++pass) {
    double* Rk = R1 + pass * nn;
    SLRA_TIMED(cx, "cholqr_gram", gram_partial_kernel<NP><<<gg, kCQ, gsm_bytes, cx->stream>>>(
                                      src[pass], lds[pass], ss[pass], m, n, P, per, status);)
    SLRA_CHECK_LAUNCH(cx);
    SLRA_TIMED(cx, "cholqr_chol",
               chol_small_kernel<NP><<<nb, kCQ, 0, cx->stream>>>(P, per, (int)nch, n, pass == 0 ? shift_coef : 0.0,
                                                                 Rk, per, rinv, per, status);)
    SLRA_CHECK_LAUNCH(cx);
    SLRA_TIMED(cx, "cholqr_trsm",
               trsm_rows_kernel<NP><<<tg, 128, 0, cx->stream>>>(src[pass], lds[pass], ss[pass], m, n, Rk, per, rinv,
                                                                per, dst[pass], ldd[pass], sd[pass], status);)
    SLRA_CHECK_LAUNCH(cx);
  }
  const size_t msm_bytes = sizeof(double) * 2 * (size_t)nn;
  SLRA_CUDA(cudaFuncSetAttribute(trmm3_upper_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msm_bytes));
  SLRA_TIMED(cx, "cholqr_trmm", trmm3_upper_kernel<<<nb, kCQ, msm_bytes, cx->stream>>>(R1, R1 + nn, R1 + 2 * nn, per,
                                                                                        n, R, sR, ldr, status);)
  SLRA_CHECK_LAUNCH(cx);
  return SLRA_OK;
}

// Batched shifted CholeskyQR3 of nb problems Y_b (m x n, n <= 64): Q_b
// (ld ldq) and R_b (ld n) as thin_qr. ws: nb * cholqr3_workspace_doubles.
// status (device, nb ints) is zeroed here; status[b] != 0 marks a breakdown.
int launch_cholqr3_batched(Context* cx, const double* Y, int64_t ldy, int64_t sY, int64_t m, int n, double* Q,
                           int64_t ldq, int64_t sQ, double* R, int64_t ldr, int64_t sR, int nb, double* ws,
                           int32_t* status) {
  if (n < 1 || n > kCQMax || ldr != n || m < n) return SLRA_ERR_UNSUPPORTED;
  switch ((n + 7) / 8) {
    case 1: return cholqr3_passes<8>(cx, Y, ldy, sY, m, n, Q, ldq, sQ, R, ldr, sR, nb, ws, status);
    case 2: return cholqr3_passes<16>(cx, Y, ldy, sY, m, n, Q, ldq, sQ, R, ldr, sR, nb, ws, status);
    case 3: return cholqr3_passes<24>(cx, Y, ldy, sY, m, n, Q, ldq, sQ, R, ldr, sR, nb, ws, status);
    case 4: return cholqr3_passes<32>(cx, Y, ldy, sY, m, n, Q, ldq, sQ, R, ldr, sR, nb, ws, status);
    case 5: return cholqr3_passes<40>(cx, Y, ldy, sY, m, n, Q, ldq, sQ, R, ldr, sR, nb, ws, status);
    case 6: return cholqr3_passes<48>(cx, Y, ldy, sY, m, n, Q, ldq, sQ, R, ldr, sR, nb, ws, status);
    case 7: return cholqr3_passes<56>(cx, Y, ldy, sY, m, n, Q, ldq, sQ, R, ldr, sR, nb, ws, status);
    default: return cholqr3_passes<64>(cx, Y, ldy, sY, m, n, Q, ldq, sQ, R, ldr, sR, nb, ws, status);
  }
}

}  // namespace slra_dev
