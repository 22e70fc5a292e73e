// Tall-skinny dense kernels behind slra_thin_qr / slra_svd / slra_maxvol_rows
// / slra_select_rows_spanning, all batched over independent problems (the
// problem index rides on a grid dimension; operands are strided) so that the
// latency-bound factorisations of several sketches overlap on separate SMs.
//   * thin_qr (linalg.cpp:67-79): one CTA when the matrix fits on chip,
//     otherwise TSQR — 256-row leaves factorised by CTA-resident Householder
//     QR, their R factors stacked and reduced level by level, then Q expanded
//     top-down by re-applying each leaf's reflectors. Unconditionally stable
//     (rank-deficient strips of configs 3/5 included).
//   * svd (linalg.cpp:81-98): one-sided Jacobi (on A^T for square inputs,
//     which converges in far fewer sweeps on the graded triangles the QR
//     pre-reduction produces), QR pre-reduction for tall inputs.
#include "blocked_qr.cuh"

namespace slra_dev {

constexpr int kDT = 512;
constexpr int kLeaf = 256;  // TSQR leaf rows
constexpr int kSVT = 256;   // threads of the one-CTA SVD (8-lane group per Jacobi pair)

// cta_thin_qr with the panel-blocked factorisation (blocked_qr.cuh, m <= 256,
// c <= 64): same reflectors, the trailing updates on DMMA, one barrier per
// column. ws: qr_ws_doubles<NT>() doubles of shared memory.
template <int NT>
__device__ void cta_thin_qr_blk(double* A, int lda, int m, int c, double* Q, int ldq, double* R, int ldr, double* tau,
                                double* red, double* ws) {
  cta_blocked_house_qr<NT>(A, lda, m, c, tau, ws);
  __syncthreads();
  cta_form_q<NT>(A, lda, m, c, tau, Q, ldq);
  for (int e = threadIdx.x; e < c * c; e += NT) {
    const int i = e % c, j = e / c;
    const double rii = A[i + i * lda];
    double v = (i <= j) ? A[i + j * lda] : 0.0;
    if (rii < 0.0) v = -v;  // flip row i of R
    R[i + j * ldr] = v;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < m * c; e += NT) {
    const int i = e % m, j = e / m;
    if (A[j + j * lda] < 0.0) Q[i + (int64_t)j * ldq] = -Q[i + (int64_t)j * ldq];  // and column i of Q
  }
  __syncthreads();
}
constexpr int kQWS = qr_ws_doubles<kDT>();

// ---------------------------------------------------------------- single-CTA thin QR
__global__ void __launch_bounds__(kDT) thin_qr_cta_kernel(const double* __restrict__ A, int64_t lda, int64_t sA,
                                                          int m, int c, double* __restrict__ Q, int64_t ldq,
                                                          int64_t sQ, double* __restrict__ R, int64_t ldr,
                                                          int64_t sR) {
  extern __shared__ __align__(16) double sm[];
  double* S = sm;                  // m x c
  double* Rs = S + (size_t)m * c;  // c x c
  double* tau = Rs + c * c;        // c
  double* red = tau + c;           // >= c + 8
  double* ws = red + c + 8;        // blocked-QR scratch (m <= 256, c <= 64)
  const int64_t b = blockIdx.x;
  A += b * sA;
  Q += b * sQ;
  for (int j = 0; j < c; ++j)
    for (int i = threadIdx.x; i < m; i += kDT) S[i + j * m] = A[i + (int64_t)j * lda];
  __syncthreads();
  if (m <= 256 && c <= 64) cta_thin_qr_blk<kDT>(S, m, m, c, Q, (int)ldq, Rs, c, tau, red, ws);
  else cta_thin_qr<kDT>(S, m, m, c, Q, (int)ldq, Rs, c, tau, red);
  if (R)
    for (int j = 0; j < c; ++j)
      for (int i = threadIdx.x; i < c; i += kDT) R[b * sR + i + (int64_t)j * ldr] = Rs[i + j * c];
}

// ---------------------------------------------------------------- TSQR
// Reduce step: block x of problem y — rows [x*L, min((x+1)*L, rows)) of X,
// padded with zeros to >= c rows — is factorised in smem; reflectors + tau go
// to Vst/taust (block x: Lp x c, ld Lp), R_x to Xn rows [x*c, (x+1)*c).
__global__ void __launch_bounds__(kDT) tsqr_reduce_kernel(const double* __restrict__ X, int64_t ldx, int64_t sX,
                                                          int64_t rows, int c, int Lp, double* __restrict__ Vst,
                                                          double* __restrict__ taust, int64_t sV,
                                                          double* __restrict__ Xn, int64_t ldxn, int64_t sXn) {
  extern __shared__ __align__(16) double sm[];
  double* S = sm;
  double* tau = S + (size_t)Lp * c;
  double* red = tau + c;          // >= c + 8 (cta_house_qr)
  double* ws = red + c + 8;       // blocked-QR scratch (Lp <= 256)
  const int64_t b = blockIdx.x, pb = blockIdx.y;
  X += pb * sX;
  Xn += pb * sXn;
  const int64_t r0 = b * kLeaf;
  const int nr = (int)((rows - r0) < kLeaf ? (rows - r0) : kLeaf);
  for (int j = 0; j < c; ++j)
    for (int i = threadIdx.x; i < Lp; i += kDT) S[i + j * Lp] = i < nr ? X[(r0 + i) + (int64_t)j * ldx] : 0.0;
  __syncthreads();
  if (Lp <= 256) cta_blocked_house_qr<kDT>(S, Lp, Lp, c, tau, ws);
  else cta_house_qr<kDT>(S, Lp, Lp, c, tau, red);
  __syncthreads();
  const int64_t nblk = gridDim.x;
  double* V = Vst + pb * sV + b * (int64_t)Lp * c;
  double* T = taust + pb * (nblk * c) + b * c;
  for (int e = threadIdx.x; e < Lp * c; e += kDT) V[e] = S[e];
  for (int j = threadIdx.x; j < c; j += kDT) T[j] = tau[j];
  for (int j = 0; j < c; ++j)
    for (int i = threadIdx.x; i < c; i += kDT) Xn[(b * c + i) + (int64_t)j * ldxn] = (i <= j) ? S[i + j * Lp] : 0.0;
}

// Top: one CTA per problem, thin QR (with sign rule) of the final stack
// (c <= rows <= L); writes Qtop (rows x c) and R.
__global__ void __launch_bounds__(kDT) tsqr_top_kernel(const double* __restrict__ X, int64_t ldx, int64_t sX, int rows,
                                                       int c, int Lp, double* __restrict__ Qt, int64_t ldqt,
                                                       int64_t sQt, double* __restrict__ R, int64_t ldr, int64_t sR) {
  extern __shared__ __align__(16) double sm[];
  double* S = sm;                   // rows x c
  double* Rs = S + (size_t)Lp * c;  // c x c
  double* tau = Rs + c * c;
  double* red = tau + c;
  double* ws = red + c + 8;
  const int64_t pb = blockIdx.x;
  X += pb * sX;
  for (int j = 0; j < c; ++j)
    for (int i = threadIdx.x; i < rows; i += kDT) S[i + j * rows] = X[i + (int64_t)j * ldx];
  __syncthreads();
  if (rows <= 256) cta_thin_qr_blk<kDT>(S, rows, rows, c, Qt + pb * sQt, (int)ldqt, Rs, c, tau, red, ws);
  else cta_thin_qr<kDT>(S, rows, rows, c, Qt + pb * sQt, (int)ldqt, Rs, c, tau, red);
  if (R)
    for (int j = 0; j < c; ++j)
      for (int i = threadIdx.x; i < c; i += kDT) R[pb * sR + i + (int64_t)j * ldr] = Rs[i + j * c];
}

// Expand step: Q_x = H_0 ... H_{c-1} [Qp(x*c : x*c+c, :); 0] (Lp x c), the
// first nr rows stored at Qo rows [x*L, ...). Reflectors staged in smem; each
// warp carries its output columns in registers (no block barriers).
template <int RPL>
__global__ void __launch_bounds__(kDT) tsqr_expand_kernel(const double* __restrict__ Qp, int64_t ldqp, int64_t sQp,
                                                          const double* __restrict__ Vst,
                                                          const double* __restrict__ taust, int64_t sV, int64_t rows,
                                                          int c, int Lp, double* __restrict__ Qo, int64_t ldqo,
                                                          int64_t sQo) {
  extern __shared__ __align__(16) double sm[];
  double* V = sm;  // Lp x c reflectors
  double* tau = V + (size_t)Lp * c;
  const int64_t b = blockIdx.x, pb = blockIdx.y, nblk = gridDim.x;
  Qp += pb * sQp;
  Qo += pb * sQo;
  const int64_t r0 = b * kLeaf;
  const int nr = (int)((rows - r0) < kLeaf ? (rows - r0) : kLeaf);
  const double* Vg = Vst + pb * sV + b * (int64_t)Lp * c;
  for (int e = threadIdx.x; e < Lp * c; e += kDT) V[e] = Vg[e];
  for (int j = threadIdx.x; j < c; j += kDT) tau[j] = taust[pb * (nblk * c) + b * c + j];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = kDT / 32;
  constexpr int CPW = (64 + NW - 1) / NW;  // c <= 64: every column of this warp at once
  double y[CPW][RPL];
#pragma unroll
  for (int q = 0; q < CPW; ++q) {
    const int j = warp + q * NW;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = lane + 32 * r;
      y[q][r] = (j < c && i < c) ? Qp[(b * c + i) + (int64_t)j * ldqp] : 0.0;
    }
  }
  {  // uniform control flow around the shuffles; tau = 0 is an exact no-op
    for (int k = c - 1; k >= 0; --k) {
      const double t = tau[k];
      const double* v = V + (size_t)k * Lp;
      double vr[RPL];
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int i = lane + 32 * r;
        vr[r] = (i > k && i < Lp) ? v[i] : (i == k ? 1.0 : 0.0);  // implicit unit head
      }
      double w[CPW];
#pragma unroll
      for (int q = 0; q < CPW; ++q) {
        w[q] = 0.0;
#pragma unroll
        for (int r = 0; r < RPL; ++r) w[q] = fma(vr[r], y[q][r], w[q]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int q = 0; q < CPW; ++q) w[q] += __shfl_xor_sync(0xffffffffu, w[q], o);
#pragma unroll
      for (int q = 0; q < CPW; ++q)
#pragma unroll
        for (int r = 0; r < RPL; ++r) y[q][r] -= t * vr[r] * w[q];
    }
  }
#pragma unroll
  for (int q = 0; q < CPW; ++q) {
    const int j = warp + q * NW;
    if (j < c) {
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int i = lane + 32 * r;
        if (i < nr) Qo[(r0 + i) + (int64_t)j * ldqo] = y[q][r];
      }
    }
  }
}

static size_t qr_cta_smem(int m, int c) {
  return sizeof(double) * ((size_t)m * c + (size_t)c * c + c + 112 + (m <= 256 && c <= 64 ? kQWS : 0));
}

// Workspace doubles needed by launch_thin_qr_batched for one problem.
size_t tsqr_workspace_doubles(int64_t m, int c) {
  if (qr_cta_smem((int)m, c) <= 227 * 1024 && m <= 256) return 0;
  const int Lp = kLeaf > c ? kLeaf : c;
  size_t total = 0;
  int64_t rows = m, first_upper = -1;
  while (rows > kLeaf) {
    const int64_t nb = (rows + kLeaf - 1) / kLeaf;
    total += (size_t)nb * Lp * c + (size_t)nb * c + (size_t)nb * c * c;
    rows = nb * c;
    if (first_upper < 0) first_upper = rows;
  }
  total += 2 * (size_t)(first_upper > 0 ? first_upper : rows) * c + (size_t)rows * c;
  return total;
}

// Batched thin QR of nb problems (A + b*sA, Q + b*sQ, R + b*sR). `ws` (may
// be null -> context workspace) holds nb * tsqr_workspace_doubles(m, c).
int launch_thin_qr_batched(Context* cx, const double* A, int64_t lda, int64_t sA, int64_t m, int c, double* Q,
                           int64_t ldq, int64_t sQ, double* R, int64_t ldr, int64_t sR, int nb, double* ws) {
  if (qr_cta_smem((int)m, c) <= 227 * 1024 && m <= 256) {
    const size_t smem = qr_cta_smem((int)m, c);
    SLRA_CUDA(cudaFuncSetAttribute(thin_qr_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SLRA_TIMED(cx, "thin_qr", thin_qr_cta_kernel<<<nb, kDT, smem, cx->stream>>>(A, lda, sA, (int)m, c, Q, ldq, sQ, R,
                                                                               ldr, sR);)
    SLRA_CHECK_LAUNCH(cx);
    return SLRA_OK;
  }
  if (c > 64) return SLRA_ERR_UNSUPPORTED;
  const int Lp = kLeaf > c ? kLeaf : c;
  std::vector<int64_t> level_rows;  // rows of X at each reduce level
  int64_t rows = m;
  while (rows > kLeaf) {
    level_rows.push_back(rows);
    rows = ((rows + kLeaf - 1) / kLeaf) * c;
  }
  const int64_t top_rows = rows;
  const size_t per = tsqr_workspace_doubles(m, c);
  if (!ws) ws = static_cast<double*>(workspace(cx, sizeof(double) * per * nb));
  if (!ws) return SLRA_ERR_CUDA;
  // per-level arrays laid out problem-major inside each level region
  std::vector<double*> V(level_rows.size()), T(level_rows.size()), X(level_rows.size());
  std::vector<int64_t> sVl(level_rows.size()), sXl(level_rows.size());
  double* cur = ws;
  for (size_t lv = 0; lv < level_rows.size(); ++lv) {
    const int64_t nblk = (level_rows[lv] + kLeaf - 1) / kLeaf;
    sVl[lv] = nblk * (int64_t)Lp * c;
    V[lv] = cur;
    cur += (size_t)sVl[lv] * nb;
    T[lv] = cur;
    cur += (size_t)nblk * c * nb;
    sXl[lv] = nblk * (int64_t)c * c;
    X[lv] = cur;
    cur += (size_t)sXl[lv] * nb;
  }
  const int64_t qup = level_rows.size() > 1 ? level_rows[1] : top_rows;
  double* qbuf[2] = {cur, cur + (size_t)qup * c * nb};
  double* Qtop = cur + 2 * (size_t)qup * c * nb;
  const size_t sm_red = sizeof(double) * ((size_t)Lp * c + 2 * (size_t)c + 8 + (Lp <= 256 ? kQWS : 0) + 8);
  SLRA_CUDA(cudaFuncSetAttribute(tsqr_reduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_red));
  const double* Xc = A;
  int64_t ldx = lda, sX = sA;
  for (size_t lv = 0; lv < level_rows.size(); ++lv) {
    const int64_t lr = level_rows[lv];
    const int64_t nblk = (lr + kLeaf - 1) / kLeaf;
    SLRA_TIMED(cx, "thin_qr",
               tsqr_reduce_kernel<<<dim3((unsigned)nblk, nb), kDT, sm_red, cx->stream>>>(
                   Xc, ldx, sX, lr, c, Lp, V[lv], T[lv], sVl[lv], X[lv], nblk * c, sXl[lv]);)
    SLRA_CHECK_LAUNCH(cx);
    Xc = X[lv];
    ldx = nblk * c;
    sX = sXl[lv];
  }
  const size_t sm_top = sizeof(double) * ((size_t)Lp * c + (size_t)c * c + c + 112 + kQWS);
  SLRA_CUDA(cudaFuncSetAttribute(tsqr_top_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_top));
  SLRA_TIMED(cx, "thin_qr",
             tsqr_top_kernel<<<nb, kDT, sm_top, cx->stream>>>(Xc, ldx, sX, (int)top_rows, c, Lp, Qtop, top_rows,
                                                              top_rows * c, R, ldr, sR);)
  SLRA_CHECK_LAUNCH(cx);
  const size_t sm_exp = sizeof(double) * ((size_t)Lp * c + c);
  SLRA_CUDA(cudaFuncSetAttribute(tsqr_expand_kernel<kLeaf / 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm_exp));
  const double* Qp = Qtop;
  int64_t ldqp = top_rows, sQp = top_rows * c;
  for (int lv = (int)level_rows.size() - 1; lv >= 0; --lv) {
    const int64_t lr = level_rows[lv];
    const int64_t nblk = (lr + kLeaf - 1) / kLeaf;
    double* Qo;
    int64_t ldqo, sQo;
    if (lv == 0) {
      Qo = Q;
      ldqo = ldq;
      sQo = sQ;
    } else {
      Qo = qbuf[lv & 1];
      ldqo = lr;
      sQo = lr * c;
    }
    SLRA_TIMED(cx, "thin_qr",
               tsqr_expand_kernel<kLeaf / 32><<<dim3((unsigned)nblk, nb), kDT, sm_exp, cx->stream>>>(
                   Qp, ldqp, sQp, V[lv], T[lv], sVl[lv], lr, c, Lp, Qo, ldqo, sQo);)
    SLRA_CHECK_LAUNCH(cx);
    Qp = Qo;
    ldqp = ldqo;
    sQp = sQo;
  }
  return SLRA_OK;
}

int launch_thin_qr(Context* cx, const double* A, int64_t lda, int64_t m, int c, double* Q, int64_t ldq, double* R,
                   int64_t ldr) {
  return launch_thin_qr_batched(cx, A, lda, 0, m, c, Q, ldq, 0, R, ldr, 0, 1, nullptr);
}

// ---------------------------------------------------------------- small SVD
// One CTA per problem: W = A (p x q, m > n) or A^T (m <= n: square inputs
// take this path too), Jacobi, finish; S (m x min), sigma, T (n x min).
__global__ void __launch_bounds__(kSVT) svd_cta_kernel(const double* __restrict__ A, int64_t lda, int64_t sA, int m,
                                                       int n, double* __restrict__ S, int64_t lds, int64_t sS,
                                                       double* __restrict__ sigma, int64_t sSig,
                                                       double* __restrict__ T, int64_t ldt, int64_t sT,
                                                       double deflate) {
  extern __shared__ __align__(16) double sm[];
  const int64_t pb = blockIdx.x;
  A += pb * sA;
  S += pb * sS;
  sigma += pb * sSig;
  T += pb * sT;
  const bool tall = m > n;
  const int p = tall ? m : n, q = tall ? n : m;
  // odd leading dimensions for the Jacobi operands: the 8-lane groups of a
  // warp read four different columns, which an even ld would put on the
  // same banks
  // (square p = q in {16, 32, 48, 64}: even, and the Jacobi moves 16-byte row
  // pairs — conflict-free for any pair of columns, dense_cta.cuh)
  const bool vec = p == q && (p & 15) == 0 && p <= 64;
  const int ldw = vec ? p : (p | 1), ldv = vec ? q : (q | 1);
  double* W = sm;                     // p x q (ld ldw)
  double* V = W + (size_t)ldw * q;    // q x q (ld ldv)
  double* Ss = V + (size_t)ldv * q;   // p x q
  double* Ts = Ss + (size_t)p * q;    // q x q
  double* sg = Ts + (size_t)q * q;    // q
  double* tmp = sg + q;               // q
  int* order = reinterpret_cast<int*>(tmp + q);
  int* flag = order + q + 1;
  for (int j = 0; j < n; ++j)
    for (int i = threadIdx.x; i < m; i += kSVT) {
      const double x = A[i + (int64_t)j * lda];
      if (tall) W[i + j * ldw] = x;
      else W[j + i * ldw] = x;
    }
  __syncthreads();
  cta_jacobi<kSVT, 256, true>(W, ldw, p, q, V, ldv, flag, deflate);
  cta_svd_finish<kSVT>(W, ldw, p, q, V, ldv, sg, order, Ss, p, Ts, q, tmp);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (!tall) {
    // left vectors of A are Ts (q x q = m x m); re-apply the sign rule on them
    for (int t = warp; t < q; t += kSVT / 32) {
      ArgMax a{-1.0, INT64_MAX};
      for (int i = lane; i < q; i += 32) a = argmax_merge(a, ArgMax{fabs(Ts[i + t * q]), i});
      a = warp_argmax(a);
      const double f = (Ts[a.i + t * q] < 0.0) ? -1.0 : 1.0;
      __syncwarp();
      for (int i = lane; i < q; i += 32) Ts[i + t * q] *= f;
      for (int i = lane; i < p; i += 32) Ss[i + t * p] *= f;
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < q; t += kSVT) sigma[t] = sg[t];
  const double* Sl = tall ? Ss : Ts;
  const int ldl = tall ? p : q;
  const double* Tr = tall ? Ts : Ss;
  const int ldr = tall ? q : p;
  for (int j = 0; j < q; ++j) {
    for (int i = threadIdx.x; i < m; i += kSVT) S[i + (int64_t)j * lds] = Sl[i + j * ldl];
    for (int i = threadIdx.x; i < n; i += kSVT) T[i + (int64_t)j * ldt] = Tr[i + j * ldr];
  }
}

static size_t svd_smem(int m, int n) {
  const int p = m > n ? m : n, q = m > n ? n : m;
  return sizeof(double) * (2 * (size_t)(p + 1) * q + 2 * (size_t)(q + 1) * q + 2 * (size_t)q + 8) +
         sizeof(int) * (q + 8);
}

int launch_svd_small_batched(Context* cx, const double* A, int64_t lda, int64_t sA, int m, int n, double* S,
                             int64_t lds, int64_t sS, double* sigma, int64_t sSig, double* T, int64_t ldt, int64_t sT,
                             int nb, double deflate) {
  const size_t smem = svd_smem(m, n);
  if (smem > 220 * 1024 || (m > n ? m : n) > 256) return SLRA_ERR_UNSUPPORTED;
  SLRA_CUDA(cudaFuncSetAttribute(svd_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SLRA_TIMED(cx, "svd", svd_cta_kernel<<<nb, kSVT, smem, cx->stream>>>(A, lda, sA, m, n, S, lds, sS, sigma, sSig, T,
                                                                      ldt, sT, deflate);)
  SLRA_CHECK_LAUNCH(cx);
  return SLRA_OK;
}

int launch_svd_small(Context* cx, const double* A, int64_t lda, int m, int n, double* S, int64_t lds, double* sigma,
                     double* T, int64_t ldt, double deflate) {
  return launch_svd_small_batched(cx, A, lda, 0, m, n, S, lds, 0, sigma, 0, T, ldt, 0, 1, deflate);
}

int launch_gemm(Context* c, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
                int64_t lda, const double* B, int64_t ldb, double beta, double* Cm, int64_t ldc);

// Sign rule on an externally formed S = Q U_R: per column j of problem y, if
// the first largest-|.| entry is negative flip S(:, j) and T(:, j).
__global__ void __launch_bounds__(kDT) colsign_kernel(double* __restrict__ S, int64_t lds, int64_t sS, int64_t m,
                                                      double* __restrict__ T, int64_t ldt, int64_t sT, int64_t n) {
  __shared__ double rv[40];
  __shared__ int64_t ri[40];
  const int64_t j = blockIdx.x;
  S += blockIdx.y * sS;
  if (T) T += blockIdx.y * sT;
  ArgMax a{-1.0, INT64_MAX};
  for (int64_t i = threadIdx.x; i < m; i += kDT) a = argmax_merge(a, ArgMax{fabs(S[i + j * lds]), i});
  a = block_argmax<kDT>(a, rv, ri);
  if (S[a.i + j * lds] < 0.0) {
    for (int64_t i = threadIdx.x; i < m; i += kDT) S[i + j * lds] = -S[i + j * lds];
    if (T)
      for (int64_t i = threadIdx.x; i < n; i += kDT) T[i + j * ldt] = -T[i + j * ldt];
  }
}

int launch_colsign_batched(Context* cx, double* S, int64_t lds, int64_t sS, int64_t m, double* T, int64_t ldt,
                           int64_t sT, int64_t n, int64_t cols, int nb) {
  if (cols <= 0) return SLRA_OK;
  SLRA_TIMED(cx, "colsign", colsign_kernel<<<dim3((unsigned)cols, nb), kDT, 0, cx->stream>>>(S, lds, sS, m, T, ldt, sT,
                                                                                        n);)
  SLRA_CHECK_LAUNCH(cx);
  return SLRA_OK;
}

int launch_colsign(Context* cx, double* S, int64_t lds, int64_t m, double* T, int64_t ldt, int64_t n, int64_t cols) {
  return launch_colsign_batched(cx, S, lds, 0, m, T, ldt, 0, n, cols, 1);
}

__global__ void transpose_kernel(const double* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                                 double* __restrict__ B, int64_t ldb) {
  __shared__ double tile[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int64_t i = i0 + threadIdx.x, j = j0 + dy;
    if (i < m && j < n) tile[dy][threadIdx.x] = A[i + j * lda];
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int64_t j = j0 + threadIdx.x, i = i0 + dy;
    if (i < m && j < n) B[j + i * ldb] = tile[threadIdx.x][dy];
  }
}

int launch_transpose(Context* cx, const double* A, int64_t lda, int64_t m, int64_t n, double* B, int64_t ldb) {
  dim3 grid(ceil_div(m, 32), ceil_div(n, 32));
  SLRA_TIMED(cx, "transpose", transpose_kernel<<<grid, dim3(32, 8), 0, cx->stream>>>(A, lda, m, n, B, ldb);)
  SLRA_CHECK_LAUNCH(cx);
  return SLRA_OK;
}

// General SVD with min(m, n) <= 64: small -> one CTA; tall -> thin_qr then
// Jacobi on R and S = Q U_R (plus the sign rule on S); wide -> via A^T.
size_t svd_large_workspace_doubles(int64_t m, int64_t n, int nb);
int launch_svd_large_batched(Context* cx, const double* A, int64_t lda, int64_t sA, int m, int n, int nb,
                             double* S, int64_t lds, int64_t sS, double* sigma, int64_t sSig, double* T, int64_t ldt,
                             int64_t sT, double* ws);

int launch_svd(Context* cx, const double* A, int64_t lda, int64_t m, int64_t n, double* S, int64_t lds,
               double* sigma, double* T, int64_t ldt) {
  const int64_t q = m < n ? m : n;
  if (q > 64 && m >= n) {  // multi-CTA Jacobi in HBM (svd_large.cu)
    if (m > INT32_MAX / 2 || n > 16384) return SLRA_ERR_UNSUPPORTED;
    double* ws = static_cast<double*>(arena(cx, 10, sizeof(double) * svd_large_workspace_doubles(m, n, 1)));
    if (!ws) return SLRA_ERR_CUDA;
    return launch_svd_large_batched(cx, A, lda, 0, (int)m, (int)n, 1, S, lds, 0, sigma, 0, T, ldt, 0, ws);
  }
  if (q <= 64 && svd_smem((int)m, (int)n) <= 200 * 1024 && (m > n ? m : n) <= 256)
    return launch_svd_small(cx, A, lda, (int)m, (int)n, S, lds, sigma, T, ldt, 0.0);
  if (m < n) {
    // wide: A^T = S' Sigma T'^T (tall path), so A = T' Sigma S'^T; the sign
    // rule is then re-applied on the left vectors T' (flipping S' with them).
    double* At = static_cast<double*>(arena(cx, 6, sizeof(double) * (size_t)m * n));  // slot 3 is the tall path's
    if (!At) return SLRA_ERR_CUDA;
    SLRA_TRY(launch_transpose(cx, A, lda, m, n, At, n));
    SLRA_TRY(launch_svd(cx, At, n, n, m, T, ldt, sigma, S, lds));
    return launch_colsign(cx, S, lds, m, T, ldt, n, m);
  }
  const int c = (int)n;
  // scratch: Q (m x c), R (c x c), UR (c x c) + the TSQR workspace
  const size_t tw = tsqr_workspace_doubles(m, c);
  double* buf = static_cast<double*>(arena(cx, 3, sizeof(double) * ((size_t)m * c + 2 * (size_t)c * c + tw)));
  if (!buf) return SLRA_ERR_CUDA;
  double* Qm = buf;
  double* Rm = buf + (size_t)m * c;
  double* UR = Rm + (size_t)c * c;
  double* tws = UR + (size_t)c * c;
  SLRA_TRY(launch_thin_qr_batched(cx, A, lda, 0, m, c, Qm, m, 0, Rm, c, 0, 1, tw ? tws : nullptr));
  SLRA_TRY(launch_svd_small(cx, Rm, c, c, c, UR, c, sigma, T, ldt, 0.0));
  SLRA_TRY(launch_gemm(cx, 0, 0, m, c, c, 1.0, Qm, m, UR, c, 0.0, S, lds));
  return launch_colsign(cx, S, lds, m, T, ldt, n, c);
}

// ---------------------------------------------------------------- maxvol / select
__global__ void __launch_bounds__(kDT) maxvol_cta_kernel(const double* __restrict__ A, int64_t lda, int m, int r,
                                                         double h, int max_swaps, int qr_first, int count,
                                                         int64_t* __restrict__ idx, double* __restrict__ vol,
                                                         int32_t* __restrict__ status) {
  extern __shared__ __align__(16) double sm[];
  double* S = sm;                    // m x r
  double* W = S + (size_t)m * r;     // m x r
  double* Rs = W + (size_t)m * r;    // r x r
  double* Gt = Rs + (size_t)r * r;   // r x r
  double* tau = Gt + (size_t)r * r;  // r
  double* v = tau + r;               // r
  double* nu = v + r;                // m
  double* nd = nu + m;               // m
  double* rv = nd + m;               // 112 (reduction scratch, >= r + 8)
  int64_t* ri = reinterpret_cast<int64_t*>(rv + 112);  // 40
  int* p2r = reinterpret_cast<int*>(ri + 40);          // m
  int* I = p2r + m;                                    // count
  int* perm = I + (count > r ? count : r);             // r
  int* flag = perm + r;                                // 4
  for (int j = 0; j < r; ++j)
    for (int i = threadIdx.x; i < m; i += kDT) S[i + j * m] = A[i + (int64_t)j * lda];
  __syncthreads();
  if (qr_first) {
    cta_thin_qr<kDT>(S, m, m, r, W, m, Rs, r, tau, rv);  // Q -> W, then swap roles
    double* t = S;
    S = W;
    W = t;
  }
  const int rq = count < r ? count : r;
  ColPivScratch cs{W, m, p2r, nu, nd, v, tau, rv, ri};
  cta_colpiv_init<kDT>(S, m, m, rq, cs, I);
  __syncthreads();
  const int st = cta_maxvol_swaps<kDT>(S, m, m, rq, h, max_swaps, I, W, m, Gt, rq, perm, tau, nu, nd, rv, ri, flag);
  if (st != SLRA_OK) {
    if (threadIdx.x == 0) *status = st;
    return;
  }
  __syncthreads();
  if (count > rq) {
    for (int i = threadIdx.x; i < m; i += kDT) {
      double acc = 0.0;
      for (int j = 0; j < r; ++j) acc += S[i + j * m] * S[i + j * m];
      nu[i] = sqrt(acc);
    }
    __syncthreads();
    for (int t = rq; t < count; ++t) {
      ArgMax a{-1.0, INT64_MAX};
      for (int i = threadIdx.x; i < m; i += kDT) {
        bool used = false;
        for (int u = 0; u < t; ++u) used |= (I[u] == i);
        if (!used) a = argmax_merge(a, ArgMax{nu[i], i});
      }
      a = block_argmax<kDT>(a, rv, ri);
      if (threadIdx.x == 0) I[t] = (int)a.i;
      __syncthreads();
    }
  }
  for (int t = threadIdx.x; t < count; t += kDT) idx[t] = I[t];
  if (vol) {
    if (count == r) {
      for (int e = threadIdx.x; e < r * r; e += kDT) Gt[(e % r) + (e / r) * r] = S[I[e % r] + (e / r) * m];
      __syncthreads();
      if (threadIdx.x < 32) {
        const double dv = warp_abs_det(Gt, r, r);
        if (threadIdx.x == 0) *vol = dv;
      }
    } else if (threadIdx.x == 0) {
      *vol = 0.0;
    }
  }
  if (threadIdx.x == 0) *status = SLRA_OK;
}

static size_t maxvol_smem(int m, int r, int count) {
  const int cm = count > r ? count : r;
  return sizeof(double) * (2 * (size_t)m * r + 2 * (size_t)r * r + 2 * (size_t)r + 2 * (size_t)m + 112) +
         sizeof(int64_t) * 40 + sizeof(int) * ((size_t)m + cm + r + 8);
}

int launch_maxvol(Context* cx, const double* A, int64_t lda, int64_t m, int64_t r, double h, int64_t max_swaps,
                  int qr_first, int64_t count, int64_t* idx, double* vol) {
  const size_t smem = maxvol_smem((int)m, (int)r, (int)count);
  if (smem > 220 * 1024 || r > 64 || (qr_first && m > 256)) return SLRA_ERR_UNSUPPORTED;
  SLRA_CUDA(cudaFuncSetAttribute(maxvol_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int32_t* d_status = static_cast<int32_t*>(cx->dsmall);
  SLRA_TIMED(cx, "maxvol",
             maxvol_cta_kernel<<<1, kDT, smem, cx->stream>>>(A, lda, (int)m, (int)r, h, (int)max_swaps, qr_first,
                                                             (int)count, idx, vol, d_status);)
  SLRA_CHECK_LAUNCH(cx);
  SLRA_CUDA(cudaMemcpyAsync(cx->hsmall, cx->dsmall, 4, cudaMemcpyDeviceToHost, cx->stream));
  SLRA_CUDA(cudaStreamSynchronize(cx->stream));
  return *static_cast<int32_t*>(cx->hsmall);
}

size_t maxvol_large_scratch_doubles(int num_sms, int64_t m);
int launch_maxvol_large(Context* cx, const double* Q, int64_t ldq, int64_t m, int r, double h, int max_swaps,
                        int64_t* d_idx, double* d_vol, double* scratch);

// maxvol / select_rows_spanning on strips taller than one SM: (TSQR when
// qr_first) then the grid-wide maxvol; blocks until the status is known.
int launch_maxvol_tall(Context* cx, const double* A, int64_t lda, int64_t m, int r, double h, int max_swaps,
                       int64_t* idx, double* vol, bool qr_first) {
  const size_t tw = qr_first ? tsqr_workspace_doubles(m, r) : 0;
  const size_t mvs = maxvol_large_scratch_doubles(cx->num_sms, m);
  const size_t qsz = qr_first ? (size_t)m * r + (size_t)r * r : 0;
  double* buf = static_cast<double*>(arena(cx, 7, sizeof(double) * (qsz + tw + mvs + 64)));
  if (!buf) return SLRA_ERR_CUDA;
  const double* Q = A;
  int64_t ldq = lda;
  if (qr_first) {
    double* Qm = buf;
    SLRA_TRY(launch_thin_qr_batched(cx, A, lda, 0, m, r, Qm, m, 0, Qm + (size_t)m * r, r, 0, 1,
                                    tw ? buf + qsz : nullptr));
    Q = Qm;
    ldq = m;
  }
  SLRA_TRY(launch_maxvol_large(cx, Q, ldq, m, r, h, max_swaps, idx, vol, buf + qsz + tw));
  SLRA_CUDA(cudaMemcpyAsync(cx->hsmall, cx->dsmall, 4, cudaMemcpyDeviceToHost, cx->stream));
  SLRA_CUDA(cudaStreamSynchronize(cx->stream));
  return *static_cast<int32_t*>(cx->hsmall);
}

}  // namespace slra_dev

using namespace slra_dev;

extern "C" {

int slra_thin_qr(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t c, double* Q, int64_t ldq, double* R,
                 int64_t ldr) {
  if (!ctx || m < c || c < 1 || lda < m || ldq < m || (R && ldr < c)) return SLRA_ERR_INVALID_ARGUMENT;
  if (c > 64) return SLRA_ERR_UNSUPPORTED;
  return launch_thin_qr(C(ctx), A, lda, m, (int)c, Q, ldq, R, ldr);
}

int slra_svd(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t n, double* S, int64_t lds, double* sigma,
             double* T, int64_t ldt) {
  if (!ctx || m < 1 || n < 1 || lda < m || lds < m || ldt < n) return SLRA_ERR_INVALID_ARGUMENT;
  return launch_svd(C(ctx), A, lda, m, n, S, lds, sigma, T, ldt);
}

int slra_maxvol_rows(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t r, double h, int64_t max_swaps,
                     int64_t* idx) {
  if (!ctx || r < 1 || m < r || lda < m || h < 1.0) return SLRA_ERR_INVALID_ARGUMENT;
  if (max_swaps == 0) max_swaps = 4 * r;
  const int st = launch_maxvol(C(ctx), A, lda, m, r, h, max_swaps, 0, r, idx, nullptr);
  if (st != SLRA_ERR_UNSUPPORTED || r > 64) return st;
  return launch_maxvol_tall(C(ctx), A, lda, m, (int)r, h, (int)max_swaps, idx, nullptr, false);
}

int slra_select_rows_spanning(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t c, int64_t count,
                              double h, int64_t* idx, double* vol) {
  if (!ctx || count > m || m < c || c < 1 || lda < m) return SLRA_ERR_INVALID_ARGUMENT;
  const int64_t rq = count < c ? count : c;
  const int st = launch_maxvol(C(ctx), A, lda, m, c, h, 4 * rq, 1, count, idx, vol);
  // tall strips (config 3 and the row-sharded path): TSQR + grid-wide maxvol;
  // the padding branch (count > c, cur.cpp:125-134) is not needed there
  if (st != SLRA_ERR_UNSUPPORTED || c > 64 || count != c) return st;
  return launch_maxvol_tall(C(ctx), A, lda, m, (int)c, h, (int)(4 * c), idx, vol, true);
}

}  // extern "C"
