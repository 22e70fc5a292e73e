// CTA-resident small dense kernels (K-b / K-n building blocks). Every routine
// runs on ONE thread block over operands in shared memory, column-major,
// and restates the Eigen decomposition the reference calls:
//   cta_house_qr     Eigen HouseholderQR (linalg.cpp:69), makeHouseholder /
//                    applyHouseholderOnTheLeft arithmetic order
//   cta_form_q       householderQ() * Identity (linalg.cpp:70), LAPACK dorg2r
//   cta_thin_qr      thin_qr incl. the R(i,i) >= 0 sign rule (linalg.cpp:72-77)
//   cta_colpiv_init  ColPivHouseholderQR(A^T) pivot order (cur.cpp:95-98),
//                    LAPACK xGEQP3 norm downdate
//   warp_colpiv_qr   ColPivHouseholderQR of a small square (cur.cpp:103-106)
//   cta_maxvol_swaps maxvol swap loop (cur.cpp:100-114): B = A G^-1 by the
//                    Eigen solve (round 0) then rank-1 updates, argmax in
//                    column-major order, first max wins
//   warp_abs_det     |det| via partial-pivot LU (cur.cpp:192-197)
//   cta_jacobi_svd   one-sided Jacobi SVD (BDCSVD stand-in, linalg.cpp:81-98)
#pragma once

#include "common.cuh"

namespace slra_dev {

constexpr double kEps = 2.220446049250313e-16;

// ---------------------------------------------------------------- Householder QR
// A (m x c, ld lda) in smem. On exit: R on/above the diagonal, essential
// Householder parts below, tau[0..min(m,c)). Warp w owns columns j = w mod
// NW; the owner of column j+1 accumulates its next tail norm while applying
// reflector j, so each column costs two block barriers. `red` >= c + 8.
// Reflector j from column j (its tail norm s = sum_{i>j} A(i,j)^2 given),
// built by the warp that owns the column: Eigen makeHouseholder.
template <int RPL, bool FAST>
__device__ __forceinline__ void house_make(double* x, int j, int m, double s, double* tau) {
  const int lane = threadIdx.x & 31;
  __syncwarp();  // the column was just written by the lanes of this warp
  const double c0 = x[j];
  double t, beta;
  if (s <= DBL_MIN) {  // Eigen makeHouseholder: tau = 0, beta = c0
    t = 0.0;
    beta = c0;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = lane + 32 * r;
      if (i > j && i < m) x[i] = 0.0;
    }
  } else {
    double rden;
    if constexpr (FAST) {
      // MUFU-seeded, ~1 ulp, and arranged for the shortest dependent chain
      // (FP64 dependent latency is ~35-40 cycles and this runs once per
      // column on the critical path): y = rsqrt(v) by one cubically
      // convergent step from the seed; c0 - beta = sgn (|c0| + v y) needs no
      // corrected sqrt; tau = (beta - c0) / beta = 1 + |c0| y needs no
      // division; beta = -sgn sqrt(v) (corrected) is off the chain.
      const double v = fma(c0, c0, s), ac = fabs(c0);
      const double y0 = mufu_rsqrt(v);
      const double e = fma(-(v * y0), y0, 1.0);
      const double y = fma(y0, e * fma(0.375, e, 0.5), y0);
      const double den = fma(v, y, ac);
      const double r0 = mufu_rcp(den);
      const double er = fma(-den, r0, 1.0);
      rden = copysign(fma(r0, fma(er, er, er), r0), c0 >= 0.0 ? 1.0 : -1.0);
      const double sq = v * y;
      const double sqc = fma(0.5 * y, fma(-sq, sq, v), sq);
      beta = c0 >= 0.0 ? -sqc : sqc;
      t = fma(ac, y, 1.0);
    } else {
      beta = sqrt(c0 * c0 + s);
      if (c0 >= 0.0) beta = -beta;
      rden = 1.0 / (c0 - beta);  // essential = tail / (c0 - beta)
      t = (beta - c0) / beta;
    }
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = lane + 32 * r;
      if (i > j && i < m) x[i] *= rden;
    }
  }
  __syncwarp();
  if (lane == 0) {
    x[j] = beta;
    tau[j] = t;
  }
}

// A (m x c, ld lda) in smem. On exit: R on/above the diagonal, essential
// Householder parts below, tau[0..min(m,c)). Warp w owns columns j = w mod
// NW. ONE block barrier per column: after it every warp applies H_j to its
// columns, and the owner of column j+1 — which updates that column first and
// accumulates its next tail norm on the way — builds H_{j+1} right away,
// overlapping the other warps' updates.
template <int NT, int RPL, int CMAX = 64, bool FAST = false>
__device__ void cta_house_qr_t(double* A, int lda, int m, int c, double* tau, double* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  const int size = m < c ? m : c;
  (void)red;
  if (size > 0 && warp == 0) {
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = lane + 32 * r;
      if (i >= 1 && i < m) s += A[i] * A[i];
    }
    s = warp_sum(s);
    house_make<RPL, FAST>(A, 0, m, s, tau);
  }
  __syncthreads();
  for (int j = 0; j < size; ++j) {
    double* x = A + j * lda;
    // tau = 0 (identity reflector, incl. the rows()==1 case) leaves every
    // column unchanged through the same arithmetic, so the code below has no
    // data-dependent branches around its shuffles (those would be compiled
    // as divergence-safe "collective" sequences, several times slower).
    const double t = tau[j];
    // this warp's columns right of j: k0, k0 + NW, ... — processed together
    // (one read of the reflector, interleaved butterflies)
    const int k0 = j + 1 + ((warp - (j + 1) % NW + NW) % NW);
    constexpr int CPW = (CMAX + NW - 1) / NW;  // c <= CMAX
    double xr[RPL];
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = lane + 32 * r;
      xr[r] = (i > j && i < m) ? x[i] : 0.0;
    }
    double w[CPW], aj[CPW];
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
      const int k = k0 + q * NW;
      const double* a = A + (k < c ? k : c - 1) * lda;  // always a valid column
      w[q] = 0.0;
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int i = lane + 32 * r;
        if (i < m) w[q] = fma(xr[r], a[i], w[q]);
      }
      aj[q] = a[j];  // head, read before anyone writes it
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int q = 0; q < CPW; ++q) w[q] += __shfl_xor_sync(0xffffffffu, w[q], o);
    double s = 0.0;  // next tail norm of column j+1 (owner warp, slot q = 0)
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
      const int k = k0 + q * NW;
      if (k < c) {
        double* a = A + k * lda;
        const double wq = w[q] + aj[q];
        if (lane == 0) a[j] = aj[q] - t * wq;
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const int i = lane + 32 * r;
          if (i > j && i < m) {
            const double v = a[i] - t * xr[r] * wq;
            a[i] = v;
            if (q == 0 && i > j + 1) s = fma(v, v, s);
          }
        }
      }
    }
    s = warp_sum(s);
    if (k0 == j + 1 && k0 < size) house_make<RPL, FAST>(A + k0 * lda, k0, m, s, tau);
    __syncthreads();
  }
}

template <int NT, int CMAX = 64>
__device__ void cta_house_qr(double* A, int lda, int m, int c, double* tau, double* red) {
  if constexpr (CMAX <= 32) {  // c <= 32 (callers enforce): half the per-warp column slots, fast sqrt / rcp
    if (m <= 64) cta_house_qr_t<NT, 2, 32, true>(A, lda, m, c, tau, red);
    else cta_house_qr_t<NT, 8, 32, true>(A, lda, m, c, tau, red);  // m <= 256
  } else {
    if (m <= 64) cta_house_qr_t<NT, 2>(A, lda, m, c, tau, red);
    else if (m <= 256) cta_house_qr_t<NT, 8>(A, lda, m, c, tau, red);
    else cta_house_qr_t<NT, 16>(A, lda, m, c, tau, red);  // m <= 512 (callers enforce)
  }
}

// Explicit thin Q = H_0 H_1 ... H_{c-1} [I_c; 0] (m x c) from the reflectors
// stored below the diagonal of V (ld ldv) and tau, written to Q (ld ldq, smem
// or global, must not alias V). Column j = H_0 ... H_j e_j is built in the
// registers of the warp that owns it (RPL rows per lane): no block barriers.
template <int NT, int RPL, int CMAX = 64>
__device__ void cta_form_q_regs(const double* V, int ldv, int m, int c, const double* tau, double* Q, int ldq,
                                bool inplace = false, const double* colsign = nullptr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = NT / 32;
  constexpr int CPW = (CMAX + NW - 1) / NW;  // c <= CMAX
  // all columns of this warp travel together: one read of each reflector,
  // interleaved butterflies
  double y[CPW][RPL];
#pragma unroll
  for (int q = 0; q < CPW; ++q) {
    const int j = warp + q * NW;
#pragma unroll
    for (int r = 0; r < RPL; ++r) y[q][r] = (j < c && lane + 32 * r == j) ? 1.0 : 0.0;
  }
  // uniform trip count and no data-dependent skips around the shuffles
  // (tau = 0 is an exact no-op through the arithmetic)
  for (int k = c - 1; k >= 0; --k) {
    const double t = tau[k];
    const double* v = V + k * ldv;
    double vr[RPL];
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = lane + 32 * r;
      vr[r] = (i > k && i < m) ? v[i] : (i == k ? 1.0 : 0.0);  // implicit unit head
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
    for (int q = 0; q < CPW; ++q) {
      const int j = warp + q * NW;
      if (j >= k && j < c) {  // H_k leaves e_j (j < k) untouched
#pragma unroll
        for (int r = 0; r < RPL; ++r) y[q][r] -= t * vr[r] * w[q];
      }
    }
  }
  // in place (Q aliases V): every warp has read its last reflector before
  // any column of Q overwrites them
  if (inplace) __syncthreads();
#pragma unroll
  for (int q = 0; q < CPW; ++q) {
    const int j = warp + q * NW;
    if (j < c) {
      const double f = colsign ? colsign[j] : 1.0;
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int i = lane + 32 * r;
        if (i < m) Q[i + (int64_t)j * ldq] = f * y[q][r];
      }
    }
  }
}

template <int NT>
__device__ void cta_form_q(const double* V, int ldv, int m, int c, const double* tau, double* Q, int ldq) {
  if (m <= 64) cta_form_q_regs<NT, 2>(V, ldv, m, c, tau, Q, ldq);
  else if (m <= 256) cta_form_q_regs<NT, 8>(V, ldv, m, c, tau, Q, ldq);
  else cta_form_q_regs<NT, 8>(V, ldv, m, c, tau, Q, ldq);  // m <= 256 (callers enforce)
}

// thin_qr (linalg.cpp:67-79): A (m x c, m >= c, m <= 1024) in smem is
// factorised in place; Q (m x c, ld ldq, smem or global, distinct from A)
// and R (c x c, ld ldr, smem) are sign-fixed so R(i,i) >= 0.
template <int NT>
__device__ void cta_thin_qr(double* A, int lda, int m, int c, double* Q, int ldq, double* R, int ldr, double* tau,
                            double* red) {
  cta_house_qr<NT>(A, lda, m, c, tau, red);
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

// thin_qr's Q (sign-fixed so R(i,i) >= 0) written over A itself (m <= 256):
// Householder QR in place, the column signs of R read off its diagonal into
// `red`, then Q built in registers and stored over the reflectors. R is not
// kept (the selection path only needs the basis). red >= c + 8 doubles.
template <int NT, int CMAX = 64>
__device__ void cta_thin_qr_inplace(double* A, int lda, int m, int c, double* tau, double* red) {
  if (CMAX <= 32 || c <= 32) cta_house_qr<NT, 32>(A, lda, m, c, tau, red);
  else if constexpr (CMAX > 32) cta_house_qr<NT>(A, lda, m, c, tau, red);
  __syncthreads();
  SLRA_PROF(2);
  for (int j = threadIdx.x; j < c; j += NT) red[j] = A[j + j * lda] < 0.0 ? -1.0 : 1.0;
  __syncthreads();
  if (CMAX <= 32 || c <= 32) {  // half the register columns (the C-A kernel's two-CTA budget)
    if (m <= 64) cta_form_q_regs<NT, 2, 32>(A, lda, m, c, tau, A, lda, true, red);
    else cta_form_q_regs<NT, 8, 32>(A, lda, m, c, tau, A, lda, true, red);
  } else if constexpr (CMAX > 32) {
    if (m <= 64) cta_form_q_regs<NT, 2>(A, lda, m, c, tau, A, lda, true, red);
    else cta_form_q_regs<NT, 8>(A, lda, m, c, tau, A, lda, true, red);  // m <= 256 (callers enforce)
  }
  __syncthreads();
}

// ---------------------------------------------------------------- pivoted init
// Column-pivoted Householder QR of X = Q^T (r x m) — i.e. pivoting over the
// ROWS of Q (m x r, ld ldq) — reporting only the first r pivots, exactly the
// maxvol initialisation of cur.cpp:95-98. W (m x r, ld ldw) is scratch.
struct ColPivScratch {
  double* W;
  int ldw;
  int* p2r;     // position -> row
  double* nu;   // updated norms (by position)
  double* nd;   // direct norms (by position)
  double* v;    // Householder essential vector (r)
  double* tau;  // [0] = tau
  double* rv;   // >= 33
  int64_t* ri;  // >= 33
};

template <int NT>
__device__ void cta_colpiv_init(const double* Q, int ldq, int m, int r, const ColPivScratch& s, int* I_out) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double sqrt_eps = 1.4901161193847656e-08;  // sqrt(DBL_EPSILON)
  for (int i = tid; i < m; i += NT) {
    double acc = 0.0;
    for (int j = 0; j < r; ++j) {
      const double x = Q[i + j * ldq];
      s.W[i + j * s.ldw] = x;
      acc += x * x;
    }
    s.nu[i] = s.nd[i] = sqrt(acc);
    s.p2r[i] = i;
  }
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    ArgMax a{-1.0, INT64_MAX};
    for (int p = k + tid; p < m; p += NT) a = argmax_merge(a, ArgMax{s.nu[p], p});
    a = block_argmax<NT>(a, s.rv, s.ri);
    const int big = static_cast<int>(a.i);
    if (tid == 0 && big != k) {
      int ti = s.p2r[k]; s.p2r[k] = s.p2r[big]; s.p2r[big] = ti;
      double tv = s.nu[k]; s.nu[k] = s.nu[big]; s.nu[big] = tv;
      tv = s.nd[k]; s.nd[k] = s.nd[big]; s.nd[big] = tv;
    }
    __syncthreads();
    const int row = s.p2r[k];
    if (warp == 0) {
      double tail = 0.0;
      for (int j = k + 1 + lane; j < r; j += 32) {
        const double x = s.W[row + j * s.ldw];
        tail += x * x;
      }
      tail = warp_sum(tail);
      const double c0 = s.W[row + k * s.ldw];
      double t, beta;
      if (tail <= DBL_MIN) {
        t = 0.0;
        beta = c0;
        for (int j = k + 1 + lane; j < r; j += 32) s.v[j] = 0.0;
      } else {
        beta = sqrt(c0 * c0 + tail);
        if (c0 >= 0.0) beta = -beta;
        const double den = c0 - beta;
        for (int j = k + 1 + lane; j < r; j += 32) s.v[j] = s.W[row + j * s.ldw] / den;
        t = (beta - c0) / beta;
      }
      __syncwarp();
      if (lane == 0) {
        s.tau[0] = t;
        s.W[row + k * s.ldw] = beta;
        I_out[k] = row;
      }
    }
    __syncthreads();
    const double t = s.tau[0];
    for (int p = k + 1 + tid; p < m; p += NT) {
      const int i = s.p2r[p];
      if (r - k > 1 && t != 0.0) {
        double w = 0.0;
        for (int j = k + 1; j < r; ++j) w += s.v[j] * s.W[i + j * s.ldw];
        w += s.W[i + k * s.ldw];
        s.W[i + k * s.ldw] -= t * w;
        for (int j = k + 1; j < r; ++j) s.W[i + j * s.ldw] -= t * s.v[j] * w;
      }
      double nu = s.nu[p];
      if (nu != 0.0) {
        double temp = fabs(s.W[i + k * s.ldw]) / nu;
        temp = (1.0 + temp) * (1.0 - temp);
        temp = temp < 0.0 ? 0.0 : temp;
        const double ratio = nu / s.nd[p];
        const double temp2 = temp * ratio * ratio;
        if (temp2 <= sqrt_eps) {
          double acc = 0.0;
          for (int j = k + 1; j < r; ++j) acc += s.W[i + j * s.ldw] * s.W[i + j * s.ldw];
          s.nd[p] = sqrt(acc);
          s.nu[p] = s.nd[p];
        } else {
          s.nu[p] = nu * sqrt(temp);
        }
      }
    }
    __syncthreads();
  }
}

// The same pivot order with the working copy of Q^T in REGISTERS: thread t
// owns row t of Q (m <= NT, r <= RMAX), so no m x r shared scratch is needed
// (the C-A kernel then fits two CTAs per SM). Rows keep their thread while
// positions are swapped through p2r / r2p; each row's update is the same
// arithmetic, in the same order, as cta_colpiv_init.
template <int NT, int RMAX>
__device__ void cta_colpiv_init_regs(const double* Q, int ldq, int m, int r, double* nu, double* nd, int* p2r,
                                     int* r2p, double* vbuf, double* tauv, double* rv, int64_t* ri, int* I_out,
                                     double* Wx = nullptr, double* Rsv = nullptr, int ldr = 0,
                                     double* pv = nullptr) {
  // Wx / Rsv / pv (optional): keep the factorisation for maxvol round 0.
  // The first r pivots are the rows I, so these reflectors are those of
  // ColPivQR(Q(I, :)^T) with the identity permutation (same columns, same
  // arithmetic in the same order as warp_colpiv_qr): Rsv (r x r, ld ldr)
  // gets R on and above the diagonal and the Householder vectors below it,
  // tauv[k] the k-th tau, pv[k] the k-th pivot norm, and Wx (= Q in place,
  // ld ldq) every row after the reflectors applied to it (all r for the
  // other rows, those before its own step for a pivot row).
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double sqrt_eps = 1.4901161193847656e-08;  // sqrt(DBL_EPSILON)
  double x[RMAX];
  const bool own = tid < m;
  {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < RMAX; ++j) {
      x[j] = (own && j < r) ? Q[tid + j * ldq] : 0.0;
      acc += x[j] * x[j];
    }
    if (own) {
      nu[tid] = nd[tid] = sqrt(acc);
      p2r[tid] = tid;
      r2p[tid] = tid;
    }
  }
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    ArgMax a{-1.0, INT64_MAX};
    for (int p = k + tid; p < m; p += NT) a = argmax_merge(a, ArgMax{nu[p], p});
    a = block_argmax<NT>(a, rv, ri);
    const int big = static_cast<int>(a.i);
    if (pv && tid == 0) pv[k] = a.v;
    if (tid == 0 && big != k) {
      const int rk = p2r[k], rb = p2r[big];
      p2r[k] = rb;
      p2r[big] = rk;
      r2p[rb] = k;
      r2p[rk] = big;
      double tv = nu[k]; nu[k] = nu[big]; nu[big] = tv;
      tv = nd[k]; nd[k] = nd[big]; nd[big] = tv;
    }
    __syncthreads();
    const int row = p2r[k];
    if (tid == row) {
#pragma unroll
      for (int j = 0; j < RMAX; ++j)
        if (j >= k && j < r) vbuf[j] = x[j];
    }
    __syncthreads();
    if (warp == 0) {
      double tail = 0.0;
      for (int j = k + 1 + lane; j < r; j += 32) tail += vbuf[j] * vbuf[j];
      tail = warp_sum(tail);
      const double c0 = vbuf[k];
      double t;
      __syncwarp();
      double beta = c0;
      if (tail <= DBL_MIN) {
        t = 0.0;
        for (int j = k + 1 + lane; j < r; j += 32) vbuf[j] = 0.0;
      } else {
        beta = sqrt(c0 * c0 + tail);
        if (c0 >= 0.0) beta = -beta;
        const double den = c0 - beta;
        for (int j = k + 1 + lane; j < r; j += 32) vbuf[j] = vbuf[j] / den;
        t = (beta - c0) / beta;
      }
      __syncwarp();
      if (Rsv)
        for (int j = k + 1 + lane; j < r; j += 32) Rsv[j + k * ldr] = vbuf[j];
      if (lane == 0) {
        tauv[k] = t;
        I_out[k] = row;
        if (Rsv) Rsv[k + k * ldr] = beta;
      }
    }
    __syncthreads();
    const double t = tauv[k];
    const int p = own ? r2p[tid] : -1;
    if (p > k) {
      if (r - k > 1 && t != 0.0) {
        double w = 0.0;
#pragma unroll
        for (int j = 0; j < RMAX; ++j)
          if (j > k && j < r) w += vbuf[j] * x[j];
#pragma unroll
        for (int j = 0; j < RMAX; ++j)
          if (j == k) w += x[j];
#pragma unroll
        for (int j = 0; j < RMAX; ++j) {
          if (j == k) x[j] -= t * w;
          if (j > k && j < r) x[j] -= t * vbuf[j] * w;
        }
      }
      const double nuv = nu[p];
      if (nuv != 0.0) {
        double xk = 0.0;
#pragma unroll
        for (int j = 0; j < RMAX; ++j)
          if (j == k) xk = x[j];
        double temp = fabs(xk) / nuv;
        temp = (1.0 + temp) * (1.0 - temp);
        temp = temp < 0.0 ? 0.0 : temp;
        const double ratio = nuv / nd[p];
        const double temp2 = temp * ratio * ratio;
        if (temp2 <= sqrt_eps) {
          double acc = 0.0;
#pragma unroll
          for (int j = 0; j < RMAX; ++j)
            if (j > k && j < r) acc += x[j] * x[j];
          nd[p] = sqrt(acc);
          nu[p] = nd[p];
        } else {
          nu[p] = nuv * sqrt(temp);
        }
      }
    }
    __syncthreads();
  }
  if (Wx && own) {
    const int p = r2p[tid];
#pragma unroll
    for (int j = 0; j < RMAX; ++j) {
      if (j < r) Wx[tid + j * ldq] = x[j];
      if (p < r && j < p) Rsv[j + p * ldr] = x[j];  // R(0:p, p): final entries of pivot row p
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------- small ColPivQR (one warp)
// Eigen ColPivHouseholderQR on a small n x n matrix G (ld ldg, in smem), run
// by the calling warp. Outputs: perm (n), tau (n), nonzero pivots and rank
// with the prescribed threshold. `nu`, `nd` scratch (n).
struct SmallColPiv {
  int nonzero_pivots;
  int rank;
};

template <bool SPLIT = false>
__device__ inline SmallColPiv warp_colpiv_qr(double* G, int ldg, int n, double threshold, int* perm, double* tau,
                                      double* nu, double* nd) {
  const int lane = threadIdx.x & 31;
  const double eps = kEps;
  const double sqrt_eps = 1.4901161193847656e-08;
  double maxnorm = 0.0;
  for (int j = lane; j < n; j += 32) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc += G[i + j * ldg] * G[i + j * ldg];
    nu[j] = nd[j] = sqrt(acc);
    perm[j] = j;
    maxnorm = fmax(maxnorm, nu[j]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) maxnorm = fmax(maxnorm, __shfl_xor_sync(0xffffffffu, maxnorm, o));
  __syncwarp();
  const double thr_helper = (maxnorm * eps) * (maxnorm * eps) / (double)n;
  int nonzero = n;
  double maxpivot = 0.0;
  for (int k = 0; k < n; ++k) {
    ArgMax a{-1.0, INT64_MAX};
    for (int j = k + lane; j < n; j += 32) a = argmax_merge(a, ArgMax{nu[j], j});
    a = warp_argmax(a);
    const int big = (int)a.i;
    if (nonzero == n && a.v * a.v < thr_helper * (double)(n - k)) nonzero = k;
    // transposition k <-> big (columns, norms, permutation: Eigen applies
    // the transpositions to an identity permutation in order)
    if (big != k) {
      for (int i = lane; i < n; i += 32) {
        const double t0 = G[i + k * ldg];
        G[i + k * ldg] = G[i + big * ldg];
        G[i + big * ldg] = t0;
      }
      if (lane == 0) {
        double t1 = nu[k]; nu[k] = nu[big]; nu[big] = t1;
        t1 = nd[k]; nd[k] = nd[big]; nd[big] = t1;
        const int p = perm[k]; perm[k] = perm[big]; perm[big] = p;
      }
    }
    __syncwarp();
    double* x = G + k * ldg;
    double tail = 0.0;
    for (int i = k + 1 + lane; i < n; i += 32) tail += x[i] * x[i];
    tail = warp_sum(tail);
    const double c0 = x[k];
    double t, beta;
    if (tail <= DBL_MIN) {
      t = 0.0;
      beta = c0;
      for (int i = k + 1 + lane; i < n; i += 32) x[i] = 0.0;
    } else {
      beta = sqrt(c0 * c0 + tail);
      if (c0 >= 0.0) beta = -beta;
      const double den = c0 - beta;
      for (int i = k + 1 + lane; i < n; i += 32) x[i] = x[i] / den;
      t = (beta - c0) / beta;
    }
    __syncwarp();
    if (lane == 0) {
      x[k] = beta;
      tau[k] = t;
    }
    if (fabs(beta) > maxpivot) maxpivot = fabs(beta);
    __syncwarp();
    if (n - k > 1 && t != 0.0) {
      for (int j = k + 1 + lane; j < n; j += 32) {
        double* a2 = G + j * ldg;
        double w = 0.0;
        if (SPLIT) {  // four independent chains (a preconditioner: order-insensitive)
          double w1 = 0.0, w2 = 0.0, w3 = 0.0;
          int i = k + 1;
          for (; i + 3 < n; i += 4) {
            w = fma(x[i], a2[i], w);
            w1 = fma(x[i + 1], a2[i + 1], w1);
            w2 = fma(x[i + 2], a2[i + 2], w2);
            w3 = fma(x[i + 3], a2[i + 3], w3);
          }
          for (; i < n; ++i) w = fma(x[i], a2[i], w);
          w = (w + w1) + (w2 + w3);
        } else {
          for (int i = k + 1; i < n; ++i) w += x[i] * a2[i];
        }
        w += a2[k];
        a2[k] -= t * w;
        for (int i = k + 1; i < n; ++i) a2[i] -= t * x[i] * w;
      }
    }
    __syncwarp();
    for (int j = k + 1 + lane; j < n; j += 32) {
      if (nu[j] != 0.0) {
        double temp = fabs(G[k + j * ldg]) / nu[j];
        temp = (1.0 + temp) * (1.0 - temp);
        temp = temp < 0.0 ? 0.0 : temp;
        const double ratio = nu[j] / nd[j];
        const double temp2 = temp * ratio * ratio;
        if (temp2 <= sqrt_eps) {
          double acc = 0.0;
          for (int i = k + 1; i < n; ++i) acc += G[i + j * ldg] * G[i + j * ldg];
          nd[j] = sqrt(acc);
          nu[j] = nd[j];
        } else {
          nu[j] *= sqrt(temp);
        }
      }
    }
    __syncwarp();
  }
  // rank() with the prescribed threshold
  const double pre = fabs(maxpivot) * threshold;
  int rank = 0;
  for (int i = 0; i < nonzero; ++i) rank += (fabs(G[i + i * ldg]) > pre) ? 1 : 0;
  return SmallColPiv{nonzero, rank};
}

// ---------------------------------------------------------------- maxvol swap loop
// A (m x r, ld lda) in smem, I (r current rows, smem, updated in place).
// Returns SLRA_OK or SLRA_ERR_SELECTION_FAILURE. Scratch: W (m x r), Gt
// (r x r), perm/tau/nu/nd (r each), rv/ri.
template <int NT>
__device__ int cta_maxvol_swaps(const double* A, int lda, int m, int r, double h, int max_swaps, int* I,
                                double* W, int ldw, double* Gt, int ldg, int* perm, double* tau, double* nu,
                                double* nd, double* rv, int64_t* ri, int* shared_flag, double* vol_out = nullptr,
                                const int* pre_r2p = nullptr, const double* pre_pv = nullptr) {
  const int tid = threadIdx.x, warp = tid >> 5;
  // swap round 0 exactly as the reference: ColPivQR(G^T) and its solve for
  // every row. G^T(c, t) = A(I[t], c). Prefactored (pre_r2p): the pivoted-QR
  // initialisation already holds that factorisation (cta_colpiv_init_regs
  // with Wx = W = A, Rsv = Gt): identity permutation, and each row continues
  // from the reflectors already applied to it.
  if (pre_r2p) {
    if (tid == 0) {
      // warp_colpiv_qr's nonzero-pivot and rank rules on the saved pivot norms
      const double thr_helper = (pre_pv[0] * kEps) * (pre_pv[0] * kEps) / (double)r;
      int nonzero = r;
      double maxpivot = 0.0;
      for (int k = 0; k < r; ++k) {
        if (nonzero == r && pre_pv[k] * pre_pv[k] < thr_helper * (double)(r - k)) nonzero = k;
        maxpivot = fmax(maxpivot, fabs(Gt[k + k * ldg]));
      }
      int rank = 0;
      for (int i = 0; i < nonzero; ++i) rank += (fabs(Gt[i + i * ldg]) > fabs(maxpivot) * 1e-12) ? 1 : 0;
      shared_flag[0] = rank < r ? 1 : 0;
    }
    for (int t = tid; t < r; t += NT) perm[t] = t;
  } else {
    for (int e = tid; e < r * r; e += NT) {
      const int cc = e % r, t = e / r;
      Gt[cc + t * ldg] = A[I[t] + cc * lda];
    }
    __syncthreads();
    if (warp == 0) {
      SmallColPiv q = warp_colpiv_qr(Gt, ldg, r, 1e-12, perm, tau, nu, nd);
      if ((tid & 31) == 0) shared_flag[0] = q.rank < r ? 1 : 0;  // rank == r implies r nonzero pivots
    }
  }
  __syncthreads();
  if (shared_flag[0]) return SLRA_ERR_SELECTION_FAILURE;
  // |det A(I, :)| = prod |R_ii| of the round-0 QR (Q orthogonal), then times
  // |B(piv, j)| per swap (the maxvol volume update): thread 0 keeps it, so the
  // caller may overwrite A with B (W == A) and still get the volume proxy
  double vol = 0.0;
  if (vol_out && tid == 0) {
    vol = 1.0;
    for (int i = 0; i < r; ++i) vol *= fabs(Gt[i + i * ldg]);
  }
  // W(i, t) holds B(i, perm[t]) (storage order of the solve)
  for (int i = tid; i < m; i += NT) {
    double* c = W + i;  // row i of W as a strided vector (stride ldw)
    int k0 = 0;
    if (pre_r2p) {
      k0 = pre_r2p[i] < r ? pre_r2p[i] : r;  // reflectors 0..k0-1 already applied (in place)
    } else {
      for (int j = 0; j < r; ++j) c[j * ldw] = A[i + j * lda];
    }
    for (int k = k0; k < r; ++k) {
      const double t = tau[k];
      if (r - k == 1) {
        c[k * ldw] *= (1.0 - t);
      } else if (t != 0.0) {
        double w = 0.0;
        for (int j = k + 1; j < r; ++j) w += Gt[j + k * ldg] * c[j * ldw];
        w += c[k * ldw];
        c[k * ldw] -= t * w;
        for (int j = k + 1; j < r; ++j) c[j * ldw] -= t * Gt[j + k * ldg] * w;
      }
    }
    for (int t2 = r - 1; t2 >= 0; --t2) {
      double sacc = c[t2 * ldw];
      for (int u = t2 + 1; u < r; ++u) sacc -= Gt[t2 + u * ldg] * c[u * ldw];
      c[t2 * ldw] = sacc / Gt[t2 + t2 * ldg];
    }
  }
  int* iperm = reinterpret_cast<int*>(nd);  // B column -> storage column
  for (int t = tid; t < r; t += NT) iperm[perm[t]] = t;
  __syncthreads();
  // swap rounds: argmax |B| (column-major first maximum), then the rank-1
  // update B <- B - B(:, j) (B(i, :) - e_j) / B(i, j) for row i placed at
  // slot j: the same B = A G^-1 the reference re-solves each round, at
  // O(m r) instead of O(m r^2 + r^3) per round.
  double* g = tau;  // snapshot of the pivot row (r)
  for (int swap = 0; swap <= max_swaps; ++swap) {
    ArgMax best{-1.0, INT64_MAX};
    for (int i = tid; i < m; i += NT)
      for (int t2 = 0; t2 < r; ++t2)
        best = argmax_merge(best, ArgMax{fabs(W[i + t2 * ldw]), (int64_t)perm[t2] * m + i});
    best = block_argmax<NT>(best, rv, ri);
    if (best.v <= h || swap == max_swaps) {
      if (vol_out && tid == 0) *vol_out = vol;
      return SLRA_OK;
    }
    const int j = (int)(best.i / m), piv = (int)(best.i % m);
    const int ts = iperm[j];
    // the pivot is read by every thread BEFORE the barrier: after it, the
    // thread owning row piv overwrites W(piv, :)
    const double p = W[piv + ts * ldw];
    for (int t2 = tid; t2 < r; t2 += NT) g[t2] = W[piv + t2 * ldw] - (t2 == ts ? 1.0 : 0.0);
    __syncthreads();
    if (tid == 0) {
      I[j] = piv;
      vol *= fabs(p);
    }
    for (int i = tid; i < m; i += NT) {
      const double f = W[i + ts * ldw] / p;
      for (int t2 = 0; t2 < r; ++t2) W[i + t2 * ldw] -= f * g[t2];
    }
    __syncthreads();
  }
  return SLRA_OK;
}

// |det(M)| of an n x n smem matrix (destroyed) by partial-pivot LU, one warp.
__device__ inline double warp_abs_det(double* M, int ld, int n) {
  const int lane = threadIdx.x & 31;
  double det = 1.0;
  for (int k = 0; k < n; ++k) {
    ArgMax a{-1.0, INT64_MAX};
    for (int i = k + lane; i < n; i += 32) a = argmax_merge(a, ArgMax{fabs(M[i + k * ld]), i});
    a = warp_argmax(a);
    const int p = (int)a.i;
    if (a.v == 0.0) return 0.0;
    if (p != k)
      for (int j = lane; j < n; j += 32) {
        const double t = M[k + j * ld];
        M[k + j * ld] = M[p + j * ld];
        M[p + j * ld] = t;
      }
    __syncwarp();
    const double piv = M[k + k * ld];
    det *= piv;
    for (int i = k + 1 + lane; i < n; i += 32) {
      const double f = M[i + k * ld] / piv;
      for (int j = k + 1; j < n; ++j) M[i + j * ld] -= f * M[k + j * ld];
    }
    __syncwarp();
  }
  return fabs(det);
}

// ---------------------------------------------------------------- Jacobi SVD
// One-sided Jacobi on the columns of W (p x n, ld ldw, p >= n, n <= 64),
// accumulating V (n x n, ld ldv). Parallel round-robin ordering; each warp
// owns disjoint column pairs per round. On exit W's columns are
// U_j sigma_j (unsorted).
// Rows per lane: p <= 32*RPL (W), n <= 64 (V, two rows per lane).
// `deflate` > 0 skips pairs whose columns both have norm below deflate times
// the largest column norm of the sweep start (range finder only: those
// directions fall under the rank cut and are never used individually).
template <int NT, int RPL>
__device__ void cta_jacobi_t(double* W, int ldw, int p, int n, double* V, int ldv, int* flag, double deflate) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  __shared__ unsigned short pair_tab[64 * 32];  // round-robin schedule: (a << 8) | b
  __shared__ double dmax2;
  for (int e = tid; e < n * n; e += NT) V[e % n + (e / n) * ldv] = (e % n == e / n) ? 1.0 : 0.0;
  const int ne = n + (n & 1);  // even number of players (dummy = n)
  for (int e = tid; e < (ne - 1) * (ne / 2); e += NT) {
    const int rd = e / (ne / 2), pi = e % (ne / 2);
    int a, b;
    if (pi == 0) {
      a = rd;
      b = ne - 1;
    } else {
      a = (rd + pi) % (ne - 1);
      b = (rd - pi + ne - 1) % (ne - 1);
    }
    if (a > b) { const int t = a; a = b; b = t; }
    pair_tab[e] = (unsigned short)((a << 8) | b);
  }
  // orthogonality threshold: dgesvj's sqrt(p)*eps sits below the rounding
  // floor of the rotated columns (measured ~p*eps here: the sweeps never
  // stop); 16*p*eps keeps sigma accurate to O(tol^2) relative and the
  // vectors to O(tol / gap)
  const double tol = 16.0 * (double)p * kEps;
  if (tid == 0) flag[0] = flag[1] = 0;
  __syncthreads();
  for (int sweep = 0; sweep < 40; ++sweep) {
    const int fl = sweep & 1;  // double-buffered "rotated" flag
    double thr2 = 0.0;
    if (deflate > 0.0) {
      if (warp == 0) {
        double mx = 0.0;
        for (int j = 0; j < n; ++j) {
          double s = 0.0;
#pragma unroll
          for (int r = 0; r < RPL; ++r) {
            const int i = lane + 32 * r;
            if (i < p) s = fma(W[i + j * ldw], W[i + j * ldw], s);
          }
          s = warp_sum(s);
          mx = fmax(mx, s);
        }
        if (lane == 0) dmax2 = mx;
      }
      __syncthreads();
      thr2 = deflate * deflate * dmax2;
    }
    const int npairs = ne / 2;
    const int iters = (npairs + NW - 1) / NW;  // uniform trip count for every warp
    for (int rd = 0; rd < ne - 1; ++rd) {
      for (int it = 0; it < iters; ++it) {
        const int pi = warp + it * NW;
        const int ab = pair_tab[rd * npairs + (pi < npairs ? pi : 0)];
        const bool valid = pi < npairs && (ab & 255) < n;
        const int a = ab >> 8, b = valid ? (ab & 255) : a;
        double* wp = W + a * ldw;
        double* wq = W + b * ldw;
        double x[RPL], y[RPL];
        double aa = 0.0, bb = 0.0, gg = 0.0;
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const int i = lane + 32 * r;
          x[r] = i < p ? wp[i] : 0.0;
          y[r] = i < p ? wq[i] : 0.0;
          aa = fma(x[r], x[r], aa);
          bb = fma(y[r], y[r], bb);
          gg = fma(x[r], y[r], gg);
        }
        // three interleaved butterflies, in uniform control flow (a branch
        // on shared data before them makes nvcc emit divergence-safe
        // collective shuffles, several times slower)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          aa += __shfl_xor_sync(0xffffffffu, aa, o);
          bb += __shfl_xor_sync(0xffffffffu, bb, o);
          gg += __shfl_xor_sync(0xffffffffu, gg, o);
        }
        // convergence test of LAPACK dgesvj: |<w_p, w_q>| <= sqrt(p) eps ||w_p|| ||w_q||
        // (a bare eps threshold never settles once the dot products are
        // evaluated in a different order than the rotation was computed)
        if (!valid || gg == 0.0 || fabs(gg) <= tol * sqrt(aa * bb)) continue;
        if (aa < thr2 && bb < thr2) continue;
        const double zeta = (bb - aa) * __drcp_rn(2.0 * gg);
        const double t = copysign(__drcp_rn(fabs(zeta) + sqrt(fma(zeta, zeta, 1.0))), zeta);
        const double cs = rsqrt(fma(t, t, 1.0));
        const double sn = cs * t;
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const int i = lane + 32 * r;
          if (i < p) {
            wp[i] = cs * x[r] - sn * y[r];
            wq[i] = sn * x[r] + cs * y[r];
          }
        }
        double* vp = V + a * ldv;
        double* vq = V + b * ldv;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int i = lane + 32 * r;
          if (i < n) {
            const double u = vp[i], v = vq[i];
            vp[i] = cs * u - sn * v;
            vq[i] = sn * u + cs * v;
          }
        }
        if (lane == 0) flag[fl] = 1;
      }
      __syncthreads();
    }
    const int rotated = flag[fl];
    if (tid == 0) flag[fl ^ 1] = 0;  // next sweep's flag; this one is read by all before the barrier below
    __syncthreads();
    if (!rotated) break;
  }
}

// The same sweeps for p, n <= 64 with an 8-lane group per column pair (4 pairs
// per warp): a pair's dot products reduce in 3 shuffle levels instead of 5
// and one warp-instruction advances 4 pairs, which cuts the instruction count
// per round ~4x — the round is instruction-throughput bound on FP64.
struct JacobiShared {
  unsigned short pair_tab[64 * 32];  // round-robin schedule: (a << 8) | b
  double dmax2;
  double cmax2[32];
};
__device__ inline JacobiShared& jacobi_shared() {
  __shared__ JacobiShared s;
  return s;
}

template <int NT, int RPG, bool EXACT, bool VEC2 = false>
__device__ void cta_jacobi_g8(double* W, int ldw, int p, int n, double* V, int ldv, int* flag, double deflate) {
  // RPG rows per lane (p <= 8 RPG, n <= p); EXACT: p == n == 8 RPG (no row predicates).
  // VEC2 (EXACT, RPG even, even ldw / ldv): a lane owns row pairs 2 sub + 16 rr
  // and moves them as 16-byte accesses — an 8-lane group then covers all 32
  // banks once per access whatever columns the other groups of the warp read
  // (with 8-byte accesses two groups of a half-warp collide on most column
  // pairs: the load and store phases of a round were shared-memory bound)
  static_assert(!VEC2 || (EXACT && RPG % 2 == 0), "VEC2 needs p == n == 8 RPG, RPG even");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = lane >> 3, sub = lane & 7;
  constexpr int NW = NT / 32;
  // one shared scratch for every instantiation (static __shared__ in a
  // template would be allocated once per instantiation)
  JacobiShared& js = jacobi_shared();
  unsigned short* pair_tab = js.pair_tab;
  double& dmax2 = js.dmax2;
  double* cmax2 = js.cmax2;
  for (int e = tid; e < n * n; e += NT) V[e % n + (e / n) * ldv] = (e % n == e / n) ? 1.0 : 0.0;
  const int ne = n + (n & 1);
  for (int e = tid; e < (ne - 1) * (ne / 2); e += NT) {
    const int rd = e / (ne / 2), pi = e % (ne / 2);
    int a, b;
    if (pi == 0) {
      a = rd;
      b = ne - 1;
    } else {
      a = (rd + pi) % (ne - 1);
      b = (rd - pi + ne - 1) % (ne - 1);
    }
    if (a > b) { const int t = a; a = b; b = t; }
    pair_tab[e] = (unsigned short)((a << 8) | b);
  }
  // orthogonality threshold: dgesvj's sqrt(p)*eps sits below the rounding
  // floor of the rotated columns (measured ~p*eps here: the sweeps never
  // stop); 16*p*eps keeps sigma accurate to O(tol^2) relative and the
  // vectors to O(tol / gap)
  const double tol = 16.0 * (double)p * kEps;
  const double tol2 = tol * tol;
  if (tid == 0) flag[0] = flag[1] = 0;
  __syncthreads();
  const int npairs = ne / 2;
  const int iters = (npairs + 4 * NW - 1) / (4 * NW);
#ifdef SLRA_JAC_PROF
  long long jp[6] = {0, 0, 0, 0, 0, 0};
  long long jt0 = 0, jt1 = 0;
  int jrounds = 0;
#define JAC_MARK(i) do { jt1 = clock64(); jp[i] += jt1 - jt0; jt0 = jt1; } while (0)
#else
#define JAC_MARK(i) do { } while (0)
#endif
  for (int sweep = 0; sweep < 40; ++sweep) {
    int rot_any = 0;  // this thread rotated a pair during the sweep
    double thr2 = 0.0;
    if (deflate > 0.0) {  // largest squared column norm, columns spread over the warps
      double mx = 0.0;
      for (int j = warp; j < n; j += NW) {
        double s = 0.0;
        for (int i = lane; i < p; i += 32) s = fma(W[i + j * ldw], W[i + j * ldw], s);
        mx = fmax(mx, warp_sum(s));
      }
      if (lane == 0) cmax2[warp] = mx;
      __syncthreads();
      if (tid == 0) {
        double m2 = 0.0;
        for (int w = 0; w < NW; ++w) m2 = fmax(m2, cmax2[w]);
        dmax2 = m2;
      }
      __syncthreads();
      thr2 = deflate * deflate * dmax2;
    }
    int ab_next = pair_tab[(warp * 4 + grp) < npairs ? (warp * 4 + grp) : 0];
    for (int rd = 0; rd < ne - 1; ++rd) {
#ifdef SLRA_JAC_PROF
      jt0 = clock64();
      ++jrounds;
#endif
      for (int it = 0; it < iters; ++it) {
        const int pi = (warp + it * NW) * 4 + grp;
        const int ab = (iters == 1) ? ab_next : pair_tab[rd * npairs + (pi < npairs ? pi : 0)];
        const bool valid = pi < npairs && (ab & 255) < n;
        const int a = ab >> 8, b = valid ? (ab & 255) : a;
        double* wp = W + a * ldw;
        double* wq = W + b * ldw;
        double* vp = V + a * ldv;
        double* vq = V + b * ldv;
        // W and V rows of both columns up front: every load is in flight
        // before the reduction and rotation chain starts
        double x[RPG], y[RPG], u[RPG], v[RPG];
        double aa = 0.0, bb = 0.0, gg = 0.0;
        if constexpr (VEC2) {
#pragma unroll
          for (int rr = 0; rr < RPG / 2; ++rr) {
            const int i = 2 * sub + 16 * rr;
            const double2 tx = *reinterpret_cast<const double2*>(wp + i);
            const double2 ty = *reinterpret_cast<const double2*>(wq + i);
            x[2 * rr] = tx.x, x[2 * rr + 1] = tx.y;
            y[2 * rr] = ty.x, y[2 * rr + 1] = ty.y;
          }  // (the V rows are loaded after the rotate / skip decision, behind the rotation's arithmetic)
        } else {
#pragma unroll
          for (int r = 0; r < RPG; ++r) {
            const int i = sub + 8 * r;
            x[r] = (EXACT || i < p) ? wp[i] : 0.0;
            y[r] = (EXACT || i < p) ? wq[i] : 0.0;
            u[r] = (EXACT || i < n) ? vp[i] : 0.0;
            v[r] = (EXACT || i < n) ? vq[i] : 0.0;
          }
        }
        {  // two accumulators per product: FP64 FMA latency is ~24 cycles on sm_100
          double a1 = 0.0, b1 = 0.0, g1 = 0.0;
#pragma unroll
          for (int r = 0; r + 1 < RPG; r += 2) {
            aa = fma(x[r], x[r], aa);
            bb = fma(y[r], y[r], bb);
            gg = fma(x[r], y[r], gg);
            a1 = fma(x[r + 1], x[r + 1], a1);
            b1 = fma(y[r + 1], y[r + 1], b1);
            g1 = fma(x[r + 1], y[r + 1], g1);
          }
          if (RPG & 1) {  // odd rows per lane: the last one (no read past x/y)
            aa = fma(x[RPG - 1], x[RPG - 1], aa);
            bb = fma(y[RPG - 1], y[RPG - 1], bb);
            gg = fma(x[RPG - 1], y[RPG - 1], gg);
          }
          aa += a1;
          bb += b1;
          gg += g1;
        }
        JAC_MARK(0);  // loads + partial dots
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {  // within the 8-lane group
          aa += __shfl_xor_sync(0xffffffffu, aa, o);
          bb += __shfl_xor_sync(0xffffffffu, bb, o);
          gg += __shfl_xor_sync(0xffffffffu, gg, o);
        }
        JAC_MARK(1);  // shuffle reduction
        // the next round's pair, read before this round's barrier
        if (iters == 1 && rd + 1 < ne - 1) ab_next = pair_tab[(rd + 1) * npairs + (pi < npairs ? pi : 0)];
        // |g| <= tol sqrt(a b), squared (no sqrt on the chain)
        if (!valid || gg == 0.0 || gg * gg <= tol2 * (aa * bb)) continue;
        if (aa < thr2 && bb < thr2) continue;
        // t = sign(z) / (|z| + sqrt(1 + z^2)), z = (b - a) / (2g), from the
        // hardware rsqrt / rcp seeds; c refined to full precision
        // (common.cuh: jacobi_rotation). This chain is most of a round.
        if constexpr (VEC2) {
#pragma unroll
          for (int rr = 0; rr < RPG / 2; ++rr) {
            const int i = 2 * sub + 16 * rr;
            const double2 tu = *reinterpret_cast<const double2*>(vp + i);
            const double2 tv = *reinterpret_cast<const double2*>(vq + i);
            u[2 * rr] = tu.x, u[2 * rr + 1] = tu.y;
            v[2 * rr] = tv.x, v[2 * rr + 1] = tv.y;
          }
        }
        double cs, sn;
        jacobi_rotation(aa, bb, gg, cs, sn);
#ifdef SLRA_JAC_PROF
        jp[5] += (long long)(cs != 2.0);  // keeps the rotation before the mark
#endif
        JAC_MARK(2);  // rotation
        if constexpr (VEC2) {
#pragma unroll
          for (int rr = 0; rr < RPG / 2; ++rr) {
            const int i = 2 * sub + 16 * rr, r = 2 * rr;
            *reinterpret_cast<double2*>(wp + i) = make_double2(cs * x[r] - sn * y[r], cs * x[r + 1] - sn * y[r + 1]);
            *reinterpret_cast<double2*>(wq + i) = make_double2(sn * x[r] + cs * y[r], sn * x[r + 1] + cs * y[r + 1]);
            *reinterpret_cast<double2*>(vp + i) = make_double2(cs * u[r] - sn * v[r], cs * u[r + 1] - sn * v[r + 1]);
            *reinterpret_cast<double2*>(vq + i) = make_double2(sn * u[r] + cs * v[r], sn * u[r + 1] + cs * v[r + 1]);
          }
        } else {
#pragma unroll
          for (int r = 0; r < RPG; ++r) {
            const int i = sub + 8 * r;
            if (EXACT || i < p) {
              wp[i] = cs * x[r] - sn * y[r];
              wq[i] = sn * x[r] + cs * y[r];
            }
            if (EXACT || i < n) {
              vp[i] = cs * u[r] - sn * v[r];
              vq[i] = sn * u[r] + cs * v[r];
            }
          }
        }
        rot_any = 1;
        JAC_MARK(3);  // apply + stores
      }
#ifdef SLRA_JAC_PROF
      jt0 = clock64();
#endif
      __syncthreads();
      JAC_MARK(4);  // barrier
    }
    if (tid == 0) flag[2] = sweep + 1;  // sweeps used (diagnostics)
    if (!__syncthreads_or(rot_any)) break;
  }
#ifdef SLRA_JAC_PROF
  if (tid == 0 && blockIdx.x == 0)
    printf("jacobi %dx%d sweeps %d rounds %d | per round: loads+dots %lld shuffles %lld rotation %lld apply %lld barrier %lld (rotated %lld)\n",
           p, n, flag[2], jrounds, jp[0] / jrounds, jp[1] / jrounds, jp[2] / jrounds, jp[3] / jrounds, jp[4] / jrounds,
           jp[5]);
#endif
#undef JAC_MARK
}

// PMAX < 256: only the rows-per-lane variants up to PMAX / 8 are instantiated
// (callers with a register budget, p <= PMAX guaranteed).
template <int NT, int PMAX = 256, bool VEC = false>
__device__ void cta_jacobi(double* W, int ldw, int p, int n, double* V, int ldv, int* flag, double deflate = 0.0) {
  if (p <= 64) {
    const int rpg = (p + 7) / 8;
    const bool exact = p == 8 * rpg && n == p;
    if constexpr (VEC) {  // 16-byte row pairs (even leading dimensions, 16-byte aligned W and V)
      if (exact && ((ldw | ldv) & 1) == 0) {
        if (rpg == 2) return cta_jacobi_g8<NT, 2, true, true>(W, ldw, p, n, V, ldv, flag, deflate);
        if (rpg == 4) return cta_jacobi_g8<NT, 4, true, true>(W, ldw, p, n, V, ldv, flag, deflate);
        if (rpg == 6) return cta_jacobi_g8<NT, 6, true, true>(W, ldw, p, n, V, ldv, flag, deflate);
        if (rpg == 8) return cta_jacobi_g8<NT, 8, true, true>(W, ldw, p, n, V, ldv, flag, deflate);
      }
    }
#define SLRA_G8(R)                                                                   \
  if constexpr (R <= (PMAX + 7) / 8) {                                               \
    if (rpg == R) {                                                                  \
      if (exact) cta_jacobi_g8<NT, R, true>(W, ldw, p, n, V, ldv, flag, deflate);    \
      else cta_jacobi_g8<NT, R, false>(W, ldw, p, n, V, ldv, flag, deflate);         \
      return;                                                                        \
    }                                                                                \
  }
    SLRA_G8(1) SLRA_G8(2) SLRA_G8(3) SLRA_G8(4) SLRA_G8(5) SLRA_G8(6) SLRA_G8(7) SLRA_G8(8)
#undef SLRA_G8
  }
  else if constexpr (PMAX > 64) cta_jacobi_t<NT, 8>(W, ldw, p, n, V, ldv, flag, deflate);  // p <= 256 (callers enforce)
}

// Finish an SVD after cta_jacobi: sigma_j = ||w_j||, descending stable order
// (order[t] = source column), S(:, t) = w_j / sigma_j with the sign rule
// "largest-|.| entry of each left vector >= 0" (linalg.cpp:87-96), T from V.
// S (p x n, ld lds) and T (n x n, ld ldt) may not alias W/V.
template <int NT>
__device__ void cta_svd_finish(const double* W, int ldw, int p, int n, const double* V, int ldv, double* sigma,
                               int* order, double* S, int lds, double* T, int ldt, double* sgn) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  for (int j = warp; j < n; j += NW) {
    double acc = 0.0;
    for (int i = lane; i < p; i += 32) acc += W[i + j * ldw] * W[i + j * ldw];
    acc = warp_sum(acc);
    if (lane == 0) sgn[j] = sqrt(acc);  // temp: unsorted sigma
  }
  __syncthreads();
  if (tid == 0) {
    for (int j = 0; j < n; ++j) order[j] = j;
    for (int a = 1; a < n; ++a) {  // stable insertion sort, descending
      const int o = order[a];
      int b = a - 1;
      while (b >= 0 && sgn[order[b]] < sgn[o]) {
        order[b + 1] = order[b];
        --b;
      }
      order[b + 1] = o;
    }
    for (int t = 0; t < n; ++t) sigma[t] = sgn[order[t]];
  }
  __syncthreads();
  for (int t = warp; t < n; t += NW) {
    const int j = order[t];
    const double s = sigma[t];
    const double inv = s > 0.0 ? 1.0 / s : 0.0;
    // sign: first index of the largest |w_ij| (same for w and w/s)
    ArgMax a{-1.0, INT64_MAX};
    for (int i = lane; i < p; i += 32) a = argmax_merge(a, ArgMax{fabs(W[i + j * ldw]), i});
    a = warp_argmax(a);
    const double f = (W[a.i + j * ldw] < 0.0) ? -1.0 : 1.0;
    for (int i = lane; i < p; i += 32) S[i + t * lds] = f * W[i + j * ldw] * inv;
    for (int i = lane; i < n; i += 32) T[i + t * ldt] = f * V[i + j * ldv];
  }
  __syncthreads();
}

}  // namespace slra_dev
