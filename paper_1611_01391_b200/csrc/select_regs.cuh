// Row selection of select_rows_spanning (cur.cpp:88-135) on an orthonormal
// strip basis Q (m x r, m <= NT, r <= RMAX), one row of Q per thread held in
// registers for the whole selection:
//
//   1. ColPivHouseholderQR(Q^T) and its first r pivots (cur.cpp:95-98): the
//      columns of Q^T are the rows of Q, so every thread owns one column of
//      the factorisation. Eigen's column order is tracked as a per-thread
//      position (the transposition k <-> big of step k is a register update
//      in every thread), the pivot is the first maximum of the updated norms
//      in that order, and the norms follow LAPACK xGEQP3's downdate with the
//      sqrt(eps) recompute guard.
//   2. maxvol round 0 (cur.cpp:100-106): B = Q G^-1 with G = Q(I,:) solved
//      through ColPivQR(G^T). The pivots of step 1 are I in order, so that
//      factorisation is step 1's (same columns, identity permutation): every
//      thread applies every reflector to its own row (what the solve does to
//      each right-hand side), then back-substitutes with R.
//   3. The swap rounds (cur.cpp:107-114): argmax |B| in column-major order,
//      first maximum wins; B is updated by the rank-1 formula (the same B the
//      reference re-solves each round).
//
// Two block barriers per pivot step (argmax, reflector) and two per swap.
// The reflector v of step k is kept with its unit head and zeros above it,
// so the dot product and the update run over whole 8-wide chunks of the
// register row (chunks entirely above k are skipped on a uniform branch)
// with four independent accumulators.
#pragma once

#include "dense_cta.cuh"

namespace slra_dev {

struct SelScratch {
  double* av;   // 2 * (NT / 32) argmax values (double-buffered)
  int* ai;      // 2 * (NT / 32) argmax keys
  double* v;    // RMAX: reflector of the current step
  double* R;    // RMAX x r (ld ldr >= RMAX, even, 16-byte aligned): R of ColPivQR(G^T) on and above the diagonal
  int ldr;
  double* pv;   // r: pivot norms (nonzero-pivot rule)
  double* g;    // RMAX + 1: pivot-row snapshot of a swap round, [RMAX] = pivot value
  double* tau;  // [0]: tau of the current step; [1]: volume
  int* flag;    // [0]: SelectionFailure
};

__host__ __device__ constexpr size_t sel_scratch_doubles(int nt, int rmax) {
  return 2 * (size_t)(nt / 32) + (size_t)rmax + (size_t)rmax * (rmax | 1) + rmax + rmax + 1 + 2;
}

struct ArgMaxI {
  double v;
  int i;
};
__device__ __forceinline__ ArgMaxI argmaxi_merge(ArgMaxI a, ArgMaxI b) {
  return (b.v > a.v || (b.v == a.v && b.i < a.i)) ? b : a;
}
__device__ __forceinline__ ArgMaxI warp_argmaxi(ArgMaxI a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgMaxI b;
    b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
    b.i = __shfl_xor_sync(0xffffffffu, a.i, o);
    a = argmaxi_merge(a, b);
  }
  return a;
}
// Block argmax with ONE barrier: warp results go to slot buffer `buf` and
// every thread reduces the NW entries itself. Consecutive calls must
// alternate `buf` (a slot is rewritten only after the next barrier).
template <int NT>
__device__ __forceinline__ ArgMaxI block_argmaxi(ArgMaxI a, double* av, int* ai, int buf) {
  constexpr int NW = NT / 32;
  a = warp_argmaxi(a);
  if ((threadIdx.x & 31) == 0) {
    av[buf * NW + (threadIdx.x >> 5)] = a.v;
    ai[buf * NW + (threadIdx.x >> 5)] = a.i;
  }
  __syncthreads();
  ArgMaxI r{av[buf * NW], ai[buf * NW]};
#pragma unroll
  for (int w = 1; w < NW; ++w) r = argmaxi_merge(r, ArgMaxI{av[buf * NW + w], ai[buf * NW + w]});
  return r;
}

// Argmax of NON-NEGATIVE doubles with the first-index tie rule by three
// warp reductions (redux.sync): their bit patterns order like the values, so
// the maximum is the max of the high words, then of the low words among
// those, then the min index among the lanes holding it. Exact (no rounding,
// same winner as argmaxi_merge).
__device__ __forceinline__ ArgMaxI warp_argmaxu(double v, int i) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  const unsigned hi = static_cast<unsigned>(b >> 32), lo = static_cast<unsigned>(b);
  const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
  const int mi = __reduce_min_sync(0xffffffffu, (hi == mh && lo == ml) ? i : INT32_MAX);
  return ArgMaxI{__longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(mh) << 32) | ml)), mi};
}
template <int NT>
__device__ __forceinline__ ArgMaxI block_argmaxu(double v, int i, double* av, int* ai, int buf) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31;
  const ArgMaxI a = warp_argmaxu(v, i);
  if (lane == 0) {
    av[buf * NW + (threadIdx.x >> 5)] = a.v;
    ai[buf * NW + (threadIdx.x >> 5)] = a.i;
  }
  __syncthreads();
  return warp_argmaxu(lane < NW ? av[buf * NW + lane] : 0.0, lane < NW ? ai[buf * NW + lane] : INT32_MAX);
}

// Returns SLRA_OK / SLRA_ERR_SELECTION_FAILURE; I_out (smem, r entries) gets
// the selected rows in order; the volume |det Q(I,:)| goes to s.tau[1].
template <int NT, int RMAX>
__device__ int cta_select_regs(const double* Q, int ldq, int m, int r, double h, int max_swaps, int* I_out,
                               const SelScratch& s) {
  static_assert(RMAX % 8 == 0, "chunked register rows");
  constexpr int NCH = RMAX / 8;
  const int tid = threadIdx.x;
  const bool own = tid < m;
  const double sqrt_eps = 1.4901161193847656e-08;
  double x[RMAX];
  double nu, nd;
  {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
    for (int j = 0; j < RMAX; j += 4) {
      x[j] = (own && j < r) ? Q[tid + j * ldq] : 0.0;
      x[j + 1] = (own && j + 1 < r) ? Q[tid + (j + 1) * ldq] : 0.0;
      x[j + 2] = (own && j + 2 < r) ? Q[tid + (j + 2) * ldq] : 0.0;
      x[j + 3] = (own && j + 3 < r) ? Q[tid + (j + 3) * ldq] : 0.0;
      a0 = fma(x[j], x[j], a0);
      a1 = fma(x[j + 1], x[j + 1], a1);
      a2 = fma(x[j + 2], x[j + 2], a2);
      a3 = fma(x[j + 3], x[j + 3], a3);
    }
    nd = sqrt((a0 + a1) + (a2 + a3));
    nu = nd;
  }
  // reciprocals of the two norms, kept in step with them (the downdate then
  // needs one rsqrt on its chain instead of two divisions and a sqrt)
  double rnu = nu > 0.0 ? 1.0 / nu : 0.0, rnd = rnu;
  int pos = tid;  // position of this row (= column of Q^T) in Eigen's permuted order
  int buf = 0;
  for (int k = 0; k < r; ++k) {
    // ---- pivot: first maximum of the updated norms over positions >= k
    const bool cand = own && pos >= k;
    const ArgMaxI best = block_argmaxu<NT>(cand ? nu : 0.0, cand ? pos : INT32_MAX, s.av, s.ai, buf);
    buf ^= 1;
    SLRA_PROF(4);
    const int big = best.i;
    if (pos == big) pos = k;
    else if (pos == k) pos = big;
    // ---- the winner's warp builds H_k from the winning row's tail x[k..r)
    // (Eigen makeHouseholder): the winning lane stages its row, every lane
    // then owns one entry (tail norm by a warp sum, v and R column stored
    // one entry per lane)
    const unsigned wb = __ballot_sync(0xffffffffu, own && pos == k);
    if (wb) {
      const int lane = tid & 31, wl = __ffs(wb) - 1;
      if (lane == wl) {
#pragma unroll
        for (int j = 0; j < RMAX; j += 2) *reinterpret_cast<double2*>(s.g + j) = make_double2(x[j], x[j + 1]);
      }
      __syncwarp();
      const double xl = lane < RMAX ? s.g[lane] : 0.0;
      const double c0 = s.g[k];
      const double tail = warp_sum(lane > k && lane < r ? xl * xl : 0.0);
      // tail == 0: Eigen's tau = 0, beta = c0
      const bool zero = tail <= DBL_MIN;
      double beta, rden, tauk;
      fast_reflector(c0, zero ? 1.0 : tail, beta, rden, tauk);
      beta = zero ? c0 : beta;
      rden = zero ? 0.0 : rden;
      if (lane < RMAX) {
        s.v[lane] = lane < k ? 0.0 : (lane == k ? 1.0 : (lane < r ? xl * rden : 0.0));
        // column k of R: entries above the diagonal (this pivot column after
        // H_0..H_{k-1}), beta on it, zeros below (never read)
        s.R[lane + k * s.ldr] = lane < k ? xl : (lane == k ? beta : 0.0);
      }
      if (lane == 0) {
        s.tau[0] = zero ? 0.0 : tauk;
        s.pv[k] = best.v;
        I_out[k] = (tid & ~31) + wl;
      }
    }
    __syncthreads();
    SLRA_PROF(5);
    // ---- apply H_k to every row (non-pivot rows: the factorisation; pivot
    // rows: the solve's Q_g^T applied to that right-hand side)
    const double t = s.tau[0];
    double w[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // eight chains: 4 deep for RMAX = 32
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      if (8 * c + 7 >= k) {
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
          const double2 vv = *reinterpret_cast<const double2*>(s.v + 8 * c + u);
          w[u] = fma(vv.x, x[8 * c + u], w[u]);
          w[u + 1] = fma(vv.y, x[8 * c + u + 1], w[u + 1]);
        }
      }
    }
    const double tw = t * (((w[0] + w[1]) + (w[2] + w[3])) + ((w[4] + w[5]) + (w[6] + w[7])));
    double xk = 0.0, rest = 0.0;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      if (8 * c + 7 >= k) {
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
          const int j = 8 * c + u;
          const double2 vv = *reinterpret_cast<const double2*>(s.v + j);
          x[j] = fma(-tw, vv.x, x[j]);
          x[j + 1] = fma(-tw, vv.y, x[j + 1]);
          if (j == k) xk = x[j];
          if (j + 1 == k) xk = x[j + 1];
        }
      }
    }
    // ---- xGEQP3 norm downdate of the remaining candidates
    if (own && pos > k && nu != 0.0) {
      double temp = fabs(xk) * rnu;
      temp = (1.0 + temp) * (1.0 - temp);
      temp = temp < 0.0 ? 0.0 : temp;
      const double ratio = nu * rnd;
      if (temp * ratio * ratio <= sqrt_eps) {
#pragma unroll
        for (int j = 0; j < RMAX; ++j)
          if (j > k && j < r) rest = fma(x[j], x[j], rest);
        nd = fast_sqrt(rest);
        nu = nd;
        rnd = rnu = nd > 0.0 ? fast_rcp(nd) : 0.0;
      } else {  // temp > sqrt_eps / ratio^2 > 0 here
        const double y = fast_rsqrt(temp);
        nu = nu * (temp * y);
        rnu = rnu * y;
      }
    }
  }
  SLRA_PROF(6);
  // ---- rank of R with the solve's threshold (ColPivQR(G^T), cur.cpp:103-106)
  if (tid == 0) {
    const double thr_helper = (s.pv[0] * kEps) * (s.pv[0] * kEps) / (double)r;
    int nonzero = r;
    double maxpivot = 0.0;
    for (int k = 0; k < r; ++k) {
      if (nonzero == r && s.pv[k] * s.pv[k] < thr_helper * (double)(r - k)) nonzero = k;
      maxpivot = fmax(maxpivot, fabs(s.R[k + k * s.ldr]));
    }
    int rank = 0;
    double vol = 1.0;
    for (int i = 0; i < nonzero; ++i) rank += (fabs(s.R[i + i * s.ldr]) > maxpivot * 1e-12) ? 1 : 0;
    for (int i = 0; i < r; ++i) vol *= fabs(s.R[i + i * s.ldr]);
    s.flag[0] = rank < r ? 1 : 0;
    s.tau[1] = vol;
  }
  if (tid < r) s.g[tid] = 1.0 / s.R[tid + tid * s.ldr];  // pivot reciprocals for the back substitution
  __syncthreads();
  if (s.flag[0]) return SLRA_ERR_SELECTION_FAILURE;
  // ---- round 0: B(i,:) = R^-1 (Q_g^T a_i), column-oriented back substitution
#pragma unroll
  for (int tt = RMAX - 1; tt >= 0; --tt) {
    if (tt < r) {
      x[tt] *= s.g[tt];
      const double2* rc = reinterpret_cast<const double2*>(s.R + tt * s.ldr);  // ldr even: 16-byte columns
#pragma unroll
      for (int u = 0; u < tt; u += 2) {
        const double2 rr = rc[u >> 1];
        x[u] = fma(-rr.x, x[tt], x[u]);
        if (u + 1 < tt) x[u + 1] = fma(-rr.y, x[tt], x[u + 1]);
      }
    }
    asm volatile("" ::: "memory");  // one column of R live at a time
  }
  SLRA_PROF(7);
  // ---- swap rounds
  double vol = s.tau[1];
  for (int sw = 0; sw <= max_swaps; ++sw) {
    ArgMaxI mine{-1.0, INT32_MAX};
    if (own) {
#pragma unroll
      for (int tt = 0; tt < RMAX; ++tt) {
        const double a = fabs(x[tt]);
        if (tt < r && a > mine.v) {  // column-major order within the row: lower column first
          mine.v = a;
          mine.i = tt * m + tid;
        }
      }
    }
    const ArgMaxI best = block_argmaxu<NT>(own ? mine.v : 0.0, mine.i, s.av, s.ai, buf);
    buf ^= 1;
    if (best.v <= h || sw == max_swaps) break;
    const int j = best.i / m, piv = best.i % m;
    if (tid == piv) {
      double p = 0.0;
#pragma unroll
      for (int tt = 0; tt < RMAX; ++tt)
        if (tt == j) p = x[tt];
#pragma unroll
      for (int tt = 0; tt < RMAX; ++tt) s.g[tt] = x[tt] - (tt == j ? 1.0 : 0.0);
      s.g[RMAX] = p;
      I_out[j] = piv;
    }
    __syncthreads();
    const double p = s.g[RMAX];
    vol *= fabs(p);
    double bij = 0.0;
#pragma unroll
    for (int tt = 0; tt < RMAX; ++tt)
      if (tt == j) bij = x[tt];
    const double f = bij / p;
#pragma unroll
    for (int tt = 0; tt < RMAX; ++tt) x[tt] = fma(-f, s.g[tt], x[tt]);
  }
  __syncthreads();
  if (tid == 0) s.tau[1] = vol;
  __syncthreads();
  SLRA_PROF(8);
  return SLRA_OK;
}

// Column-pivoted Householder QR of a small square G (n x n, n <= 32, ld ldg,
// smem) by ONE warp, each column in a lane's registers — the preconditioner
// of the generator SVD (G Pi = Q R). Eigen's rules as in cta_select_regs
// (first maximum of the updated norms in position order, xGEQP3 downdate),
// no block barriers. Writes R^T (n x n, ld ldr: row k = column k of R, zeros
// above the diagonal of R^T must be pre-filled by the caller), the unit-lower
// reflectors V (n x n, ld ldv), tau[k], perm[k] = original column at position
// k. `vb` (32 doubles, 16-byte aligned) is scratch.
__device__ inline void warp_colpiv_regs(const double* G, int ldg, int n, double* Rt, int ldr, double* V, int ldv,
                                        double* tau, int* perm, double* vb) {
  const int lane = threadIdx.x & 31;
  const bool own = lane < n;
  const double sqrt_eps = 1.4901161193847656e-08;
  double x[32];
  double nu, nd;
  {
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      x[i] = (own && i < n) ? G[i + lane * ldg] : 0.0;
      x[i + 1] = (own && i + 1 < n) ? G[i + 1 + lane * ldg] : 0.0;
      a0 = fma(x[i], x[i], a0);
      a1 = fma(x[i + 1], x[i + 1], a1);
    }
    nd = fast_sqrt(a0 + a1);
    nu = nd;
  }
  int pos = lane;
  for (int k = 0; k < n; ++k) {
    const bool cand = own && pos >= k;
    const ArgMaxI best = warp_argmaxu(cand ? nu : 0.0, cand ? pos : INT32_MAX);
    const int big = best.i;
    if (pos == big) pos = k;
    else if (pos == k) pos = big;
    const unsigned wb = __ballot_sync(0xffffffffu, own && pos == k);
    const int wl = __ffs(wb) - 1;
    if (lane == wl) {
#pragma unroll
      for (int i = 0; i < 32; i += 2) *reinterpret_cast<double2*>(vb + i) = make_double2(x[i], x[i + 1]);
      perm[k] = lane;
    }
    __syncwarp();
    const double xl = vb[lane];
    const double c0 = vb[k];
    const double tail = warp_sum(lane > k && lane < n ? xl * xl : 0.0);
    const bool zero = tail <= DBL_MIN;
    double beta, rden, t;
    fast_reflector(c0, zero ? 1.0 : tail, beta, rden, t);
    beta = zero ? c0 : beta;
    rden = zero ? 0.0 : rden;
    t = zero ? 0.0 : t;
    const double vl = lane < k ? 0.0 : (lane == k ? 1.0 : (lane < n ? xl * rden : 0.0));
    if (own) {
      V[lane + k * ldv] = vl;
      if (lane <= k) Rt[k + lane * ldr] = lane < k ? xl : beta;
    }
    if (lane == 0) tau[k] = t;
    __syncwarp();
    vb[lane] = vl;  // the reflector for every lane's dot product
    __syncwarp();
    double w0 = 0.0, w1 = 0.0, w2 = 0.0, w3 = 0.0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (8 * c + 7 >= k) {
#pragma unroll
        for (int u = 0; u < 8; u += 4) {
          const double2 va = *reinterpret_cast<const double2*>(vb + 8 * c + u);
          const double2 vc = *reinterpret_cast<const double2*>(vb + 8 * c + u + 2);
          w0 = fma(va.x, x[8 * c + u], w0);
          w1 = fma(va.y, x[8 * c + u + 1], w1);
          w2 = fma(vc.x, x[8 * c + u + 2], w2);
          w3 = fma(vc.y, x[8 * c + u + 3], w3);
        }
      }
    }
    const double tw = t * ((w0 + w1) + (w2 + w3));
    double xk = 0.0, rest = 0.0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (8 * c + 7 >= k) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = 8 * c + u;
          x[i] = fma(-tw, vb[i], x[i]);
          if (i == k) xk = x[i];
        }
      }
    }
    if (own && pos > k && nu != 0.0) {
      double temp = fabs(xk) * fast_rcp(nu);
      temp = (1.0 + temp) * (1.0 - temp);
      temp = temp < 0.0 ? 0.0 : temp;
      const double ratio = nu * fast_rcp(nd);
      if (temp * ratio * ratio <= sqrt_eps) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i > k && i < n) rest = fma(x[i], x[i], rest);
        nd = fast_sqrt(rest);
        nu = nd;
      } else {
        nu = nu * fast_sqrt(temp);
      }
    }
    __syncwarp();
  }
}

// Unpivoted Householder QR of a small X (n x nc, n <= 32, nc <= n, ld ldx,
// smem) by ONE warp, a column per lane in registers: the second QR of the
// QLP preconditioner (R_top^T = Q1 R1). Writes W = R1^T (nc x nc, ld ldw;
// the caller zero-fills it), the unit-lower reflectors V1 over X itself
// (ld ldx) and tau1 (nc). `vb` (32 doubles, 16-byte aligned) is scratch.
__device__ inline void warp_house_regs(double* X, int ldx, int n, int nc, double* W, int ldw, double* tau1,
                                       double* vb) {
  const int lane = threadIdx.x & 31;
  const bool own = lane < nc;
  double x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = (own && i < n) ? X[i + lane * ldx] : 0.0;
  __syncwarp();  // every column read before the reflectors overwrite X
  for (int k = 0; k < nc; ++k) {
    if (lane == k) {
#pragma unroll
      for (int i = 0; i < 32; i += 2) *reinterpret_cast<double2*>(vb + i) = make_double2(x[i], x[i + 1]);
    }
    __syncwarp();
    const double xl = vb[lane];
    const double c0 = vb[k];
    const double tail = warp_sum(lane > k && lane < n ? xl * xl : 0.0);
    const bool zero = tail <= DBL_MIN;
    double beta, rden, t;
    fast_reflector(c0, zero ? 1.0 : tail, beta, rden, t);
    beta = zero ? c0 : beta;
    rden = zero ? 0.0 : rden;
    t = zero ? 0.0 : t;
    const double vl = lane < k ? 0.0 : (lane == k ? 1.0 : (lane < n ? xl * rden : 0.0));
    if (lane < n) X[lane + k * ldx] = vl;
    if (lane <= k) W[k + lane * ldw] = lane < k ? xl : beta;  // R1(lane, k) = W(k, lane)
    if (lane == 0) tau1[k] = t;
    __syncwarp();
    vb[lane] = vl;
    __syncwarp();
    double w0 = 0.0, w1 = 0.0, w2 = 0.0, w3 = 0.0;
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      const double2 va = *reinterpret_cast<const double2*>(vb + i);
      const double2 vc = *reinterpret_cast<const double2*>(vb + i + 2);
      w0 = fma(va.x, x[i], w0);
      w1 = fma(va.y, x[i + 1], w1);
      w2 = fma(vc.x, x[i + 2], w2);
      w3 = fma(vc.y, x[i + 3], w3);
    }
    const double tw = t * ((w0 + w1) + (w2 + w3));
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = fma(-tw, vb[i], x[i]);
    __syncwarp();
  }
}

}  // namespace slra_dev
