// Householder QR of a strip held in shared memory, blocked for the FP64
// tensor cores (thin_qr, linalg.cpp:67-79; Eigen HouseholderQR's reflectors):
// panels of PB = NT/32 columns — a warp per panel column, ONE block barrier
// per column (the owner of column j+1 builds H_{j+1}, Eigen makeHouseholder,
// while the other warps apply H_j) — and each panel's trailing update applied
// as the compact-WY block reflector H = I - V T V^T through DMMA 8x8x4:
// X = V^T [V | A] with the rows split over the warps (deterministic fixed-order
// reduction), T from V^T V and tau (LAPACK dlarft), Z = T^T W, A -= V Z.
// The same reflectors as the column-at-a-time factorisation — only the
// trailing updates are regrouped — so R / Q agree with it to rounding.
//
//   cta_blocked_house_qr: S (m x c, ld lds, m <= 256, c <= 4 PB) -> R on and
//     above the diagonal, the essential reflector parts below, tau (c).
//   cta_blocked_qr_q: the same, then the explicit thin Q in place with the
//     sign rule R(i,i) >= 0 applied to its columns (red[j] = sign).
// ws: shared scratch of qr_ws_doubles<NT>() doubles.
#pragma once

#include "dense_cta.cuh"

namespace slra_dev {

// warps that split the (<= 256) rows of the V^T [V | A] product: 8 for
// 8-column panels, 4 for 16-column panels (bounds the partials' smem)
template <int NT>
__host__ __device__ constexpr int qr_row_warps() {
  return NT / 32 == 8 ? 8 : 4;
}
template <int NT>
__host__ __device__ constexpr int qr_ws_doubles() {
  // T (4 panels x PB x PB) + X (PB x 4 PB) + Z (PB x 3 PB) + partials (row-warps x PB x 4 PB)
  return 4 * (NT / 32) * (NT / 32) + 4 * (NT / 32) * (NT / 32) + 3 * (NT / 32) * (NT / 32) +
         qr_row_warps<NT>() * 4 * (NT / 32) * (NT / 32);
}

// V(i, j) of the reflector stored in column j: unit diagonal, zeros above
__device__ __forceinline__ double qr_v(const double* S, int lds, int m, int i, int j) {
  const double x = S[(i < m ? i : m - 1) + j * lds];
  return i == j ? 1.0 : (i > j && i < m ? x : 0.0);
}

// X = V_p^T [V_p | Y(:, n0 : n0 + nt)] (PB x (PB + nt8), col-major, ld PB).
// Warp w < RW takes rows [RR w, RR (w + 1)); fixed-order sum over them.
template <int NT>
__device__ void qr_vt_product(const double* S, int lds, int m, int p0, int pb, int n0, int nt, double* part,
                              double* X) {
  constexpr int PB = NT / 32, MT = PB / 8, NTMAX = 4 * PB / 8;
  constexpr int RW = qr_row_warps<NT>(), RR = 256 / RW;  // row-warps, rows each
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int ntile = MT + (nt + 7) / 8;  // V tiles, then the Y tiles
  const int N = 8 * ntile;
  double acc[MT][NTMAX][2];
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int n = 0; n < NTMAX; ++n) acc[a][n][0] = acc[a][n][1] = 0.0;
  const int r0 = warp * RR;
  if (warp < RW && r0 + RR - 1 >= p0 && r0 < m) {  // rows below p0 carry V = 0
#pragma unroll 2
    for (int ks = 0; ks < RR / 4; ++ks) {
      const int k = r0 + 4 * ks + t;
      double av[MT];
#pragma unroll
      for (int a = 0; a < MT; ++a) av[a] = 8 * a + g < pb ? qr_v(S, lds, m, k, p0 + 8 * a + g) : 0.0;
#pragma unroll
      for (int n = 0; n < NTMAX; ++n) {
        if (n < ntile) {
          double b;
          if (n < MT) {
            b = 8 * n + g < pb ? qr_v(S, lds, m, k, p0 + 8 * n + g) : 0.0;
          } else {
            const int col = n0 + 8 * (n - MT) + g;
            const bool ok = k < m && col < n0 + nt;
            b = load_sel(S, (int64_t)k + (int64_t)(ok ? col : n0) * lds, ok);
          }
#pragma unroll
          for (int a = 0; a < MT; ++a) dmma_8x8x4(acc[a][n][0], acc[a][n][1], av[a], b);
        }
      }
    }
  }
  if (warp < RW) {
#pragma unroll
    for (int a = 0; a < MT; ++a)
#pragma unroll
      for (int n = 0; n < NTMAX; ++n)
        if (n < ntile) {
          part[warp * PB * N + (8 * n + 2 * t) * PB + 8 * a + g] = acc[a][n][0];
          part[warp * PB * N + (8 * n + 2 * t + 1) * PB + 8 * a + g] = acc[a][n][1];
        }
  }
  __syncthreads();
  for (int e = tid; e < PB * N; e += NT) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < RW; ++w) s += part[w * PB * N + e];
    X[e] = s;
  }
  __syncthreads();
}

// Y(:, n0 : n0 + nt) -= V_p Z (rows p0..m-1); Z PB x nt col-major (ld PB)
template <int NT>
__device__ void qr_vz_update(double* S, int lds, int m, int p0, int pb, int n0, int nt, const double* Z) {
  constexpr int PB = NT / 32, KS = PB / 4, NW = NT / 32, NTMAX = 3 * PB / 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int ntile = (nt + 7) / 8;
  for (int mt = warp; mt < (m + 7) / 8; mt += NW) {
    const int row = 8 * mt + g;
    if (8 * mt + 7 < p0) continue;  // V is zero above p0 (warp-uniform)
    double a[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int j = 4 * ks + t;
      a[ks] = j < pb ? -qr_v(S, lds, m, row, p0 + j) : 0.0;
    }
#pragma unroll
    for (int n = 0; n < NTMAX; ++n) {
      if (n < ntile) {
        const int col = n0 + 8 * n + 2 * t;
        const bool ok0 = row < m && col < n0 + nt, ok1 = row < m && col + 1 < n0 + nt;
        double c0 = load_sel(S, (int64_t)row + (int64_t)(ok0 ? col : n0) * lds, ok0);
        double c1 = load_sel(S, (int64_t)row + (int64_t)(ok1 ? col + 1 : n0) * lds, ok1);
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) dmma_8x8x4(c0, c1, a[ks], Z[(4 * ks + t) + (8 * n + g) * PB]);
        if (ok0) S[row + (int64_t)col * lds] = c0;
        if (ok1) S[row + (int64_t)(col + 1) * lds] = c1;
      }
    }
  }
}

template <int NT>
__device__ void cta_blocked_house_qr(double* S, int lds, int m, int c, double* tau, double* ws) {
  constexpr int PB = NT / 32;  // panel width = warps
  static_assert(PB % 8 == 0, "panels of 8 or 16 columns");
  constexpr int RPL = 8;       // m <= 256
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* Tst = ws;                       // 4 panels x PB x PB
  double* X = Tst + 4 * PB * PB;          // PB x 4 PB
  double* Z = X + 4 * PB * PB;            // PB x 3 PB
  double* part = Z + 3 * PB * PB;         // row-warps x PB x 4 PB
  const int size = m < c ? m : c;
  const int np = (size + PB - 1) / PB;
  for (int p = 0; p < np; ++p) {
    const int p0 = PB * p, p1 = p0 + PB < size ? p0 + PB : size, pb = p1 - p0;
    // panel: column p0 + w belongs to warp w; H_{p0} built by warp 0
    if (warp == 0) {
      double s = 0.0;
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int i = lane + 32 * r;
        if (i > p0 && i < m) s = fma(S[i + p0 * lds], S[i + p0 * lds], s);
      }
      s = warp_sum(s);
      house_make<RPL, true>(S + p0 * lds, p0, m, s, tau);
    }
    __syncthreads();
    for (int j = p0; j < p1; ++j) {
      const int k = p0 + warp;  // this warp's panel column
      if (k > j && k < p1) {    // warp-uniform
        const double* x = S + j * lds;
        double* a = S + k * lds;
        const double tj = tau[j];
        double xr[RPL], w = 0.0;
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const int i = lane + 32 * r;
          xr[r] = (i > j && i < m) ? x[i] : 0.0;
          if (i < m) w = fma(xr[r], a[i], w);
        }
        const double aj = a[j];
        w = warp_sum(w) + aj;
        if (lane == 0) a[j] = aj - tj * w;
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const int i = lane + 32 * r;
          if (i > j && i < m) {
            const double v = a[i] - tj * xr[r] * w;
            a[i] = v;
            if (i > j + 1) s = fma(v, v, s);
          }
        }
        if (k == j + 1) {
          s = warp_sum(s);
          house_make<RPL, true>(a, k, m, s, tau);
        }
      }
      __syncthreads();
    }
    const int nt = c - p1;  // trailing columns (past `size` too: R's rightmost block)
    if (nt > 0) {
      qr_vt_product<NT>(S, lds, m, p0, pb, p1, nt, part, X);
      // T (LAPACK dlarft, forward / columnwise): row `lane` of T per lane
      if (warp == 0 && lane < PB) {
        double trow[PB];
#pragma unroll
        for (int j = 0; j < PB; ++j) {
          double v = 0.0;
          if (j < pb) {
            const double tj = tau[p0 + j];
            if (lane < j) {
#pragma unroll
              for (int u = 0; u < PB; ++u)
                if (u >= lane && u < j) v = fma(trow[u], X[u + j * PB], v);  // X(u, j) = v_u . v_j
              v *= -tj;
            } else if (lane == j) {
              v = tj;
            }
          }
          trow[j] = v;
        }
#pragma unroll
        for (int j = 0; j < PB; ++j) Tst[p * PB * PB + lane + PB * j] = trow[j];
      }
      __syncthreads();
      // A_t <- (I - V T^T V^T) A_t: Z = T^T W, W = X(:, PB : PB + nt)
      for (int e = tid; e < PB * nt; e += NT) {
        const int i = e % PB, n = e / PB;
        double z = 0.0;
#pragma unroll
        for (int j = 0; j < PB; ++j)
          if (j <= i) z = fma(Tst[p * PB * PB + j + PB * i], X[j + (PB + n) * PB], z);
        Z[e] = z;
      }
      __syncthreads();
      qr_vz_update<NT>(S, lds, m, p0, pb, p1, nt, Z);
      __syncthreads();
    }
  }
}

template <int NT>
__device__ void cta_blocked_qr_q(double* S, int lds, int m, int c, double* tau, double* ws, double* red) {
  cta_blocked_house_qr<NT>(S, lds, m, c, tau, ws);
  // R's diagonal signs (thin_qr flips Q column / R row so that R(i,i) >= 0)
  for (int j = threadIdx.x; j < c; j += NT) red[j] = S[j + j * lds] < 0.0 ? -1.0 : 1.0;
  __syncthreads();
  SLRA_PROF(2);
  // Q column by column in each warp's registers (no block barriers), the sign
  // rule folded into the store
  if (c <= 32) cta_form_q_regs<NT, 8, 32>(S, lds, m, c, tau, S, lds, true, red);
  else if constexpr (NT >= 512) cta_form_q_regs<NT, 8, 64>(S, lds, m, c, tau, S, lds, true, red);
  __syncthreads();
}

}  // namespace slra_dev
