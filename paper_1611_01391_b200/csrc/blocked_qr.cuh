// thin_qr (linalg.cpp:67-79) of a C-A strip held in shared memory, blocked
// for the FP64 tensor cores: Householder QR in 8-column panels (Eigen
// makeHouseholder reflectors, one block barrier per column, a warp per panel
// column) with each panel's trailing update applied as the compact-WY block
// reflector H = I - V T V^T through DMMA 8x8x4 (W = V^T A split over the
// warps' row ranges, Z = T^T W, A -= V Z), then the explicit Q formed in
// place backwards panel by panel (LAPACK dorgqr: the block reflector on the
// columns to the right through DMMA, the panel's own columns unblocked), and
// the sign rule R(i,i) >= 0 applied to Q's columns. The same reflectors as
// the column-at-a-time factorisation — only the trailing updates are
// regrouped — so Q agrees with it to rounding.
//
// S: m x c (ld lds, m <= 256, c <= 32) in shared memory, overwritten by Q.
// ws: >= 2560 doubles of shared scratch (split-K partials, the panel's
// products, the four T factors). tau: c doubles. red: >= c + 8 doubles.
#pragma once

#include "dense_cta.cuh"

namespace slra_dev {

// V(i, j) of the reflector stored in column j: unit diagonal, zeros above
__device__ __forceinline__ double qr_v(const double* S, int lds, int m, int i, int j) {
  const double x = S[(i < m ? i : m - 1) + j * lds];
  return i == j ? 1.0 : (i > j && i < m ? x : 0.0);
}

// X = V_p^T [V_p | Y(:, n0 : n0 + nt)] (8 x (8 + nt8), col-major, ld 8) by
// DMMA with the rows split over the warps; withV = false skips the V tile
// (X then holds V_p^T Y only, from column 0).
template <int NT>
__device__ void qr_vt_product(const double* S, int lds, int m, int p0, int pb, int n0, int nt, bool withV,
                              double* part, double* X) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  const int g = lane >> 2, t = lane & 3;
  const int ntile = (withV ? 1 : 0) + (nt + 7) / 8;  // <= 4
  double acc[4][2];
#pragma unroll
  for (int n = 0; n < 4; ++n) acc[n][0] = acc[n][1] = 0.0;
  const int r0 = warp * 32;
  if (r0 + 31 >= p0 && r0 < m) {  // rows below p0 carry V = 0
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int k = r0 + 4 * ks + t;
      const double a = g < pb ? qr_v(S, lds, m, k, p0 + g) : 0.0;
#pragma unroll
      for (int n = 0; n < 4; ++n) {
        if (n < ntile) {
          double b;
          if (withV && n == 0) {
            b = a;  // B = V tile: the same element V(k, p0 + g)
          } else {
            const int col = n0 + 8 * (n - (withV ? 1 : 0)) + g;
            const bool ok = k < m && col < n0 + nt;
            b = load_sel(S, (int64_t)k + (int64_t)(ok ? col : n0) * lds, ok);
          }
          dmma_8x8x4(acc[n][0], acc[n][1], a, b);
        }
      }
    }
  }
  const int N8 = 8 * ntile;
#pragma unroll
  for (int n = 0; n < 4; ++n)
    if (n < ntile) {
      part[warp * 8 * N8 + (8 * n + 2 * t) * 8 + g] = acc[n][0];
      part[warp * 8 * N8 + (8 * n + 2 * t + 1) * 8 + g] = acc[n][1];
    }
  __syncthreads();
  for (int e = tid; e < 8 * N8; e += NT) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += part[w * 8 * N8 + e];
    X[e] = s;
  }
  __syncthreads();
}

// Y(:, n0 : n0 + nt) -= V_p Z (rows p0..m-1), Z 8 x nt col-major (ld 8) in smem
template <int NT>
__device__ void qr_vz_update(double* S, int lds, int m, int p0, int pb, int n0, int nt, const double* Z) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = NT / 32;
  const int g = lane >> 2, t = lane & 3;
  const int ntile = (nt + 7) / 8;
  for (int mt = warp; mt < (m + 7) / 8; mt += NW) {
    const int row = 8 * mt + g;
    if (8 * mt + 7 < p0) continue;  // V is zero above p0 (warp-uniform)
    double a[2];
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int j = 4 * ks + t;
      a[ks] = j < pb ? -qr_v(S, lds, m, row, p0 + j) : 0.0;
    }
#pragma unroll
    for (int n = 0; n < 3; ++n) {
      if (n < ntile) {
        const int col = n0 + 8 * n + 2 * t;
        const bool ok0 = row < m && col < n0 + nt, ok1 = row < m && col + 1 < n0 + nt;
        double c0 = load_sel(S, (int64_t)row + (int64_t)(ok0 ? col : n0) * lds, ok0);
        double c1 = load_sel(S, (int64_t)row + (int64_t)(ok1 ? col + 1 : n0) * lds, ok1);
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const double b = Z[(4 * ks + t) + (8 * n + g) * 8];
          dmma_8x8x4(c0, c1, a[ks], b);
        }
        if (ok0) S[row + (int64_t)col * lds] = c0;
        if (ok1) S[row + (int64_t)(col + 1) * lds] = c1;
      }
    }
  }
}

template <int NT>
__device__ void cta_blocked_qr_q(double* S, int lds, int m, int c, double* tau, double* ws, double* red,
                                 bool blocked_q = false) {
  static_assert(NT == 256, "a warp per panel column: 8 warps, 8-column panels");
  constexpr int RPL = 8;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* Tst = ws;             // 4 x 64: T of each panel (col-major 8 x 8)
  double* X = ws + 256;         // 8 x 32: V^T [V | A]
  double* Z = ws + 512;         // 8 x 24
  double* part = ws + 768;      // NW x 8 x 32 split-K partials
  const int np = (c + 7) / 8;
  // ---------------- factorisation
  for (int p = 0; p < np; ++p) {
    const int p0 = 8 * p, p1 = p0 + 8 < c ? p0 + 8 : c, pb = p1 - p0;
    if (p0 >= m) break;
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
    for (int j = p0; j < p1 && j < m; ++j) {
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
    // T of the panel (LAPACK dlarft, forward / columnwise): from V^T V and tau
    const int nt = c - p1;
    qr_vt_product<NT>(S, lds, m, p0, pb, p1, nt, true, part, X);
    if (warp == 0 && lane < 8) {
      double trow[8];  // row `lane` of T
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        double v = 0.0;
        if (j < pb) {
          const double tj = tau[p0 + j];
          if (lane < j) {
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (u >= lane && u < j) v = fma(trow[u], X[u + j * 8], v);  // X(u, j) = v_u . v_j
            v *= -tj;
          } else if (lane == j) {
            v = tj;
          }
        }
        trow[j] = v;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) Tst[p * 64 + lane + 8 * j] = trow[j];
    }
    __syncthreads();
    if (nt > 0) {
      // A_t <- (I - V T^T V^T) A_t: Z = T^T W, W = X(:, 8:8+nt)
      for (int e = tid; e < 8 * nt; e += NT) {
        const int i = e & 7, n = e >> 3;
        double z = 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j <= i) z = fma(Tst[p * 64 + j + 8 * i], X[j + (8 + n) * 8], z);
        Z[e] = z;
      }
      __syncthreads();
      qr_vz_update<NT>(S, lds, m, p0, pb, p1, nt, Z);
      __syncthreads();
    }
  }
  // R's diagonal signs (thin_qr flips Q column / R row so that R(i,i) >= 0)
  for (int j = tid; j < c; j += NT) red[j] = S[j + j * lds] < 0.0 ? -1.0 : 1.0;
  __syncthreads();
  SLRA_PROF(2);
  if (!blocked_q) {
    // Q column by column in each warp's registers (no block barriers), the
    // sign rule folded into the store
    cta_form_q_regs<NT, 8, 32>(S, lds, m, c, tau, S, lds, true, red);
    __syncthreads();
    return;
  }
  // ---------------- explicit Q, in place, panels backwards (dorgqr)
  for (int p = np - 1; p >= 0; --p) {
    const int p0 = 8 * p, p1 = p0 + 8 < c ? p0 + 8 : c, pb = p1 - p0;
    const int nt = c - p1;
    if (nt > 0) {  // Y_t <- (I - V T V^T) Y_t
      qr_vt_product<NT>(S, lds, m, p0, pb, p1, nt, false, part, X);
      for (int e = tid; e < 8 * nt; e += NT) {
        const int i = e & 7, n = e >> 3;
        double z = 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j >= i) z = fma(Tst[p * 64 + i + 8 * j], X[j + n * 8], z);
        Z[e] = z;
      }
      __syncthreads();
      qr_vz_update<NT>(S, lds, m, p0, pb, p1, nt, Z);
      __syncthreads();
    }
    // the panel's own columns, unblocked (dorg2r), i = p1-1 .. p0
    for (int i = p1 - 1; i >= p0; --i) {
      const int k = p0 + warp;
      const double ti = tau[i];
      if (k > i && k < p1) {  // apply H_i to column k (rows i..m-1)
        const double* x = S + i * lds;
        double* a = S + k * lds;
        double xr[RPL], w = 0.0;
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const int ii = lane + 32 * r;
          xr[r] = (ii > i && ii < m) ? x[ii] : 0.0;
          if (ii < m) w = fma(xr[r], a[ii], w);
        }
        const double ai = a[i];
        w = warp_sum(w) + ai;
        if (lane == 0) a[i] = ai - ti * w;
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const int ii = lane + 32 * r;
          if (ii > i && ii < m) a[ii] -= ti * xr[r] * w;
        }
      }
      __syncthreads();
      if (k == i) {  // column i = H_i e_i (its reflector is no longer read)
        double* a = S + i * lds;
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const int ii = lane + 32 * r;
          if (ii < m) a[ii] = ii < i ? 0.0 : (ii == i ? 1.0 - ti : -ti * a[ii]);
        }
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < m * c; e += NT) {
    const int i = e % m, j = e / m;
    S[i + j * lds] *= red[j];
  }
  __syncthreads();
}

}  // namespace slra_dev
