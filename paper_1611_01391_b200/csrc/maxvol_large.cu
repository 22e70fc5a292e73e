// K-b for tall strips that do not fit one SM (config 3: 16384 x 64): maxvol
// (cur.cpp:88-116) as ONE cooperative kernel. Each CTA keeps its slice of
// rows of the orthonormal basis Q in shared memory; every pivot step is a
// grid-wide argmax (one grid barrier, double-buffered candidate slots) after
// which all CTAs rebuild the same Householder reflector from the winning row
// and update their own rows — the exact ColPivHouseholderQR(Q^T) pivot rule
// (largest downdated norm, ties to the lowest current position, LAPACK
// xGEQP3 downdate). The swap rounds solve B = Q G^-1 for the local rows with
// every CTA holding the same small ColPivQR(G^T) factorisation.
#include <cooperative_groups.h>

#include "dense_cta.cuh"

namespace cg = cooperative_groups;

namespace slra_dev {

constexpr int kMT = 256;   // threads per CTA
constexpr int kMRB = 128;  // max rows per CTA
constexpr int kMR = 64;    // max r

struct MaxvolLargeArgs {
  const double* Q;
  int64_t ldq, m;
  int r;
  double h;
  int max_swaps;
  int64_t* I_out;     // r
  double* vol_out;    // nullable
  int32_t* status;
  // global scratch: 2 x grid candidate slots (value, pos, row) + vectors
  double* cand_v;     // 2 x G
  int64_t* cand_pos;  // 2 x G
  int64_t* cand_row;  // 2 x G
  double* cand_vec;   // 2 x G x kMR
};

__global__ void __launch_bounds__(kMT) maxvol_large_kernel(MaxvolLargeArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sm[];
  const int G = gridDim.x, b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = a.r;
  const int64_t rows_per = (a.m + G - 1) / G;
  const int64_t row0 = b * rows_per;
  const int nr = (int)((a.m - row0) < rows_per ? ((a.m - row0) > 0 ? (a.m - row0) : 0) : rows_per);
  double* W = sm;                       // nr x r, row-major (ld r): W[i*r + j]
  double* Gt = W + kMRB * kMR;          // r x r (ld r)
  double* vv = Gt + kMR * kMR;          // reflector (r)
  double* nu = vv + kMR;                // nr
  double* nd = nu + kMRB;               // nr
  double* tau = nd + kMRB;              // r
  double* nu2 = tau + kMR;              // r  (small colpiv scratch)
  double* nd2 = nu2 + kMR;              // r
  double* rv = nd2 + kMR;               // 40
  int64_t* ri = reinterpret_cast<int64_t*>(rv + 40);  // 40
  int64_t* pos = ri + 40;                              // nr current positions
  int* chosen = reinterpret_cast<int*>(pos + kMRB);     // nr
  int* perm = chosen + kMRB;                            // r
  int* Iloc = perm + kMR;                               // r
  __shared__ int sflag[4];
  __shared__ double sbeta;
  // load my rows (first r columns of Q) and their norms
  for (int i = tid; i < nr; i += kMT) {
    double s = 0.0;
    for (int j = 0; j < r; ++j) {
      const double x = a.Q[(row0 + i) + (int64_t)j * a.ldq];
      W[i * r + j] = x;
      s += x * x;
    }
    nu[i] = nd[i] = sqrt(s);
    pos[i] = row0 + i;
    chosen[i] = 0;
  }
  __syncthreads();
  const double sqrt_eps = 1.4901161193847656e-08;
  // ---------------- phase 1: ColPivHouseholderQR(Q^T) pivot order
  for (int k = 0; k < r; ++k) {
    const int slot = k & 1;
    ArgMax best{-1.0, INT64_MAX};  // key: value, then lowest current position
    for (int i = tid; i < nr; i += kMT)
      if (!chosen[i]) best = argmax_merge(best, ArgMax{nu[i], pos[i]});
    best = block_argmax<kMT>(best, rv, ri);
    if (tid == 0) {
      a.cand_v[slot * G + b] = best.v;
      a.cand_pos[slot * G + b] = best.i;
      int64_t row = -1;
      for (int i = 0; i < nr; ++i)
        if (!chosen[i] && pos[i] == best.i) row = row0 + i;
      a.cand_row[slot * G + b] = row;
      if (row >= 0)
        for (int j = 0; j < r; ++j) a.cand_vec[(slot * G + b) * kMR + j] = W[(row - row0) * r + j];
    }
    grid.sync();
    // every CTA reduces the G candidates identically
    if (warp == 0) {
      ArgMax g{-1.0, INT64_MAX};
      for (int c = lane; c < G; c += 32) {
        if (a.cand_row[slot * G + c] < 0) continue;
        g = argmax_merge(g, ArgMax{a.cand_v[slot * G + c], a.cand_pos[slot * G + c]});
      }
      g = warp_argmax(g);
      if (lane == 0) {
        int win = -1;
        for (int c = 0; c < G; ++c)
          if (a.cand_row[slot * G + c] >= 0 && a.cand_pos[slot * G + c] == g.i) win = c;
        sflag[0] = win;
        ri[0] = g.i;  // winning position
      }
    }
    __syncthreads();
    const int win = sflag[0];
    const int64_t big = ri[0];
    const int64_t wrow = a.cand_row[slot * G + win];
    const double* xv = a.cand_vec + (slot * G + win) * kMR;
    // Householder of x = winner row components k..r-1 (warp 0), Eigen arithmetic
    if (warp == 0) {
      double tail = 0.0;
      for (int j = k + 1 + lane; j < r; j += 32) tail += xv[j] * xv[j];
      tail = warp_sum(tail);
      const double c0 = xv[k];
      double t, beta;
      if (tail <= DBL_MIN) {
        t = 0.0;
        beta = c0;
        for (int j = k + 1 + lane; j < r; j += 32) vv[j] = 0.0;
      } else {
        beta = sqrt(c0 * c0 + tail);
        if (c0 >= 0.0) beta = -beta;
        const double den = c0 - beta;
        for (int j = k + 1 + lane; j < r; j += 32) vv[j] = xv[j] / den;
        t = (beta - c0) / beta;
      }
      if (lane == 0) {
        tau[0] = t;
        sbeta = beta;
      }
    }
    // position swap k <-> big, mark the winner chosen
    for (int i = tid; i < nr; i += kMT) {
      if (row0 + i == wrow) chosen[i] = 1;
      if (pos[i] == k) pos[i] = big;
      else if (pos[i] == big) pos[i] = k;
    }
    if (tid == 0) Iloc[k] = (int)wrow;
    __syncthreads();
    const double t = tau[0];
    // update my remaining rows and downdate their norms
    for (int i = tid; i < nr; i += kMT) {
      if (chosen[i]) continue;
      double* wi = W + i * r;
      if (r - k > 1 && t != 0.0) {
        double w = 0.0;
        for (int j = k + 1; j < r; ++j) w += vv[j] * wi[j];
        w += wi[k];
        wi[k] -= t * w;
        for (int j = k + 1; j < r; ++j) wi[j] -= t * vv[j] * w;
      }
      const double nuv = nu[i];
      if (nuv != 0.0) {
        double temp = fabs(wi[k]) / nuv;
        temp = (1.0 + temp) * (1.0 - temp);
        temp = temp < 0.0 ? 0.0 : temp;
        const double ratio = nuv / nd[i];
        const double temp2 = temp * ratio * ratio;
        if (temp2 <= sqrt_eps) {
          double s = 0.0;
          for (int j = k + 1; j < r; ++j) s += wi[j] * wi[j];
          nd[i] = sqrt(s);
          nu[i] = nd[i];
        } else {
          nu[i] = nuv * sqrt(temp);
        }
      }
    }
    __syncthreads();
  }
  // ---------------- phase 2: swap rounds B = Q G^-1 (cur.cpp:100-114)
  for (int swap = 0; swap <= a.max_swaps; ++swap) {
    const int slot = (r + swap) & 1;
    for (int e = tid; e < r * r; e += kMT) {
      const int cc = e % r, t2 = e / r;
      Gt[cc + t2 * r] = a.Q[Iloc[t2] + (int64_t)cc * a.ldq];
    }
    __syncthreads();
    if (warp == 0) {
      SmallColPiv q = warp_colpiv_qr(Gt, r, r, 1e-12, perm, tau, nu2, nd2);
      if (lane == 0) {
        sflag[1] = q.rank < r ? 1 : 0;
        sflag[2] = q.nonzero_pivots;
      }
    }
    __syncthreads();
    if (sflag[1]) {
      if (b == 0 && tid == 0) *a.status = SLRA_ERR_SELECTION_FAILURE;
      return;  // uniform across the grid: every CTA holds the same G
    }
    const int np = sflag[2];
    ArgMax best{-1.0, INT64_MAX};
    for (int i = tid; i < nr; i += kMT) {
      double c[kMR];
      for (int j = 0; j < r; ++j) c[j] = a.Q[(row0 + i) + (int64_t)j * a.ldq];
      for (int k = 0; k < np; ++k) {
        const double t2 = tau[k];
        if (r - k == 1) {
          c[k] *= (1.0 - t2);
        } else if (t2 != 0.0) {
          double w = 0.0;
          for (int j = k + 1; j < r; ++j) w += Gt[j + k * r] * c[j];
          w += c[k];
          c[k] -= t2 * w;
          for (int j = k + 1; j < r; ++j) c[j] -= t2 * Gt[j + k * r] * w;
        }
      }
      for (int t2 = np - 1; t2 >= 0; --t2) {
        double s = c[t2];
        for (int u = t2 + 1; u < np; ++u) s -= Gt[t2 + u * r] * c[u];
        c[t2] = s / Gt[t2 + t2 * r];
      }
      for (int t2 = 0; t2 < r; ++t2) {
        const double v = t2 < np ? fabs(c[t2]) : 0.0;
        best = argmax_merge(best, ArgMax{v, (int64_t)perm[t2] * a.m + (row0 + i)});
      }
    }
    best = block_argmax<kMT>(best, rv, ri);
    if (tid == 0) {
      a.cand_v[slot * G + b] = best.v;
      a.cand_pos[slot * G + b] = best.i;
    }
    grid.sync();
    if (warp == 0) {
      ArgMax g{-1.0, INT64_MAX};
      for (int c = lane; c < G; c += 32) g = argmax_merge(g, ArgMax{a.cand_v[slot * G + c], a.cand_pos[slot * G + c]});
      g = warp_argmax(g);
      if (lane == 0) {
        rv[0] = g.v;
        ri[0] = g.i;
      }
    }
    __syncthreads();
    const double mx = rv[0];
    const int64_t lin = ri[0];
    __syncthreads();
    if (mx <= a.h || swap == a.max_swaps) break;
    if (tid == 0) Iloc[lin / a.m] = (int)(lin % a.m);
    __syncthreads();
  }
  if (b == 0) {
    for (int t2 = tid; t2 < r; t2 += kMT) a.I_out[t2] = Iloc[t2];
    if (a.vol_out) {
      for (int e = tid; e < r * r; e += kMT) Gt[(e % r) + (e / r) * r] = a.Q[Iloc[e % r] + (int64_t)(e / r) * a.ldq];
      __syncthreads();
      if (tid < 32) {
        const double dv = warp_abs_det(Gt, r, r);
        if (tid == 0) *a.vol_out = dv;
      }
    }
    if (tid == 0) *a.status = SLRA_OK;
  }
}

static int maxvol_large_grid(int num_sms, int64_t m) {
  int64_t G = (m + kMRB - 1) / kMRB;
  const int64_t floor_g = num_sms < m ? num_sms : m;
  if (G < floor_g) G = floor_g;
  return (int)G;
}

static size_t maxvol_large_smem() {
  return sizeof(double) * ((size_t)kMRB * kMR + (size_t)kMR * kMR + kMR + 2 * kMRB + 3 * kMR + 40) +
         sizeof(int64_t) * (40 + kMRB) + sizeof(int) * (kMRB + 2 * kMR) + 64;
}

// Grid-wide maxvol over an orthonormal m x r basis Q (device), r <= 64.
int launch_maxvol_large(Context* cx, const double* Q, int64_t ldq, int64_t m, int r, double h, int max_swaps,
                        int64_t* d_idx, double* d_vol, double* scratch) {
  if (r > kMR) return SLRA_ERR_UNSUPPORTED;
  int G = maxvol_large_grid(cx->num_sms, m);
  const int64_t rows_per = (m + G - 1) / G;
  if (rows_per > kMRB) return SLRA_ERR_UNSUPPORTED;
  const size_t smem = maxvol_large_smem();
  SLRA_CUDA(cudaFuncSetAttribute(maxvol_large_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  SLRA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, maxvol_large_kernel, kMT, smem));
  if (per_sm * cx->num_sms < G) return SLRA_ERR_UNSUPPORTED;
  MaxvolLargeArgs args;
  args.Q = Q;
  args.ldq = ldq;
  args.m = m;
  args.r = r;
  args.h = h;
  args.max_swaps = max_swaps;
  args.I_out = d_idx;
  args.vol_out = d_vol;
  args.status = static_cast<int32_t*>(cx->dsmall);
  args.cand_v = scratch;
  args.cand_pos = reinterpret_cast<int64_t*>(scratch + 2 * G);
  args.cand_row = reinterpret_cast<int64_t*>(scratch + 4 * G);
  args.cand_vec = scratch + 6 * G;
  void* kargs[] = {&args};
  {
    KernelTimer kt(cx, "maxvol");
    SLRA_CUDA(cudaLaunchCooperativeKernel((const void*)maxvol_large_kernel, dim3(G), dim3(kMT), kargs, smem,
                                          cx->stream));
  }
  SLRA_CHECK_LAUNCH(cx);
  return SLRA_OK;
}

size_t maxvol_large_scratch_doubles(int num_sms, int64_t m) {
  const size_t G = (size_t)maxvol_large_grid(num_sms, m);
  return 6 * G + 2 * G * kMR + 64;
}

}  // namespace slra_dev
