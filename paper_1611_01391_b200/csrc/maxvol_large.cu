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
constexpr int kMRB = 256;  // max rows per CTA (one row per thread: fewer CTAs, fewer candidates per step)
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
  // global scratch: 2 x grid candidate slots (value, key, row) + vectors
  double* cand_v;     // 2 x G
  int64_t* cand_pos;  // 2 x G
  int64_t* cand_row;  // 2 x G
  double* cand_vec;   // 2 x G x kMR
  unsigned* gbar;     // grid barrier arrival counter (zeroed before the launch)
};

// Grid barrier for the co-resident (cooperatively launched) grid: one
// arrival per CTA on a monotonic counter and a spin on its acquire load
// (the cooperative-groups grid.sync was a third of each pivot step).
// target = G * (number of barriers so far, this one included).
__device__ __forceinline__ void grid_barrier(unsigned* gbar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(gbar, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gbar) : "memory");
    } while (v < target);
    __threadfence();
  }
  __syncthreads();
}

// Publish this CTA's candidate (value, key, global row, r-vector) into slot.
__device__ __forceinline__ void publish(const MaxvolLargeArgs& a, int slot, int G, int b, double v, int64_t key,
                                        int64_t row, const double* vec, int r) {
  if (threadIdx.x == 0) {
    a.cand_v[slot * G + b] = v;
    a.cand_pos[slot * G + b] = key;
    a.cand_row[slot * G + b] = row;
  }
  if (row >= 0)
    for (int j = threadIdx.x; j < r; j += kMT) a.cand_vec[(size_t)(slot * G + b) * kMR + j] = vec[j];
}

// After grid.sync: every CTA reduces the G candidates identically (warp 0)
// and returns the winning CTA (first slot holding the winning key).
__device__ __forceinline__ int reduce_candidates(const MaxvolLargeArgs& a, int slot, int G, double* rv, int64_t* ri,
                                                 int* sflag) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    ArgMax g{-1.0, INT64_MAX};
    for (int c = lane; c < G; c += 32) {
      if (__ldcg(a.cand_row + slot * G + c) < 0) continue;
      g = argmax_merge(g, ArgMax{__ldcg(a.cand_v + slot * G + c), __ldcg(a.cand_pos + slot * G + c)});
    }
    g = warp_argmax(g);
    int win = G;
    for (int c = lane; c < G; c += 32)
      if (__ldcg(a.cand_row + slot * G + c) >= 0 && __ldcg(a.cand_pos + slot * G + c) == g.i) win = min(win, c);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) win = min(win, __shfl_xor_sync(0xffffffffu, win, o));
    if (lane == 0) {
      sflag[0] = win;
      rv[0] = g.v;
      ri[0] = g.i;
    }
  }
  __syncthreads();
  return sflag[0];
}

__global__ void __launch_bounds__(kMT) maxvol_large_kernel(MaxvolLargeArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sm[];
  const int G = gridDim.x, b = blockIdx.x;
  const int tid = threadIdx.x;
  const int r = a.r;
  const int ldw = r | 1;  // odd row stride: conflict-free column access by row-threads
  const int64_t rows_per = (a.m + G - 1) / G;
  const int64_t row0 = b * rows_per;
  const int nr = (int)((a.m - row0) < rows_per ? ((a.m - row0) > 0 ? (a.m - row0) : 0) : rows_per);
  double* W = sm;                       // nr x r, row-major (ld ldw): Q rows, then B rows
  double* Rm = W + kMRB * (kMR + 1);    // r x r (ld r): R11 of ColPivQR(Q^T) restricted to I
  double* vv = Rm + kMR * kMR;          // reflector (r)
  double* nu = vv + kMR;                // nr
  double* nd = nu + kMRB;               // nr
  double* fr = nd + kMRB;               // nr (swap factors)
  double* bi = fr + kMRB;               // r (winning row of B)
  double* rv = bi + kMR;                // 40
  int64_t* ri = reinterpret_cast<int64_t*>(rv + 40);  // 40
  int64_t* pos = ri + 40;                              // nr current positions
  int* chosen = reinterpret_cast<int*>(pos + kMRB);     // nr: 0, or 1 + pivot step
  int* Iloc = chosen + kMRB;                            // r
  __shared__ int sflag[4];
  __shared__ double sbeta, stau, smaxpivot;
  int sync_no = 0;
  // load my rows (first r columns of Q) and their norms
  for (int i = tid; i < nr; i += kMT) {
    double s = 0.0;
    for (int j = 0; j < r; ++j) {
      const double x = a.Q[(row0 + i) + (int64_t)j * a.ldq];
      W[i * ldw + j] = x;
      s += x * x;
    }
    nu[i] = nd[i] = sqrt(s);
    pos[i] = row0 + i;
    chosen[i] = 0;
  }
  if (tid == 0) smaxpivot = 0.0;
  __syncthreads();
  const double sqrt_eps = 1.4901161193847656e-08;
  // ---------------- phase 1: ColPivHouseholderQR(Q^T) pivot order. Its
  // reflectors and R11 are exactly those of ColPivQR(G^T) for G = Q[I,:]
  // (same columns, same greedy order), so the first solve B = Q G^-1 reuses
  // them (cur.cpp:100-108).
  for (int k = 0; k < r; ++k) {
    const int slot = (sync_no++) & 1;
    // key: value, then the lowest current position; the local row rides in
    // the key's low 16 bits (positions are unique, so the order is unchanged)
    ArgMax best{-1.0, INT64_MAX};
    for (int i = tid; i < nr; i += kMT)
      if (!chosen[i]) best = argmax_merge(best, ArgMax{nu[i], (pos[i] << 16) | i});
    best = block_argmax<kMT>(best, rv, ri);
    const int li = best.i == INT64_MAX ? -1 : (int)(best.i & 0xffff);
    publish(a, slot, G, b, best.v, best.i, li >= 0 ? row0 + li : -1, li >= 0 ? W + li * ldw : nullptr, r);
    grid_barrier(a.gbar, (unsigned)(G * sync_no));
    const int win = reduce_candidates(a, slot, G, rv, ri, sflag);
    const int64_t big = ri[0] >> 16;
    const double pivnorm = rv[0];
    const int64_t wrow = __ldcg(a.cand_row + slot * G + win);
    const double* xv = a.cand_vec + (size_t)(slot * G + win) * kMR;
    // Householder of x = winner row components k..r-1 (warp 0), Eigen arithmetic
    if (tid < 32) {
      const int lane = tid;
      double tail = 0.0;
      for (int j = k + 1 + lane; j < r; j += 32) tail += __ldcg(xv + j) * __ldcg(xv + j);
      tail = warp_sum(tail);
      const double c0 = __ldcg(xv + k);
      double t, beta;
      if (tail <= DBL_MIN) {
        t = 0.0;
        beta = c0;
        for (int j = k + 1 + lane; j < r; j += 32) vv[j] = 0.0;
      } else {
        beta = sqrt(c0 * c0 + tail);
        if (c0 >= 0.0) beta = -beta;
        const double den = c0 - beta;
        for (int j = k + 1 + lane; j < r; j += 32) vv[j] = __ldcg(xv + j) / den;
        t = (beta - c0) / beta;
      }
      if (lane == 0) {
        stau = t;
        sbeta = beta;
        if (fabs(beta) > smaxpivot) smaxpivot = fabs(beta);
      }
    } else {
      // R11 column k: entries above the diagonal are the winner's first k components
      for (int t2 = tid - 32; t2 < k; t2 += kMT - 32) Rm[t2 + k * r] = __ldcg(xv + t2);
    }
    // position swap k <-> big, mark the winner chosen
    for (int i = tid; i < nr; i += kMT) {
      if (row0 + i == wrow) chosen[i] = 1 + k;
      if (pos[i] == k) pos[i] = big;
      else if (pos[i] == big) pos[i] = k;
    }
    if (tid == 0) Iloc[k] = (int)wrow;
    __syncthreads();
    (void)pivnorm;
    const double t = stau;
    if (tid == 0) Rm[k + k * r] = sbeta;
    // update my remaining rows and downdate their norms
    for (int i = tid; i < nr; i += kMT) {
      if (chosen[i]) continue;
      double* wi = W + i * ldw;
      if (r - k > 1 && t != 0.0) {
        double w0 = 0.0, w1 = 0.0, w2 = 0.0, w3 = 0.0;  // four chains (FP64 FMA latency ~24)
        int j = k + 1;
        for (; j + 3 < r; j += 4) {
          w0 = fma(vv[j], wi[j], w0);
          w1 = fma(vv[j + 1], wi[j + 1], w1);
          w2 = fma(vv[j + 2], wi[j + 2], w2);
          w3 = fma(vv[j + 3], wi[j + 3], w3);
        }
        for (; j < r; ++j) w0 = fma(vv[j], wi[j], w0);
        double w = (w0 + w1) + (w2 + w3);
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
  // rank() of ColPivQR(G^T) with threshold 1e-12 (cur.cpp:103-104): the R11
  // diagonal is the same for every CTA, so the exit is grid-uniform.
  {
    const double pre = smaxpivot * 1e-12;
    int rank = 0;
    for (int k = 0; k < r; ++k) rank += fabs(Rm[k + k * r]) > pre ? 1 : 0;
    if (rank < r) {
      if (b == 0 && tid == 0) *a.status = SLRA_ERR_SELECTION_FAILURE;
      return;
    }
  }
  // ---------------- phase 2: B = Q G^-1 for my rows (R11 back substitution
  // of the reflected rows), then swap rounds with the rank-1 update
  // B <- B - B[:,j] (B[i,:] - e_j) / B[i,j] after placing row i at slot j.
  for (int i = tid; i < nr; i += kMT) {
    double* c = W + i * ldw;
    if (chosen[i]) {
      const int pk = chosen[i] - 1;
      for (int j = 0; j < r; ++j) c[j] = j == pk ? 1.0 : 0.0;
      continue;
    }
    // (the last reflector has tau = 0: nothing left to apply)
    for (int t2 = r - 1; t2 >= 0; --t2) {
      double s = c[t2];
      for (int u = t2 + 1; u < r; ++u) s -= Rm[t2 + u * r] * c[u];
      c[t2] = s / Rm[t2 + t2 * r];
    }
  }
  __syncthreads();
  for (int swap = 0; swap <= a.max_swaps; ++swap) {
    const int slot = (sync_no++) & 1;
    // B.cwiseAbs().maxCoeff: column-major first maximum -> key j*m + row
    ArgMax best{-1.0, INT64_MAX};
    for (int e = tid; e < nr * r; e += kMT) {
      const int i = e / r, j = e - i * r;
      best = argmax_merge(best, ArgMax{fabs(W[i * ldw + j]), (int64_t)j * a.m + (row0 + i)});
    }
    best = block_argmax<kMT>(best, rv, ri);
    const int64_t lrow = best.i == INT64_MAX ? -1 : (best.i % a.m);
    publish(a, slot, G, b, best.v, best.i, lrow, lrow >= 0 ? W + (lrow - row0) * ldw : nullptr, r);
    grid_barrier(a.gbar, (unsigned)(G * sync_no));
    const int win = reduce_candidates(a, slot, G, rv, ri, sflag);
    const double mx = rv[0];
    const int64_t lin = ri[0];
    if (mx <= a.h || swap == a.max_swaps) break;
    const int j = (int)(lin / a.m);
    const double* xv = a.cand_vec + (size_t)(slot * G + win) * kMR;
    for (int c = tid; c < r; c += kMT) bi[c] = __ldcg(xv + c) - (c == j ? 1.0 : 0.0);
    const double p = __ldcg(xv + j);
    for (int i = tid; i < nr; i += kMT) fr[i] = W[i * ldw + j] / p;
    if (tid == 0) Iloc[j] = (int)(lin % a.m);
    __syncthreads();
    for (int e = tid; e < nr * r; e += kMT) {
      const int i = e / r, c = e - i * r;
      W[i * ldw + c] -= fr[i] * bi[c];
    }
    __syncthreads();
  }
  if (b == 0) {
    for (int t2 = tid; t2 < r; t2 += kMT) a.I_out[t2] = Iloc[t2];
    if (a.vol_out) {
      __syncthreads();
      for (int e = tid; e < r * r; e += kMT) Rm[(e % r) + (e / r) * r] = a.Q[Iloc[e % r] + (int64_t)(e / r) * a.ldq];
      __syncthreads();
      if (tid < 32) {
        const double dv = warp_abs_det(Rm, r, r);
        if (tid == 0) *a.vol_out = dv;
      }
    }
    if (tid == 0) *a.status = SLRA_OK;
  }
}

static int maxvol_large_grid(int num_sms, int64_t m) {
  (void)num_sms;  // as few CTAs as the rows allow: fewer candidates to reduce per step
  return (int)((m + kMRB - 1) / kMRB);
}

static size_t maxvol_large_smem() {
  return sizeof(double) * ((size_t)kMRB * (kMR + 1) + (size_t)kMR * kMR + kMR + 3 * kMRB + kMR + 40) +
         sizeof(int64_t) * (40 + kMRB) + sizeof(int) * (kMRB + kMR) + 64;
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
  args.gbar = reinterpret_cast<unsigned*>(scratch + 6 * G + 2 * (size_t)G * kMR);
  SLRA_CUDA(cudaMemsetAsync(args.gbar, 0, sizeof(unsigned), cx->stream));
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
