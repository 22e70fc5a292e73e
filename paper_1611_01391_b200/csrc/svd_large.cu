// SVD (linalg.cpp:81-98) of operands too large for one CTA's shared memory
// (min(m, n) > 64 or max(m, n) > 256), batched over equally-shaped problems:
// the HSS builder's off-diagonal blocks (hss.cpp:69-96), one level at a time.
//
// One-sided (Hestenes) Jacobi on W = A (m >= n) in HBM/L2, V accumulated
// alongside, as ONE cooperative kernel: each round of the round-robin
// schedule gives every warp of the grid one column pair (of any problem),
// then a grid barrier. Jacobi computes small singular values to high
// relative accuracy, which is what the HSS rank search's tail norms need.
// A finishing pass forms sigma_j = ||w_j||, a stable descending order (rank
// counting, parallel), S = w / sigma with the reference's sign rule, T = V.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace slra_dev {

constexpr double kEpsL = 2.220446049250313e-16;
constexpr int kJT = 256;  // threads per CTA of the sweep kernel
constexpr int kJMaxSweeps = 60;

struct JacobiGlobalArgs {
  double* W;
  int64_t ldw, sW;
  double* V;
  int64_t ldv, sV;
  int m, n, nb;
  int* rotated;  // kJMaxSweeps flags (zeroed before launch)
  int* sweeps_used;
  double tol2;
};

__device__ __forceinline__ void rr_pair(int rd, int pi, int ne, int& a, int& b) {
  if (pi == 0) {
    a = rd;
    b = ne - 1;
  } else {
    a = (rd + pi) % (ne - 1);
    b = (rd - pi + ne - 1) % (ne - 1);
  }
  if (a > b) {
    const int t = a;
    a = b;
    b = t;
  }
}

__global__ void __launch_bounds__(kJT) jacobi_global_kernel(JacobiGlobalArgs g) {
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = ((int64_t)blockIdx.x * kJT + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kJT) >> 5;
  const int m = g.m, n = g.n;
  const int ne = n + (n & 1), npairs = ne / 2;
  const int64_t tasks = (int64_t)g.nb * npairs;
  for (int sweep = 0; sweep < kJMaxSweeps; ++sweep) {
    bool any = false;
    for (int rd = 0; rd < ne - 1; ++rd) {
      for (int64_t task = gwarp; task < tasks; task += nwarps) {
        const int b = (int)(task / npairs), pi = (int)(task % npairs);
        int ca, cb;
        rr_pair(rd, pi, ne, ca, cb);
        if (cb >= n) continue;
        double* wp = g.W + b * g.sW + (int64_t)ca * g.ldw;
        double* wq = g.W + b * g.sW + (int64_t)cb * g.ldw;
        double aa = 0.0, bb = 0.0, gg = 0.0, a1 = 0.0, b1 = 0.0, g1 = 0.0;
        int i = lane;
        for (; i + 32 < m; i += 64) {
          const double x0 = wp[i], y0 = wq[i], x1 = wp[i + 32], y1 = wq[i + 32];
          aa = fma(x0, x0, aa);
          bb = fma(y0, y0, bb);
          gg = fma(x0, y0, gg);
          a1 = fma(x1, x1, a1);
          b1 = fma(y1, y1, b1);
          g1 = fma(x1, y1, g1);
        }
        if (i < m) {
          const double x0 = wp[i], y0 = wq[i];
          aa = fma(x0, x0, aa);
          bb = fma(y0, y0, bb);
          gg = fma(x0, y0, gg);
        }
        aa = warp_sum(aa + a1);
        bb = warp_sum(bb + b1);
        gg = warp_sum(gg + g1);
        if (gg == 0.0 || gg * gg <= g.tol2 * (aa * bb)) continue;
        const double d = bb - aa, g2 = 2.0 * gg;
        const double rr = (g2 * g2 < 1e-17 * (d * d)) ? fabs(d) : sqrt(fma(d, d, g2 * g2));
        const double t = copysign(1.0, d) * g2 / (fabs(d) + rr);
        const double cs = rsqrt(fma(t, t, 1.0));
        const double sn = cs * t;
        for (int k = lane; k < m; k += 32) {
          const double x = wp[k], y = wq[k];
          wp[k] = cs * x - sn * y;
          wq[k] = sn * x + cs * y;
        }
        double* vp = g.V + b * g.sV + (int64_t)ca * g.ldv;
        double* vq = g.V + b * g.sV + (int64_t)cb * g.ldv;
        for (int k = lane; k < n; k += 32) {
          const double x = vp[k], y = vq[k];
          vp[k] = cs * x - sn * y;
          vq[k] = sn * x + cs * y;
        }
        any = true;
      }
      grid.sync();
    }
    // per-sweep flag (zeroed before launch): no reset race between sweeps
    if (__syncthreads_or(any) && threadIdx.x == 0) atomicOr(g.rotated + sweep, 1);
    grid.sync();
    if (*(volatile int*)(g.rotated + sweep) == 0) {
      if (blockIdx.x == 0 && threadIdx.x == 0) *g.sweeps_used = sweep + 1;
      return;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *g.sweeps_used = kJMaxSweeps;
}

// sigma_j = ||w_j|| per (column, problem): one warp each.
__global__ void col_norms_kernel(const double* __restrict__ W, int64_t ldw, int64_t sW, int m, int n,
                                 double* __restrict__ sg, int64_t sSg) {
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int b = blockIdx.y;
  if (j >= n) return;
  const double* w = W + b * sW + (int64_t)j * ldw;
  double s = 0.0;
  for (int i = lane; i < m; i += 32) s = fma(w[i], w[i], s);
  s = warp_sum(s);
  if (lane == 0) sg[b * sSg + j] = sqrt(s);
}

// Stable descending order by rank counting: pos(j) = #{k : s_k > s_j or
// (s_k == s_j and k < j)}; order[pos(j)] = j, sigma[pos(j)] = s_j.
__global__ void rank_order_kernel(const double* __restrict__ sg, int64_t sSg, int n, int* __restrict__ order,
                                  double* __restrict__ sigma, int64_t sSig) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (j >= n) return;
  const double* s = sg + b * sSg;
  const double v = s[j];
  int pos = 0;
  for (int k = 0; k < n; ++k) pos += (s[k] > v || (s[k] == v && k < j)) ? 1 : 0;
  order[(int64_t)b * n + pos] = j;
  sigma[b * sSig + pos] = v;
}

// S(:, t) = f w_j / sigma_t, T(:, t) = f v_j with j = order[t] and f the sign
// making the first largest-|.| entry of S(:, t) nonnegative.
__global__ void svd_emit_kernel(const double* __restrict__ W, int64_t ldw, int64_t sW, const double* __restrict__ V,
                                int64_t ldv, int64_t sV, int m, int n, const int* __restrict__ order,
                                const double* __restrict__ sigma, int64_t sSig, double* __restrict__ S, int64_t lds,
                                int64_t sS, double* __restrict__ T, int64_t ldt, int64_t sT) {
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int b = blockIdx.y;
  if (t >= n) return;
  const int j = order[(int64_t)b * n + t];
  const double* w = W + b * sW + (int64_t)j * ldw;
  const double* v = V + b * sV + (int64_t)j * ldv;
  ArgMax a{-1.0, INT64_MAX};
  for (int i = lane; i < m; i += 32) a = argmax_merge(a, ArgMax{fabs(w[i]), i});
  a = warp_argmax(a);
  const double f = w[a.i] < 0.0 ? -1.0 : 1.0;
  const double s = sigma[b * sSig + t];
  const double inv = s > 0.0 ? 1.0 / s : 0.0;
  double* So = S + b * sS + (int64_t)t * lds;
  double* To = T + b * sT + (int64_t)t * ldt;
  for (int i = lane; i < m; i += 32) So[i] = f * w[i] * inv;
  for (int i = lane; i < n; i += 32) To[i] = f * v[i];
}

__global__ void copy_identity_kernel(const double* __restrict__ A, int64_t lda, int64_t sA, int m, int n,
                                     double* __restrict__ W, int64_t sW, double* __restrict__ V, int64_t sV) {
  const int b = blockIdx.y;
  const int64_t tw = (int64_t)m * n, tv = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tw + tv; e += (int64_t)gridDim.x * blockDim.x) {
    if (e < tw) {
      const int64_t i = e % m, j = e / m;
      W[b * sW + e] = A[b * sA + i + j * lda];
    } else {
      const int64_t f = e - tw, i = f % n, j = f / n;
      V[b * sV + f] = i == j ? 1.0 : 0.0;
    }
  }
}

size_t svd_large_workspace_doubles(int64_t m, int64_t n, int nb) {
  return (size_t)nb * ((size_t)m * n + (size_t)n * n + 2 * (size_t)n) + (size_t)kJMaxSweeps + 64;
}

// nb problems A_b = A + b sA (m x n, m >= n, ld lda) -> S_b (m x n), sigma_b
// (n), T_b (n x n). ws: svd_large_workspace_doubles(m, n, nb).
int launch_svd_large_batched(Context* cx, const double* A, int64_t lda, int64_t sA, int m, int n, int nb,
                             double* S, int64_t lds, int64_t sS, double* sigma, int64_t sSig, double* T, int64_t ldt,
                             int64_t sT, double* ws) {
  if (m < n || n < 1 || nb < 1) return SLRA_ERR_INVALID_ARGUMENT;
  const int64_t sW = (int64_t)m * n, sV = (int64_t)n * n;
  double* W = ws;
  double* V = W + (size_t)nb * sW;
  double* sg = V + (size_t)nb * sV;                                      // nb x n unsorted norms
  int* order = reinterpret_cast<int*>(sg + (size_t)nb * n);              // nb x n (n doubles of room)
  int* flags = reinterpret_cast<int*>(sg + (size_t)nb * 2 * n);          // kJMaxSweeps + 1
  {
    int64_t g = ceil_div((int64_t)m * n + (int64_t)n * n, 256);
    if (g > cx->num_sms * 4) g = cx->num_sms * 4;
    SLRA_TIMED(cx, "svd_large", copy_identity_kernel<<<dim3((unsigned)g, nb), 256, 0, cx->stream>>>(
                                    A, lda, sA, m, n, W, sW, V, sV);)
    SLRA_CHECK_LAUNCH(cx);
  }
  SLRA_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * (kJMaxSweeps + 1), cx->stream));
  int per_sm = 0;
  SLRA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_global_kernel, kJT, 0));
  if (per_sm < 1) return SLRA_ERR_UNSUPPORTED;
  const int64_t tasks = (int64_t)nb * ((n + 1) / 2);
  int64_t G = ceil_div(tasks, kJT / 32);
  const int64_t gmax = (int64_t)per_sm * cx->num_sms;
  if (G > gmax) G = gmax;
  if (G < 1) G = 1;
  JacobiGlobalArgs args{W, m, sW, V, n, sV, m, n, nb, flags, flags + kJMaxSweeps, 0.0};
  const double tol = 16.0 * (double)m * kEpsL;
  args.tol2 = tol * tol;
  void* kargs[] = {&args};
  {
    KernelTimer kt(cx, "svd_large");
    SLRA_CUDA(cudaLaunchCooperativeKernel((const void*)jacobi_global_kernel, dim3((unsigned)G), dim3(kJT), kargs, 0,
                                          cx->stream));
  }
  SLRA_CHECK_LAUNCH(cx);
  const unsigned gw = (unsigned)ceil_div(n, 8);
  SLRA_TIMED(cx, "svd_large", col_norms_kernel<<<dim3(gw, nb), 256, 0, cx->stream>>>(W, m, sW, m, n, sg, n);)
  SLRA_CHECK_LAUNCH(cx);
  SLRA_TIMED(cx, "svd_large", rank_order_kernel<<<dim3((unsigned)ceil_div(n, 128), nb), 128, 0, cx->stream>>>(
                                  sg, n, n, order, sigma, sSig);)
  SLRA_CHECK_LAUNCH(cx);
  SLRA_TIMED(cx, "svd_large", svd_emit_kernel<<<dim3(gw, nb), 256, 0, cx->stream>>>(W, m, sW, V, n, sV, m, n, order,
                                                                                    sigma, sSig, S, lds, sS, T, ldt,
                                                                                    sT);)
  SLRA_CHECK_LAUNCH(cx);
  return SLRA_OK;
}

}  // namespace slra_dev
