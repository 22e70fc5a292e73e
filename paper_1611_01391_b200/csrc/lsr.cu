// K-d: sketched least squares (sketch_solve, lsr.cpp:37-67) and the residual
// pass (residual_norm, lsr.cpp:26-28).
//
// Device formulation: FW = F (A|b) through a compiled left plan (one pass,
// only the k sampled/sketched rows are touched), then two solvers:
//  * fast path — the Gram [FA Fb]^T [FA Fb] on the DMMA GEMM (split-K,
//    deterministic), a blocked Cholesky of FA^T FA in one CTA (right-looking,
//    32-column panels), two triangular solves, one step of iterative
//    refinement, and the sketched residual ||FA x - Fb|| by a direct pass.
//    It is taken only when the sketch is well conditioned: every Cholesky
//    pivot above 1e-6 of its column's squared norm (the sine of the angle
//    between a column and the span of the earlier ones above 1e-3), so that
//    the reference's rank() == d and one refinement step reaches ~eps.
//  * exact path — otherwise (near or exact dependence): Eigen's
//    ColPivHouseholderQR of FA itself (colpiv_lsq_kernel: first maximum of
//    the updated norms, xGEQP3 downdate, nonzero-pivot rule, rank() with
//    threshold 1e-10 → SketchRankFailure exactly where the reference throws,
//    lsr.cpp:52-55), Q^T Fb carried along as an extra column, and the solve
//    x = P R^-1 (Q^T Fb). The same kernel (without the rank test) gives R
//    and Q^T b for solve_exact's pseudo-inverse (lsr.cpp:21-24).
// One host synchronisation at the end of the fast path (status, residual).
#include <cstring>

#include "common.cuh"

namespace slra_dev {

int launch_sketch_rows(Context* c, const double* Wm, int64_t ldw, int64_t ncols, const int64_t* src,
                       const double* coef, const int32_t* q, int64_t width, int tree, int64_t k, double* out,
                       int64_t ldo);
int launch_gemm(Context* c, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
                int64_t lda, const double* B, int64_t ldb, double beta, double* Cm, int64_t ldc);

constexpr int kLT = 256;
constexpr int kPW = 32;  // Cholesky panel width

// In-place lower Cholesky of G (d x d, ld d, global/L2), one CTA,
// right-looking with 32-column panels. The panel is factorised in shared
// memory with one thread per row (no index arithmetic in the inner loops),
// written back, and the trailing lower triangle is updated
// G22 -= L21 L21^T with L21 read from shared memory.
// status[0] = 0 ok, 1 rank failure.
__global__ void __launch_bounds__(kLT) cholesky_kernel(double* __restrict__ G, int d, double tol_rel,
                                                       int32_t* __restrict__ status) {
  extern __shared__ __align__(16) double P[];  // rows x kPW panel, ld = d + 1 (odd: row-threads conflict-free)
  __shared__ int fail, illc;
  __shared__ double red[33];
  const int tid = threadIdx.x;
  const int ldp = d + 1;
  double* gdiag = P + (size_t)ldp * kPW;  // original diagonal ||FA(:,j)||^2
  double dm = 0.0;
  for (int i = tid; i < d; i += kLT) {
    gdiag[i] = G[i + (int64_t)i * d];
    dm = fmax(dm, gdiag[i]);
  }
  if (tid == 0) fail = illc = 0;
  // the rank floor from the largest squared column norm of FA (all d columns)
  {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
    if ((tid & 31) == 0) red[tid >> 5] = dm;
    __syncthreads();
    if (tid == 0) {
      double mx = 0.0;
      for (int w = 0; w < kLT / 32; ++w) mx = fmax(mx, red[w]);
      red[32] = mx;
    }
    __syncthreads();
  }
  const double tol2 = tol_rel * red[32];
  for (int p0 = 0; p0 < d; p0 += kPW) {
    const int pw = (d - p0) < kPW ? (d - p0) : kPW;
    const int rows = d - p0;
    for (int i = tid; i < rows; i += kLT) {  // all 32 loads of a row in flight at once
      double g[kPW];
      const double* gi = G + (p0 + i) + (int64_t)p0 * d;
#pragma unroll
      for (int c = 0; c < kPW; ++c) g[c] = load_sel(gi, (int64_t)c * d, c < pw && i >= c);
#pragma unroll
      for (int c = 0; c < kPW; ++c)
        if (c < pw) P[i + c * ldp] = g[c];
    }
    __syncthreads();
    // (a) the pw x pw diagonal block: thread (row ti, phase tc) owns L(ti, c)
    // for c = tc, tc + 8, ...; each column step stages its operands in registers
    // and writes after a barrier (no dependent shared-memory chains)
    {
      const int ti = tid & 31, tc = tid >> 5;  // 8 phases: columns tc, tc + 8, tc + 16, tc + 24
      for (int j = 0; j < pw; ++j) {
        const double piv = P[j + j * ldp];
        // rank failure: the pivot (squared distance of column j from the span
        // of the earlier ones) is non-positive, below the global floor, or
        // below 64 eps of the column's own squared norm — a column dependent
        // at the sqrt(eps) level, which is as fine as the Gram resolves
        if (!(piv > tol2) || !(piv > 64.0 * 2.220446049250313e-16 * gdiag[p0 + j])) {  // uniform
          if (tid == 0) fail = 1;
          break;
        }
        if (!(piv > 1e-6 * gdiag[p0 + j]) && tid == 0) illc = 1;  // leave to the exact path
        const double ljj = sqrt(piv);
        const double inv = 1.0 / ljj;
        const bool row = ti > j && ti < pw;
        const double lij = row ? P[ti + j * ldp] * inv : 0.0;
        double lcj[4], cur[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = tc + 8 * q;
          const bool act = row && c > j && c <= ti;
          lcj[q] = load_sel(P + c, (int64_t)j * ldp, act) * inv;
          cur[q] = load_sel(P + ti, (int64_t)c * ldp, act);
        }
        __syncthreads();
        if (tc == 0 && ti >= j && ti < pw) P[ti + j * ldp] = (ti == j) ? ljj : lij;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = tc + 8 * q;
          if (row && c > j && c <= ti) P[ti + c * ldp] = cur[q] - lij * lcj[q];
        }
        __syncthreads();
      }
    }
    __syncthreads();
    if (fail) break;
    // (b) rows below the block: L21(i, :) = A21(i, :) L11^-T, a thread per
    // row, right-looking in registers
    double* rdiag = gdiag + d;  // 1 / L(j, j) of this panel's block
    for (int c = tid; c < pw; c += kLT) rdiag[c] = 1.0 / P[c + c * ldp];
    __syncthreads();
    for (int i = pw + tid; i < rows; i += kLT) {
      double z[kPW];
#pragma unroll
      for (int c = 0; c < kPW; ++c) z[c] = load_sel(P + i, (int64_t)c * ldp, c < pw);
#pragma unroll
      for (int c = 0; c < kPW; ++c) {
        z[c] *= (c < pw) ? rdiag[c] : 0.0;
#pragma unroll
        for (int c2 = c + 1; c2 < kPW; ++c2) z[c2] = fma(-z[c], P[c2 + c * ldp], z[c2]);  // pw <= 32 < ld
      }
#pragma unroll
      for (int c = 0; c < kPW; ++c)
        if (c < pw) P[i + c * ldp] = z[c];
    }
    __syncthreads();
    for (int i = tid; i < rows; i += kLT) {  // a row per thread, unrolled over the panel
      double* gi = G + (p0 + i) + (int64_t)p0 * d;
#pragma unroll
      for (int c = 0; c < kPW; ++c)
        if (c < pw && i >= c) gi[(int64_t)c * d] = P[i + c * ldp];
    }
    // trailing lower triangle G22 -= L21 L21^T in 4 x 4 register tiles (16
    // independent FMA chains per thread; tiles on or below the diagonal)
    // thread (ti4, tc4) owns rows pw + ti4 + nt a and columns pw + tc4 + nt b
    // (a, b < 4): strided so a warp's row reads are consecutive (no bank
    // conflicts) and its column reads are broadcasts
    const int tr = rows - pw;
    const int nt = (tr + 3) / 4;
    for (int e = tid; e < nt * nt; e += kLT) {
      const int ti4 = e % nt, tc4 = e / nt;
      double acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
      for (int t = 0; t < pw; ++t) {
        const double* pt = P + t * ldp + pw;
        double li[4], lc[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          li[a] = load_sel(pt, ti4 + nt * a, ti4 + nt * a < tr);
          lc[a] = load_sel(pt, tc4 + nt * a, tc4 + nt * a < tr);
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fma(li[a], lc[b], acc[a][b]);
      }
      // read all 16 targets first (unconditional, clamped), then store: a
      // guarded read-modify-write would serialise the L2 latencies
      double gv[4][4];
      double* gbase = G + (p0 + pw) + (int64_t)(p0 + pw) * d;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int i = ti4 + nt * a, c = tc4 + nt * b;
          const bool ok = i < tr && c <= i;
          gv[a][b] = gbase[ok ? i + (int64_t)c * d : 0];
        }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int i = ti4 + nt * a, c = tc4 + nt * b;
          if (i < tr && c <= i) gbase[i + (int64_t)c * d] = gv[a][b] - acc[a][b];
        }
    }
    __syncthreads();
  }
  if (tid == 0) {
    status[0] = fail;
    status[1] = illc;
  }
}

// x (+)= (L L^T)^{-1} rhs for the lower Cholesky factor L (ld d), one CTA,
// by 32-wide blocks: one warp solves the diagonal block with shuffles (lane
// i holds entry i; per step a multiply, a broadcast and an FMA), then the
// whole CTA applies the block to the remaining entries (a GEMV). 2 d / 32
// barriers per solve instead of 2 d.
constexpr int kST = 256;
constexpr int kSB = 32;
__global__ void __launch_bounds__(kST) chol_solve_kernel(const double* __restrict__ L, int d,
                                                         const double* __restrict__ rhs, double* __restrict__ x,
                                                         const int32_t* __restrict__ status, int accumulate) {
  extern __shared__ __align__(16) double v[];  // d
  if (*status) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < d; i += kST) v[i] = rhs[i];
  __syncthreads();
  // forward: L y = rhs
  for (int b0 = 0; b0 < d; b0 += kSB) {
    const int bw = (d - b0) < kSB ? (d - b0) : kSB;
    if (warp == 0) {
      const bool in = lane < bw;
      double lrow[kSB];  // L(b0 + lane, b0 + c)
#pragma unroll
      for (int c = 0; c < kSB; ++c) lrow[c] = load_sel(L + (b0 + lane), (int64_t)(b0 + c) * d, in && c < lane);
      const double rd = in ? 1.0 / L[(b0 + lane) + (int64_t)(b0 + lane) * d] : 0.0;
      double yi = in ? v[b0 + lane] : 0.0;
#pragma unroll
      for (int c = 0; c < kSB; ++c) {
        if (lane == c) yi *= rd;
        const double yc = __shfl_sync(0xffffffffu, yi, c);
        if (lane > c) yi = fma(-lrow[c], yc, yi);
      }
      if (in) v[b0 + lane] = yi;
    }
    __syncthreads();
    for (int i = b0 + bw + tid; i < d; i += kST) {  // v(i) -= L(i, block) y(block)
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int c = 0; c < kSB; c += 2) {
        a0 = fma(load_sel(L + i, (int64_t)(b0 + c) * d, c < bw), v[b0 + (c < bw ? c : 0)], a0);
        a1 = fma(load_sel(L + i, (int64_t)(b0 + c + 1) * d, c + 1 < bw), v[b0 + (c + 1 < bw ? c + 1 : 0)], a1);
      }
      v[i] -= a0 + a1;
    }
    __syncthreads();
  }
  // backward: L^T x = y
  for (int b1 = d; b1 > 0; b1 -= kSB) {
    const int b0 = b1 - kSB > 0 ? b1 - kSB : 0;
    const int bw = b1 - b0;
    if (warp == 0) {
      const bool in = lane < bw;
      double lcol[kSB];  // L(b0 + c, b0 + lane) = L^T(b0 + lane, b0 + c)
#pragma unroll
      for (int c = 0; c < kSB; ++c)
        lcol[c] = load_sel(L + (int64_t)(b0 + lane) * d, (int64_t)(b0 + c), in && c < bw && c > lane);
      const double rd = in ? 1.0 / L[(b0 + lane) + (int64_t)(b0 + lane) * d] : 0.0;
      double xi = in ? v[b0 + lane] : 0.0;
#pragma unroll
      for (int c = kSB - 1; c >= 0; --c) {
        if (c < bw) {
          if (lane == c) xi *= rd;
          const double xc = __shfl_sync(0xffffffffu, xi, c);
          if (lane < c) xi = fma(-lcol[c], xc, xi);
        }
      }
      if (in) v[b0 + lane] = xi;
    }
    __syncthreads();
    for (int i = tid; i < b0; i += kST) {  // v(i) -= L(block, i)^T x(block)
      double a0 = 0.0, a1 = 0.0;
      const double* li = L + (int64_t)i * d + b0;  // column i of L, rows b0..
#pragma unroll
      for (int c = 0; c < kSB; c += 2) {
        a0 = fma(load_sel(li, c, c < bw), v[b0 + (c < bw ? c : 0)], a0);
        a1 = fma(load_sel(li, c + 1, c + 1 < bw), v[b0 + (c + 1 < bw ? c + 1 : 0)], a1);
      }
      v[i] -= a0 + a1;
    }
    __syncthreads();
  }
  for (int i = tid; i < d; i += kST) x[i] = accumulate ? x[i] + v[i] : v[i];
}

// r = Fb - FA x (k rows) and the squared-norm partials: 32 rows x 8 column
// groups per CTA, combined in shared memory.
__global__ void __launch_bounds__(256) lsq_residual_kernel(const double* __restrict__ FW, int64_t k, int d,
                                                           const double* __restrict__ x, double* __restrict__ r,
                                                           double* __restrict__ part) {
  __shared__ double red[8][33];
  __shared__ double red2[40];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int64_t i = blockIdx.x * 32LL + lane;
  double acc = 0.0;
  if (i < k)
    for (int j = grp; j < d; j += 8) acc = fma(FW[i + (int64_t)j * k], x[j], acc);
  red[grp][lane] = acc;
  __syncthreads();
  double s = 0.0;
  if (grp == 0 && i < k) {
    double a = 0.0;
#pragma unroll
    for (int g = 0; g < 8; ++g) a += red[g][lane];
    const double e = FW[i + (int64_t)d * k] - a;
    r[i] = e;
    s = e * e;
  }
  s = block_sum<256>(s, red2);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// out[b] = sum of part[b n .. b n + n) (one CTA per sum, fixed order)
__global__ void sum_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double red[40];
  double s = 0.0;
  part += (int64_t)blockIdx.x * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// ||A x_s - b||^2 for NX solutions x_s (columns of X, ld d) over a tall
// column-major A (m x d) in ONE pass over A: each thread owns two rows and
// walks the d columns with 128-bit loads (coalesced across the warp);
// deterministic per-CTA partials part[s * gridDim.x + cta].
template <int NX>
__global__ void __launch_bounds__(256) lsr_residual_kernel(const double* __restrict__ A, int64_t lda, int64_t m,
                                                           int d, const double* __restrict__ b,
                                                           const double* __restrict__ X, double* __restrict__ part) {
  extern __shared__ double xs[];  // xs[j * NX + s]
  __shared__ double red[40];
  for (int e = threadIdx.x; e < d * NX; e += blockDim.x) xs[(e % d) * NX + e / d] = X[e];
  __syncthreads();
  double sq[NX];
#pragma unroll
  for (int s = 0; s < NX; ++s) sq[s] = 0.0;
  const bool vec = (lda % 2 == 0) && (((uintptr_t)A) % 16 == 0);
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x * 2; i0 < m; i0 += (int64_t)gridDim.x * blockDim.x * 2) {
    const int64_t i = i0 + 2 * threadIdx.x;
    if (i + 1 < m && vec) {
      double a0[NX], a1[NX];
#pragma unroll
      for (int s = 0; s < NX; ++s) a0[s] = a1[s] = 0.0;
      const double2* col = reinterpret_cast<const double2*>(A + i);
      // batches of kRB columns: every load of a batch is issued before its
      // FMAs (ncu: long-scoreboard stalls with the loads interleaved)
      constexpr int kRB = 12;
      for (int j0 = 0; j0 < d; j0 += kRB) {
        double2 v[kRB];
#pragma unroll
        for (int u = 0; u < kRB; ++u) v[u] = __ldg(col + (int64_t)(j0 + u < d ? j0 + u : j0) * (lda / 2));
#pragma unroll
        for (int u = 0; u < kRB; ++u) {
          if (j0 + u < d) {
#pragma unroll
            for (int s = 0; s < NX; ++s) {
              const double xv = xs[(j0 + u) * NX + s];
              a0[s] = fma(v[u].x, xv, a0[s]);
              a1[s] = fma(v[u].y, xv, a1[s]);
            }
          }
        }
      }
      const double b0 = b[i], b1 = b[i + 1];
#pragma unroll
      for (int s = 0; s < NX; ++s) {
        const double e0 = a0[s] - b0, e1 = a1[s] - b1;
        sq[s] += e0 * e0 + e1 * e1;
      }
    } else {
      for (int64_t ii = i; ii < i + 2 && ii < m; ++ii) {
#pragma unroll
        for (int s = 0; s < NX; ++s) {
          double a0 = 0.0;
          for (int j = 0; j < d; ++j) a0 += A[ii + (int64_t)j * lda] * xs[j * NX + s];
          const double e0 = a0 - b[ii];
          sq[s] += e0 * e0;
        }
      }
    }
  }
#pragma unroll
  for (int s = 0; s < NX; ++s) {
    const double t = block_sum<256>(sq[s], red);
    if (threadIdx.x == 0) part[(int64_t)s * gridDim.x + blockIdx.x] = t;
  }
}

int launch_lsr_residual_multi(Context* c, const double* A, int64_t lda, int64_t m, int64_t d, const double* b,
                              const double* X, int nx, double* d_out) {
  if (nx < 1 || nx > 4) return SLRA_ERR_INVALID_ARGUMENT;
  int grid = c->num_sms * 4;
  const int64_t need = (m + 511) / 512;
  if (need < grid) grid = (int)(need > 0 ? need : 1);
  double* part = partials(c, grid * nx);
  if (!part) return SLRA_ERR_CUDA;
  const size_t sm = sizeof(double) * d * nx;
  switch (nx) {
    case 1: SLRA_TIMED(c, "lsr_residual", lsr_residual_kernel<1><<<grid, 256, sm, c->stream>>>(A, lda, m, (int)d, b, X, part);) break;
    case 2: SLRA_TIMED(c, "lsr_residual", lsr_residual_kernel<2><<<grid, 256, sm, c->stream>>>(A, lda, m, (int)d, b, X, part);) break;
    case 3: SLRA_TIMED(c, "lsr_residual", lsr_residual_kernel<3><<<grid, 256, sm, c->stream>>>(A, lda, m, (int)d, b, X, part);) break;
    default: SLRA_TIMED(c, "lsr_residual", lsr_residual_kernel<4><<<grid, 256, sm, c->stream>>>(A, lda, m, (int)d, b, X, part);) break;
  }
  SLRA_CHECK_LAUNCH(c);
  SLRA_TIMED(c, "reduce", sum_kernel<<<nx, 256, 0, c->stream>>>(part, grid, d_out);)
  SLRA_CHECK_LAUNCH(c);
  return SLRA_OK;
}

int launch_lsr_residual(Context* c, const double* A, int64_t lda, int64_t m, int64_t d, const double* b,
                        const double* x, double* d_out) {
  return launch_lsr_residual_multi(c, A, lda, m, d, b, x, 1, d_out);
}

}  // namespace slra_dev

using namespace slra_dev;

extern "C" {

int slra_lsr_residual(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t d, const double* b,
                      const double* x, double* d_out) {
  if (!ctx || lda < m || d < 1 || d > 4096) return SLRA_ERR_INVALID_ARGUMENT;
  return launch_lsr_residual(C(ctx), A, lda, m, d, b, x, d_out);
}

int slra_lsr_residual_multi(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t d, const double* b,
                            const double* X, int64_t nx, double* d_out) {
  if (!ctx || lda < m || d < 1 || d > 4096 || nx < 1 || nx > 4) return SLRA_ERR_INVALID_ARGUMENT;
  return launch_lsr_residual_multi(C(ctx), A, lda, m, d, b, X, (int)nx, d_out);
}

}  // extern "C"

namespace slra_dev {

// Eigen ColPivHouseholderQR (linalg.cpp restated in oracle/src/linalg.cpp:
// computeInPlace with the LAPACK xGEQP3 norm downdate) of W(:, 0:d) for a
// k x (d+1) column-major W in global memory (L2-resident), the last column
// receiving every reflector (Q^T b). One CTA of kQT threads: block argmax
// for the pivot (first maximum in position order), block reduction for the
// reflector, a warp per trailing column for its update and norm downdate.
// On exit W holds R (and the essential parts), hc the taus, perm the column
// permutation (position -> original column), piv[0] = the nonzero-pivot
// count, piv[1] = max |R_ii|. Then, with `solve` set: the rank with
// threshold 1e-10 (rank() < d -> status SketchRankFailure, the reference's
// throw, lsr.cpp:52-55), otherwise x = P R^-1 (Q^T b)(0:d).
constexpr int kQT = 1024;
__global__ void __launch_bounds__(kQT) colpiv_lsq_kernel(double* __restrict__ W, int64_t k, int d,
                                                         double* __restrict__ nu, double* __restrict__ nd,
                                                         int* __restrict__ perm, double* __restrict__ hc,
                                                         double* __restrict__ piv, int solve, double* __restrict__ x,
                                                         int32_t* __restrict__ status) {
  __shared__ double rv[33];
  __shared__ int64_t ri[33];
  __shared__ double sc[4];
  __shared__ int s_nonzero;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kQT / 32;
  const double eps = 2.220446049250313e-16, sqrt_eps = 1.4901161193847656e-08;
  for (int c = warp; c < d; c += NW) {
    double acc = 0.0;
    for (int64_t i = lane; i < k; i += 32) acc = fma(W[i + c * k], W[i + c * k], acc);
    acc = warp_sum(acc);
    if (lane == 0) nu[c] = nd[c] = sqrt(acc);
  }
  for (int c = tid; c < d; c += kQT) perm[c] = c;
  __syncthreads();
  double maxnorm = 0.0;
  {
    ArgMax a{-1.0, INT64_MAX};
    for (int c = tid; c < d; c += kQT) a = argmax_merge(a, ArgMax{nu[c], c});
    maxnorm = block_argmax<kQT>(a, rv, ri).v;
  }
  const double thr_helper = (maxnorm * eps) * (maxnorm * eps) / (double)k;
  const int size = (int64_t)d < k ? d : (int)k;
  if (tid == 0) {
    s_nonzero = size;
    sc[3] = 0.0;  // max |beta|
  }
  for (int j = 0; j < size; ++j) {
    ArgMax a{-1.0, INT64_MAX};
    for (int c = j + tid; c < d; c += kQT) a = argmax_merge(a, ArgMax{nu[c], c});
    a = block_argmax<kQT>(a, rv, ri);
    const int big = (int)a.i;
    if (tid == 0 && s_nonzero == size && a.v * a.v < thr_helper * (double)(k - j)) s_nonzero = j;
    if (big != j) {
      for (int64_t i = tid; i < k; i += kQT) {
        const double t = W[i + j * k];
        W[i + j * k] = W[i + big * k];
        W[i + big * k] = t;
      }
      if (tid == 0) {
        double t = nu[j]; nu[j] = nu[big]; nu[big] = t;
        t = nd[j]; nd[j] = nd[big]; nd[big] = t;
        const int p = perm[j]; perm[j] = perm[big]; perm[big] = p;
      }
    }
    __syncthreads();
    // reflector of column j, rows j..k-1 (Eigen makeHouseholder)
    double* xj = W + j * k;
    double tl = 0.0;
    for (int64_t i = j + 1 + tid; i < k; i += kQT) tl = fma(xj[i], xj[i], tl);
    tl = block_sum<kQT>(tl, rv);
    const double c0 = xj[j];
    double tau, beta;
    if (tl <= DBL_MIN) {
      tau = 0.0;
      beta = c0;
      for (int64_t i = j + 1 + tid; i < k; i += kQT) xj[i] = 0.0;
    } else {
      beta = sqrt(c0 * c0 + tl);
      if (c0 >= 0.0) beta = -beta;
      const double den = c0 - beta;
      for (int64_t i = j + 1 + tid; i < k; i += kQT) xj[i] /= den;
      tau = (beta - c0) / beta;
    }
    __syncthreads();
    if (tid == 0) {
      xj[j] = beta;
      hc[j] = tau;
      sc[3] = fmax(sc[3], fabs(beta));
    }
    // apply to columns j+1 .. d (the last is b), a warp per column; then the
    // xGEQP3 downdate of the column norms (re-computed when it cancels)
    for (int c = j + 1 + warp; c <= d; c += NW) {
      double* xc = W + (int64_t)c * k;
      if (k - j == 1) {
        if (lane == 0) xc[j] *= (1.0 - tau);
      } else if (tau != 0.0) {
        double w = 0.0;
        for (int64_t i = j + 1 + lane; i < k; i += 32) w = fma(xj[i], xc[i], w);
        w = warp_sum(w) + xc[j];
        if (lane == 0) xc[j] -= tau * w;
        for (int64_t i = j + 1 + lane; i < k; i += 32) xc[i] -= tau * xj[i] * w;
      }
      if (c < d) {
        __syncwarp();
        const double nuv = nu[c];
        if (nuv != 0.0) {
          double temp = fabs(xc[j]) / nuv;
          temp = (1.0 + temp) * (1.0 - temp);
          temp = temp < 0.0 ? 0.0 : temp;
          const double ratio = nuv / nd[c];
          if (temp * ratio * ratio <= sqrt_eps) {
            double acc = 0.0;
            for (int64_t i = j + 1 + lane; i < k; i += 32) acc = fma(xc[i], xc[i], acc);
            acc = warp_sum(acc);
            if (lane == 0) nu[c] = nd[c] = sqrt(acc);
          } else if (lane == 0) {
            nu[c] = nuv * sqrt(temp);
          }
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    piv[0] = (double)s_nonzero;
    piv[1] = sc[3];
  }
  if (!solve) return;
  // rank() with threshold 1e-10 over the nonzero pivots
  if (tid == 0) {
    const double pre = sc[3] * 1e-10;
    int rank = 0;
    for (int i = 0; i < s_nonzero; ++i) rank += fabs(W[i + (int64_t)i * k]) > pre ? 1 : 0;
    *status = rank < d ? SLRA_ERR_SKETCH_RANK_FAILURE : SLRA_OK;
    sc[0] = rank < d ? 1.0 : 0.0;
  }
  __syncthreads();
  if (sc[0] != 0.0) return;
  // back substitution R y = (Q^T b)(0:d), column-oriented, then x(perm) = y
  double* cvec = W + (int64_t)d * k;  // Q^T b
  for (int t = d - 1; t >= 0; --t) {
    if (tid == 0) cvec[t] /= W[t + (int64_t)t * k];
    __syncthreads();
    const double yt = cvec[t];
    for (int i = tid; i < t; i += kQT) cvec[i] -= W[i + (int64_t)t * k] * yt;
    __syncthreads();
  }
  for (int i = tid; i < d; i += kQT) x[perm[i]] = cvec[i];
}

int launch_colpiv_lsq(Context* cx, double* W, int64_t k, int d, double* ws, int solve, double* x, int32_t* status) {
  double* nu = ws;
  double* nd = nu + d;
  double* hc = nd + d;
  double* piv = hc + d;
  int* perm = reinterpret_cast<int*>(piv + 2);
  SLRA_TIMED(cx, "lsr_exact_qr", colpiv_lsq_kernel<<<1, kQT, 0, cx->stream>>>(W, k, d, nu, nd, perm, hc, piv, solve, x,
                                                                             status);)
  SLRA_CHECK_LAUNCH(cx);
  return SLRA_OK;
}

// Eigen CompleteOrthogonalDecomposition pseudo-inverse, primitive_cur's
// qr_nucleus branch (cur.cpp:146-152), restated in oracle/src/linalg.cpp
// (cod_pseudo_inverse). Runs after colpiv_lsq_kernel(solve = 0) left the
// ColPivQR of G (k x l) in W (+ taus, permutation, nonzero-pivot count and
// max pivot). One CTA, W in global memory (L2-resident; generators are
// small): the RZ step at the DEFAULT rank r_e (the constructor's), then
// pinv = P Z^T [T11^-1 (Q^T I)(0:r_t, :); 0] at the thresholded rank r_t
// (setThreshold, read by rank() and pseudoInverse()), exactly the order in
// which Eigen applies them. Warps own columns (left reflectors) or rows
// (right reflectors); one __syncthreads between dependent steps.
constexpr int kCT = 256;
__global__ void __launch_bounds__(kCT) cod_pinv_kernel(double* __restrict__ W, int k, int l,
                                                       const double* __restrict__ hc, const int* __restrict__ perm,
                                                       const double* __restrict__ piv, double threshold,
                                                       double* __restrict__ zc, double* __restrict__ Cw,
                                                       double* __restrict__ D, double* __restrict__ P, int64_t ldp,
                                                       int32_t* __restrict__ rank_out) {
  __shared__ double red[33];
  __shared__ int s_r[2];
  __shared__ double s_h[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kCT / 32;
  const int size = k < l ? k : l;
  if (tid == 0) {
    const int nz = (int)piv[0];
    const double pre_e = fabs(piv[1]) * (2.220446049250313e-16 * (double)size);
    const double pre_t = fabs(piv[1]) * threshold;
    int re = 0, rt = 0;
    for (int i = 0; i < nz; ++i) {
      const double a = fabs(W[i + (int64_t)i * k]);
      re += a > pre_e;
      rt += a > pre_t;
    }
    s_r[0] = re;
    s_r[1] = rt;
    *rank_out = rt;
  }
  for (int i = tid; i < size; i += kCT) zc[i] = 0.0;
  __syncthreads();
  const int re = s_r[0], rt = s_r[1];
  auto X = [&](int i, int j) -> double& { return W[i + (int64_t)j * k]; };
  // ---- RZ: [R11 R12] = [T11 0] Z at rank r_e (computeInPlace)
  if (re < l) {
    const int len = l - re + 1, c0 = re - 1;
    for (int kk = re - 1; kk >= 0; --kk) {
      if (kk != re - 1)
        for (int i = tid; i <= kk; i += kCT) {
          const double t = X(i, kk);
          X(i, kk) = X(i, c0);
          X(i, c0) = t;
        }
      __syncthreads();
      // makeHouseholderInPlace on row kk, columns c0 .. l-1
      double tl = 0.0;
      for (int j = 1 + tid; j < len; j += kCT) tl = fma(X(kk, c0 + j), X(kk, c0 + j), tl);
      tl = block_sum<kCT>(tl, red);
      const double x0 = X(kk, c0);
      double tau, beta;
      if (tl <= DBL_MIN) {
        tau = 0.0;
        beta = x0;
      } else {
        beta = sqrt(x0 * x0 + tl);
        if (x0 >= 0.0) beta = -beta;
        tau = (beta - x0) / beta;
      }
      __syncthreads();
      if (tl <= DBL_MIN) {
        for (int j = 1 + tid; j < len; j += kCT) X(kk, c0 + j) = 0.0;
      } else {
        const double den = x0 - beta;
        for (int j = 1 + tid; j < len; j += kCT) X(kk, c0 + j) /= den;
      }
      __syncthreads();
      if (tid == 0) {
        zc[kk] = tau;
        X(kk, c0) = beta;
      }
      // applyHouseholderOnTheRight to rows 0..kk-1, columns c0 .. l-1
      if (kk > 0 && tau != 0.0) {
        for (int i = warp; i < kk; i += NW) {
          double t = 0.0;
          for (int j = 1 + lane; j < len; j += 32) t = fma(X(i, c0 + j), X(kk, c0 + j), t);
          t = warp_sum(t) + X(i, c0);
          __syncwarp();
          if (lane == 0) X(i, c0) -= tau * t;
          for (int j = 1 + lane; j < len; j += 32) X(i, c0 + j) -= tau * t * X(kk, c0 + j);
        }
      }
      __syncthreads();
      if (kk != re - 1)
        for (int i = tid; i <= kk; i += kCT) {
          const double t = X(i, kk);
          X(i, kk) = X(i, c0);
          X(i, c0) = t;
        }
      __syncthreads();
    }
  }
  // ---- D (l x k) = pinv
  for (int64_t e = tid; e < (int64_t)l * k; e += kCT) D[e] = 0.0;
  if (rt == 0) {
    __syncthreads();
    for (int64_t e = tid; e < (int64_t)l * k; e += kCT) P[(e % l) + (e / l) * ldp] = 0.0;
    return;
  }
  // c = H_{rt-1} ... H_0 I (k x k), a warp per column
  for (int64_t e = tid; e < (int64_t)k * k; e += kCT) Cw[e] = (e % k) == (e / k) ? 1.0 : 0.0;
  __syncthreads();
  for (int j = 0; j < rt; ++j) {
    const double tau = hc[j];
    const double* ess = W + j + (int64_t)j * k;  // ess[1 .. k-j)
    for (int c = warp; c < k; c += NW) {
      double* xc = Cw + j + (int64_t)c * k;
      if (k - j == 1) {
        if (lane == 0) xc[0] *= (1.0 - tau);
      } else if (tau != 0.0) {
        double w = 0.0;
        for (int i = 1 + lane; i < k - j; i += 32) w = fma(ess[i], xc[i], w);
        w = warp_sum(w) + xc[0];
        __syncwarp();
        if (lane == 0) xc[0] -= tau * w;
        for (int i = 1 + lane; i < k - j; i += 32) xc[i] -= tau * ess[i] * w;
      }
    }
    __syncthreads();
  }
  // T11 z = c(0:rt, :): a thread per right-hand side
  for (int c = tid; c < k; c += kCT) {
    for (int i = rt - 1; i >= 0; --i) {
      double sacc = Cw[i + (int64_t)c * k];
      for (int t = i + 1; t < rt; ++t) sacc -= X(i, t) * D[t + (int64_t)c * l];
      D[i + (int64_t)c * l] = sacc / X(i, i);
    }
  }
  __syncthreads();
  // applyZAdjointOnTheLeftInPlace at rank r_t: Z(0) first
  if (rt < l) {
    const int len = l - rt + 1, r0 = rt - 1;
    for (int kk = 0; kk < rt; ++kk) {
      const double tau = zc[kk];
      for (int c = warp; c < k; c += NW) {
        double* dc = D + (int64_t)c * l;
        if (lane == 0 && kk != rt - 1) {
          const double t = dc[kk];
          dc[kk] = dc[r0];
          dc[r0] = t;
        }
        __syncwarp();
        if (tau != 0.0) {
          double w = 0.0;
          for (int j = 1 + lane; j < len; j += 32) w = fma(X(kk, r0 + j), dc[r0 + j], w);
          w = warp_sum(w) + dc[r0];
          __syncwarp();
          if (lane == 0) dc[r0] -= tau * w;
          for (int j = 1 + lane; j < len; j += 32) dc[r0 + j] -= tau * X(kk, r0 + j) * w;
        }
        __syncwarp();
        if (lane == 0 && kk != rt - 1) {
          const double t = dc[kk];
          dc[kk] = dc[r0];
          dc[r0] = t;
        }
      }
      __syncthreads();
    }
  }
  // x = P y
  for (int64_t e = tid; e < (int64_t)l * k; e += kCT) {
    const int i = (int)(e % l), c = (int)(e / l);
    P[perm[i] + (int64_t)c * ldp] = D[e];
  }
}

// Solve min ||FA x - Fb|| for a sketched system FW = (FA | Fb) (k x (d+1),
// ld k). FW == nullptr: the caller has already written FW into the arena
// (returned through *fw_slot when fw_slot != nullptr on a first call).
// fallback = 0: return SLRA_ERR_UNSUPPORTED instead of running the exact
// path when the fast path declines (the caller has its own).
int launch_gram_tn(Context* c, const char* fam, int64_t m, int64_t n, int64_t K, double alpha, const double* X,
                   int64_t ldx, const double* Y, int64_t ldy, double beta, double* Cm, int64_t ldc, int lower);
int launch_chol_cluster(Context* c, const double* Gw, int d, const double* FW, int64_t k, double tol_rel, double* x,
                        double* ws, double* out, int32_t* status);
size_t lsr_cluster_ws_doubles(int d, int64_t k, int num_sms);
int launch_gram_tn_batched(Context* c, const char* fam, int nb, int64_t m, int64_t n, int64_t K, double alpha,
                           const double* X, int64_t ldx, int64_t sX, const double* Y, int64_t ldy, int64_t sY,
                           double beta, double* Cm, int64_t ldc, int64_t sC, int lower);
int launch_chol_cluster_batched(Context* c, int nprob, const double* const* Gw, int d, const double* const* FW,
                                int64_t k, double tol_rel, double* const* x, double* const* ws, double* const* out,
                                int32_t* const* status);
static int lsr_exact(Context* cx, const double* FW, int64_t k, int64_t d, double* x_hat, double* h_sketched_residual,
                     double* r, double* part, double* out, int rgrid);

static int lsr_solve(Context* cx, const double* FWext, int64_t k, int64_t d, double* x_hat,
                     double* h_sketched_residual, double** fw_slot, int fallback = 1) {
  const int64_t dc = d + 1;
  const int rgrid = (int)((k + 31) / 32);  // lsq_residual_kernel: 32 rows per CTA
  // arena 2: FW (k x dc) | Gw (dc x dc) | G (d x d) | g (d) | r (k) | c (d) | y (2d) | part | out
  const bool cluster = d <= 256 && k <= (int64_t)1 << 16;
  const size_t need = (size_t)k * dc + (size_t)dc * dc + (size_t)d * d + 4 * (size_t)d + (size_t)k + rgrid + 16 +
                      (cluster ? lsr_cluster_ws_doubles((int)d, k, cx->num_sms) + 2 : 0);
  double* ws = static_cast<double*>(arena(cx, 2, sizeof(double) * need));
  if (!ws) return SLRA_ERR_CUDA;
  double* FW = ws;
  double* Gw = FW + (size_t)k * dc;
  double* G = Gw + (size_t)dc * dc;
  double* g = G + (size_t)d * d;
  double* cvec = g + d;
  double* y = cvec + d;
  double* r = y + 2 * d;
  double* part = r + k;
  double* out = part + rgrid;
  int32_t* d_status = static_cast<int32_t*>(cx->dsmall);
  cudaStream_t st = cx->stream;
  if (fw_slot) {
    *fw_slot = FW;
    return SLRA_OK;
  }
  if (FWext) SLRA_CUDA(cudaMemcpyAsync(FW, FWext, 8 * (size_t)k * dc, cudaMemcpyDeviceToDevice, st));
  double* hs = static_cast<double*>(cx->hsmall);
  if (cluster) {
    // ---- cluster fast path (lsr_cluster.cu): the augmented Gram's lower
    // tiles on DMMA, then Cholesky + solve + one refinement step on one
    // 8-CTA cluster; no host synchronisation before the status read-back
    int gs = launch_gram_tn(cx, "gemm", dc, dc, k, 1.0, FW, k, FW, k, 0.0, Gw, dc, 1);
    if (gs == SLRA_ERR_UNSUPPORTED) gs = launch_gemm(cx, 1, 0, dc, dc, k, 1.0, FW, k, FW, k, 0.0, Gw, dc);
    SLRA_TRY(gs);
    double* lws = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(out + 16) + 15) & ~(uintptr_t)15);
    SLRA_TRY(launch_chol_cluster(cx, Gw, (int)d, FW, k, 1e-20, x_hat, lws, out, d_status));
    SLRA_CUDA(cudaMemcpyAsync(hs, out, 8, cudaMemcpyDeviceToHost, st));
    SLRA_CUDA(cudaMemcpyAsync(hs + 1, d_status, 8, cudaMemcpyDeviceToHost, st));
    SLRA_CUDA(cudaStreamSynchronize(st));
    const int32_t* hst = reinterpret_cast<const int32_t*>(hs + 1);
    if (hst[0] == 0 && hst[1] == 0) {
      if (h_sketched_residual) *h_sketched_residual = sqrt(hs[0]);
      return SLRA_OK;
    }
    if (!fallback) return SLRA_ERR_UNSUPPORTED;
    return lsr_exact(cx, FW, k, d, x_hat, h_sketched_residual, r, part, out, rgrid);
  }
  // ---- fast path: Gram [FA Fb]^T [FA Fb] (dc x dc); G = leading d x d block, g = FA^T Fb
  SLRA_TRY(launch_gemm(cx, 1, 0, dc, dc, k, 1.0, FW, k, FW, k, 0.0, Gw, dc));
  SLRA_CUDA(cudaMemcpy2DAsync(G, 8 * d, Gw, 8 * dc, 8 * d, d, cudaMemcpyDeviceToDevice, st));
  SLRA_CUDA(cudaMemcpyAsync(g, Gw + (size_t)d * dc, 8 * d, cudaMemcpyDeviceToDevice, st));
  const size_t smem = sizeof(double) * ((size_t)(d + 1) * kPW + (size_t)d + kPW);  // panel, diagonal, 1/L(j,j)
  SLRA_CUDA(cudaFuncSetAttribute(cholesky_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // rank floor (1e-10 max_i ||FA(:,i)||)^2 from the Gram diagonal on the device (all d columns)
  SLRA_TIMED(cx, "lsr_solve", cholesky_kernel<<<1, kLT, smem, st>>>(G, (int)d, 1e-20, d_status);)
  SLRA_CHECK_LAUNCH(cx);
  // x = G^{-1} g, then one refinement step x += G^{-1} FA^T (Fb - FA x)
  SLRA_TIMED(cx, "lsr_solve", chol_solve_kernel<<<1, kST, 8 * d, st>>>(G, (int)d, g, x_hat, d_status, 0);)
  SLRA_CHECK_LAUNCH(cx);
  SLRA_TIMED(cx, "lsr_solve", lsq_residual_kernel<<<rgrid, 256, 0, st>>>(FW, k, (int)d, x_hat, r, part);)
  SLRA_CHECK_LAUNCH(cx);
  SLRA_TRY(launch_gemm(cx, 1, 0, d, 1, k, 1.0, FW, k, r, k, 0.0, cvec, d));
  SLRA_TIMED(cx, "lsr_solve", chol_solve_kernel<<<1, kST, 8 * d, st>>>(G, (int)d, cvec, x_hat, d_status, 1);)
  SLRA_CHECK_LAUNCH(cx);
  // sketched residual ||FA x - Fb|| by a direct pass
  SLRA_TIMED(cx, "lsr_solve", lsq_residual_kernel<<<rgrid, 256, 0, st>>>(FW, k, (int)d, x_hat, r, part);)
  SLRA_CHECK_LAUNCH(cx);
  SLRA_TIMED(cx, "reduce", sum_kernel<<<1, 256, 0, st>>>(part, rgrid, out);)
  SLRA_CHECK_LAUNCH(cx);
  SLRA_CUDA(cudaMemcpyAsync(hs, out, 8, cudaMemcpyDeviceToHost, st));
  SLRA_CUDA(cudaMemcpyAsync(hs + 1, d_status, 8, cudaMemcpyDeviceToHost, st));
  SLRA_CUDA(cudaStreamSynchronize(st));
  const int32_t* hst = reinterpret_cast<const int32_t*>(hs + 1);
  if (hst[0] == 0 && hst[1] == 0) {
    if (h_sketched_residual) *h_sketched_residual = sqrt(hs[0]);
    return SLRA_OK;
  }
  if (!fallback) return SLRA_ERR_UNSUPPORTED;
  return lsr_exact(cx, FW, k, d, x_hat, h_sketched_residual, r, part, out, rgrid);
}

// ---- exact path (ill-conditioned or dependent sketch): the reference's
// ColPivHouseholderQR on a copy of FW, its rank rule, its solve
static int lsr_exact(Context* cx, const double* FW, int64_t k, int64_t d, double* x_hat, double* h_sketched_residual,
                     double* r, double* part, double* out, int rgrid) {
  const int64_t dc = d + 1;
  cudaStream_t st = cx->stream;
  int32_t* d_status = static_cast<int32_t*>(cx->dsmall);
  double* hs = static_cast<double*>(cx->hsmall);
  double* Wq = static_cast<double*>(arena(cx, 13, sizeof(double) * ((size_t)k * dc + 4 * (size_t)d + 64)));
  if (!Wq) return SLRA_ERR_CUDA;
  SLRA_CUDA(cudaMemcpyAsync(Wq, FW, 8 * (size_t)k * dc, cudaMemcpyDeviceToDevice, st));
  SLRA_TRY(launch_colpiv_lsq(cx, Wq, k, (int)d, Wq + (size_t)k * dc, 1, x_hat, d_status));
  SLRA_TIMED(cx, "lsr_solve", lsq_residual_kernel<<<rgrid, 256, 0, st>>>(FW, k, (int)d, x_hat, r, part);)
  SLRA_CHECK_LAUNCH(cx);
  SLRA_TIMED(cx, "reduce", sum_kernel<<<1, 256, 0, st>>>(part, rgrid, out);)
  SLRA_CHECK_LAUNCH(cx);
  SLRA_CUDA(cudaMemcpyAsync(hs, out, 8, cudaMemcpyDeviceToHost, st));
  SLRA_CUDA(cudaMemcpyAsync(hs + 1, d_status, 4, cudaMemcpyDeviceToHost, st));
  SLRA_CUDA(cudaStreamSynchronize(st));
  if (*reinterpret_cast<int32_t*>(hs + 1)) return SLRA_ERR_SKETCH_RANK_FAILURE;
  if (h_sketched_residual) *h_sketched_residual = sqrt(hs[0]);
  return SLRA_OK;
}

__global__ void upper_copy_kernel(const double* __restrict__ W, int64_t ldw, int d, double* __restrict__ R) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)d * d; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % d), j = (int)(e / d);
    R[e] = i <= j ? W[i + j * ldw] : 0.0;
  }
}
__global__ void perm_scatter_kernel(const double* __restrict__ y, const int* __restrict__ perm, int d,
                                    double* __restrict__ x) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d; i += gridDim.x * blockDim.x) x[perm[i]] = y[i];
}

}  // namespace slra_dev

extern "C" {

int slra_pinv(slra_ctx ctx, const double* d_A, int64_t lda, int64_t m, int64_t n, double rank_tol, double* d_P,
              int64_t ldp, int64_t* h_rank);

int slra_lsq_exact(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t d, const double* b, double* x,
                   int64_t* h_rank) {
  if (!ctx || lda < m || m <= d || d < 1) return SLRA_ERR_INVALID_ARGUMENT;
  if (d > 768) return SLRA_ERR_UNSUPPORTED;
  Context* cx = C(ctx);
  cudaStream_t st = cx->stream;
  double* FW = nullptr;
  SLRA_TRY(lsr_solve(cx, nullptr, m, d, nullptr, nullptr, &FW));
  SLRA_CUDA(cudaMemcpy2DAsync(FW, 8 * m, A, 8 * lda, 8 * m, d, cudaMemcpyDeviceToDevice, st));
  SLRA_CUDA(cudaMemcpyAsync(FW + (size_t)m * d, b, 8 * m, cudaMemcpyDeviceToDevice, st));
  // well-conditioned A: the normal-equation solve is pinv(A) b (full rank, every sigma above the cut)
  const int fs = lsr_solve(cx, nullptr, m, d, x, nullptr, nullptr, 0);
  if (fs == SLRA_OK) {
    if (h_rank) *h_rank = d;
    return SLRA_OK;
  }
  if (fs != SLRA_ERR_UNSUPPORTED) return fs;
  // otherwise pinv(A) b = Pi pinv(R) (Q^T b)(0:d) from the column-pivoted QR
  // A Pi = Q R (sigma(R) = sigma(A): the same 1e-10 cut as the reference's
  // SVD of A, linalg.cpp:111-121), the minimum-norm solution
  const size_t dc = (size_t)d + 1;
  double* Wq = static_cast<double*>(arena(cx, 13, sizeof(double) * ((size_t)m * dc + 4 * (size_t)d + 64)));
  double* R = static_cast<double*>(arena(cx, 9, sizeof(double) * (2 * (size_t)d * d + 2 * (size_t)d)));
  if (!Wq || !R) return SLRA_ERR_CUDA;
  double* P = R + (size_t)d * d;
  double* y = P + (size_t)d * d;
  SLRA_CUDA(cudaMemcpyAsync(Wq, FW, 8 * (size_t)m * dc, cudaMemcpyDeviceToDevice, st));
  double* qws = Wq + (size_t)m * dc;
  SLRA_TRY(launch_colpiv_lsq(cx, Wq, m, (int)d, qws, 0, nullptr, static_cast<int32_t*>(cx->dsmall)));
  upper_copy_kernel<<<64, 256, 0, st>>>(Wq, m, (int)d, R);
  SLRA_CHECK_LAUNCH(cx);
  SLRA_TRY(slra_pinv(ctx, R, d, d, d, 1e-10, P, d, h_rank));
  SLRA_TRY(launch_gemm(cx, 0, 0, d, 1, d, 1.0, P, d, Wq + (size_t)m * d, m, 0.0, y, d));
  const int* perm = reinterpret_cast<const int*>(qws + 3 * d + 2);
  perm_scatter_kernel<<<1, 256, 0, st>>>(y, perm, (int)d, x);
  SLRA_CHECK_LAUNCH(cx);
  return SLRA_OK;
}

int slra_cod_pinv(slra_ctx ctx, const double* G, int64_t ldg, int64_t k, int64_t l, double threshold, double* P,
                  int64_t ldp, int64_t* h_rank) {
  if (!ctx || k < 1 || l < 1 || ldg < k || ldp < l || !(threshold >= 0.0)) return SLRA_ERR_INVALID_ARGUMENT;
  if (k > 4096 || l > 4096) return SLRA_ERR_UNSUPPORTED;
  Context* cx = C(ctx);
  cudaStream_t st = cx->stream;
  // W = (G | 0): colpiv_lsq_kernel's layout (its extra column takes the reflectors)
  const size_t wq = (size_t)k * (l + 1), qws = 3 * (size_t)l + 4 + ((size_t)l + 1) / 2;
  const size_t need = wq + qws + (size_t)l + (size_t)k * k + (size_t)l * k;
  double* Wq = static_cast<double*>(arena(cx, 13, sizeof(double) * need));
  if (!Wq) return SLRA_ERR_CUDA;
  double* ws = Wq + wq;
  double* zc = ws + qws;
  double* Cw = zc + l;
  double* D = Cw + (size_t)k * k;
  SLRA_CUDA(cudaMemcpy2DAsync(Wq, 8 * k, G, 8 * ldg, 8 * k, l, cudaMemcpyDeviceToDevice, st));
  SLRA_CUDA(cudaMemsetAsync(Wq + (size_t)k * l, 0, 8 * k, st));
  int32_t* d_rank = static_cast<int32_t*>(cx->dsmall);
  SLRA_TRY(launch_colpiv_lsq(cx, Wq, k, (int)l, ws, 0, nullptr, d_rank));
  const double* hc = ws + 2 * l;
  const double* piv = hc + l;
  const int* perm = reinterpret_cast<const int*>(piv + 2);
  SLRA_TIMED(cx, "cod_pinv", cod_pinv_kernel<<<1, kCT, 0, st>>>(Wq, (int)k, (int)l, hc, perm, piv, threshold, zc, Cw, D,
                                                               P, ldp, d_rank);)
  SLRA_CHECK_LAUNCH(cx);
  if (h_rank) {
    int32_t* hs = static_cast<int32_t*>(cx->hsmall);
    SLRA_CUDA(cudaMemcpyAsync(hs, d_rank, 4, cudaMemcpyDeviceToHost, st));
    SLRA_CUDA(cudaStreamSynchronize(st));
    *h_rank = hs[0];
  }
  return SLRA_OK;
}

int slra_sketch_solve(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t d, const double* b,
                      const int64_t* src, const double* coef, const int32_t* q, int64_t width, int tree, int64_t k,
                      double* x_hat, double* h_sketched_residual) {
  if (!ctx || lda < m || m <= d || d < 1 || k <= d) return SLRA_ERR_INVALID_ARGUMENT;
  if (d > 768) return SLRA_ERR_UNSUPPORTED;
  Context* cx = C(ctx);
  double* FW = nullptr;
  SLRA_TRY(lsr_solve(cx, nullptr, k, d, nullptr, nullptr, &FW));
  // FW = F (A | b): one pass over the k sketched rows
  SLRA_TRY(launch_sketch_rows(cx, A, lda, d, src, coef, q, width, tree, k, FW, k));
  SLRA_TRY(launch_sketch_rows(cx, b, m, 1, src, coef, q, width, tree, k, FW + (size_t)k * d, k));
  return lsr_solve(cx, nullptr, k, d, x_hat, h_sketched_residual, nullptr);
}

// sketch_solve (lsr.cpp:37-67) for nsk <= 4 sketches F_s of the same (A, b)
// (config 4's two samplers): every F_s (A | b) gathered, every augmented
// Gram formed, then ONE launch of each cluster kernel runs all the solves
// side by side (a cluster per sketch) and one host synchronisation reads all
// statuses; a sketch that needs the reference's ColPivQR path takes it
// afterwards, alone. Same kernels and data as nsk separate calls, so the same
// bits (tests/test_gpu_config4.py).
int slra_sketch_solve_batched(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t d, const double* b,
                              int nsk, const int64_t* const* src, const double* const* coef,
                              const int32_t* const* q, const int64_t* width, const int* tree, int64_t k,
                              double* const* x_hat, double* h_sketched_residual) {
  if (!ctx || lda < m || m <= d || d < 1 || k <= d || nsk < 1) return SLRA_ERR_INVALID_ARGUMENT;
  if (d > 256 || k > ((int64_t)1 << 16) || nsk > 4) {
    for (int s = 0; s < nsk; ++s)
      SLRA_TRY(slra_sketch_solve(ctx, A, lda, m, d, b, src[s], coef[s], q[s], width[s], tree[s], k, x_hat[s],
                                 h_sketched_residual ? h_sketched_residual + s : nullptr));
    return SLRA_OK;
  }
  Context* cx = C(ctx);
  cudaStream_t st = cx->stream;
  const int64_t dc = d + 1;
  const int rgrid = (int)((k + 31) / 32);
  // per sketch: FW (k x dc) | Gw (dc x dc) | r (k) | part (rgrid) | out (16) | cluster ws (+2 for alignment)
  const size_t wsd = lsr_cluster_ws_doubles((int)d, k, cx->num_sms) + 2;
  const size_t per = ((size_t)k * dc + (size_t)dc * dc + (size_t)k + rgrid + 16 + wsd + 1) & ~(size_t)1;
  double* base = static_cast<double*>(arena(cx, 2, sizeof(double) * per * nsk + 64));
  if (!base) return SLRA_ERR_CUDA;
  const double* FWc[4];
  const double* Gwc[4];
  double *FW[4], *Gw[4], *r[4], *part[4], *out[4], *lws[4];
  int32_t* stt[4];
  for (int s = 0; s < nsk; ++s) {
    double* p0 = base + per * s;
    FW[s] = p0;
    Gw[s] = FW[s] + (size_t)k * dc;
    r[s] = Gw[s] + (size_t)dc * dc;
    part[s] = r[s] + k;
    out[s] = part[s] + rgrid;
    lws[s] = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(out[s] + 16) + 15) & ~(uintptr_t)15);
    stt[s] = static_cast<int32_t*>(cx->dsmall) + 2 * s;
    FWc[s] = FW[s];
    Gwc[s] = Gw[s];
    SLRA_TRY(launch_sketch_rows(cx, A, lda, d, src[s], coef[s], q[s], width[s], tree[s], k, FW[s], k));
    SLRA_TRY(launch_sketch_rows(cx, b, m, 1, src[s], coef[s], q[s], width[s], tree[s], k, FW[s] + (size_t)k * d, k));
  }
  // every sketch's augmented Gram in one launch (the sketches sit `per` apart)
  int gs = launch_gram_tn_batched(cx, "gemm", nsk, dc, dc, k, 1.0, FW[0], k, (int64_t)per, FW[0], k, (int64_t)per, 0.0,
                                  Gw[0], dc, (int64_t)per, 1);
  for (int s = 0; s < nsk && gs == SLRA_ERR_UNSUPPORTED; ++s) {
    const int g1 = launch_gemm(cx, 1, 0, dc, dc, k, 1.0, FW[s], k, FW[s], k, 0.0, Gw[s], dc);
    if (g1 != SLRA_OK) return g1;
    if (s == nsk - 1) gs = SLRA_OK;
  }
  SLRA_TRY(gs);
  SLRA_TRY(launch_chol_cluster_batched(cx, nsk, Gwc, (int)d, FWc, k, 1e-20, x_hat, lws, out, stt));
  double* hs = static_cast<double*>(cx->hsmall);  // [0..3] residuals, then the statuses
  for (int s = 0; s < nsk; ++s) SLRA_CUDA(cudaMemcpyAsync(hs + s, out[s], 8, cudaMemcpyDeviceToHost, st));
  SLRA_CUDA(cudaMemcpyAsync(hs + 4, cx->dsmall, 8 * nsk, cudaMemcpyDeviceToHost, st));
  SLRA_CUDA(cudaStreamSynchronize(st));
  double res[4];
  int32_t sts[8];
  for (int s = 0; s < nsk; ++s) res[s] = hs[s];
  std::memcpy(sts, hs + 4, 8 * nsk);
  for (int s = 0; s < nsk; ++s) {
    if (sts[2 * s] == 0 && sts[2 * s + 1] == 0) {
      if (h_sketched_residual) h_sketched_residual[s] = sqrt(res[s]);
      continue;
    }
    // the reference's ColPivHouseholderQR, its rank rule, its solve
    double one = 0.0;
    SLRA_TRY(lsr_exact(cx, FW[s], k, d, x_hat[s], &one, r[s], part[s], out[s], rgrid));
    if (h_sketched_residual) h_sketched_residual[s] = one;
  }
  return SLRA_OK;
}

int slra_lsr_solve_sketched(slra_ctx ctx, const double* FW, int64_t ldfw, int64_t k, int64_t d, double* x_hat,
                            double* h_sketched_residual) {
  if (!ctx || !FW || ldfw != k || k <= d || d < 1) return SLRA_ERR_INVALID_ARGUMENT;
  if (d > 768) return SLRA_ERR_UNSUPPORTED;
  return lsr_solve(C(ctx), FW, k, d, x_hat, h_sketched_residual, nullptr);
}

}  // extern "C"
