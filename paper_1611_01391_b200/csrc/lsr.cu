// K-d: sketched least squares (sketch_solve, lsr.cpp:37-67) and the residual
// pass (residual_norm, lsr.cpp:26-28).
//
// Device formulation: FW = F (A|b) through a compiled left plan (one pass,
// only the k sampled/sketched rows are touched), the Gram matrix
// [FA Fb]^T [FA Fb] on the DMMA GEMM (split-K, deterministic), a blocked
// Cholesky of FA^T FA in one CTA (right-looking, 32-column panels), two
// triangular solves, one step of iterative refinement, and the sketched
// residual ||FA x - Fb|| by a direct pass (never from the Gram identity).
// Rank test: a Cholesky pivot that is non-positive, below
// (1e-10 * max_i ||FA(:,i)||)^2, or below 64 eps ||FA(:,j)||^2 reports
// SketchRankFailure — the analogue of ColPivHouseholderQR's rank() < d with
// threshold 1e-10 (lsr.cpp:52-55). The Gram resolves dependence only to the
// sqrt(eps) level, so exactly dependent columns fail as in the reference,
// while sketches with sigma_min / sigma_max between 1e-10 and ~1e-7 also
// fail here (the reference solves those); DESIGN.md §8.
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
__global__ void __launch_bounds__(kLT) cholesky_kernel(double* __restrict__ G, int d, double tol2,
                                                       int32_t* __restrict__ status) {
  extern __shared__ __align__(16) double P[];  // rows x kPW panel, ld = d + 1 (odd: row-threads conflict-free)
  __shared__ int fail;
  const int tid = threadIdx.x;
  const int ldp = d + 1;
  double* gdiag = P + (size_t)ldp * kPW;  // original diagonal ||FA(:,j)||^2
  for (int i = tid; i < d; i += kLT) gdiag[i] = G[i + (int64_t)i * d];
  if (tid == 0) fail = 0;
  __syncthreads();
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
  if (tid == 0) *status = fail;
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

__global__ void sum_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double red[40];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) out[0] = s;
}

// ||A x - b||^2 over a tall column-major A (m x d): each thread owns rows,
// walks the d columns (coalesced across the warp), deterministic partials.
__global__ void __launch_bounds__(256) lsr_residual_kernel(const double* __restrict__ A, int64_t lda, int64_t m,
                                                           int d, const double* __restrict__ b,
                                                           const double* __restrict__ x, double* __restrict__ part) {
  extern __shared__ double xs[];
  __shared__ double red[40];
  for (int j = threadIdx.x; j < d; j += blockDim.x) xs[j] = x[j];
  __syncthreads();
  double s = 0.0;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x * 2; i0 < m; i0 += (int64_t)gridDim.x * blockDim.x * 2) {
    const int64_t i = i0 + 2 * threadIdx.x;
    if (i + 1 < m && (lda % 2 == 0) && (((uintptr_t)A) % 16 == 0)) {
      double a0 = 0.0, a1 = 0.0;
      const double2* col = reinterpret_cast<const double2*>(A + i);
#pragma unroll 8
      for (int j = 0; j < d; ++j) {
        const double2 v = __ldg(col + (int64_t)j * (lda / 2));
        a0 += v.x * xs[j];
        a1 += v.y * xs[j];
      }
      const double e0 = a0 - b[i], e1 = a1 - b[i + 1];
      s += e0 * e0 + e1 * e1;
    } else {
      for (int64_t ii = i; ii < i + 2 && ii < m; ++ii) {
        double a0 = 0.0;
        for (int j = 0; j < d; ++j) a0 += A[ii + (int64_t)j * lda] * xs[j];
        const double e0 = a0 - b[ii];
        s += e0 * e0;
      }
    }
  }
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

int launch_lsr_residual(Context* c, const double* A, int64_t lda, int64_t m, int64_t d, const double* b,
                        const double* x, double* d_out) {
  int grid = c->num_sms * 4;
  const int64_t need = (m + 511) / 512;
  if (need < grid) grid = (int)(need > 0 ? need : 1);
  double* part = partials(c, grid);
  if (!part) return SLRA_ERR_CUDA;
  SLRA_TIMED(c, "lsr_residual", lsr_residual_kernel<<<grid, 256, sizeof(double) * d, c->stream>>>(A, lda, m, (int)d, b, x, part);)
  SLRA_CHECK_LAUNCH(c);
  SLRA_TIMED(c, "reduce", sum_kernel<<<1, 256, 0, c->stream>>>(part, grid, d_out);)
  SLRA_CHECK_LAUNCH(c);
  return SLRA_OK;
}

}  // namespace slra_dev

using namespace slra_dev;

extern "C" {

int slra_lsr_residual(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t d, const double* b,
                      const double* x, double* d_out) {
  if (!ctx || lda < m || d < 1 || d > 4096) return SLRA_ERR_INVALID_ARGUMENT;
  return launch_lsr_residual(C(ctx), A, lda, m, d, b, x, d_out);
}

}  // extern "C"

namespace slra_dev {

// Solve min ||FA x - Fb|| for a sketched system FW = (FA | Fb) (k x (d+1),
// ld k). FW == nullptr: the caller has already written FW into the arena
// (returned through *fw_slot when fw_slot != nullptr on a first call).
static int lsr_solve(Context* cx, const double* FWext, int64_t k, int64_t d, double* x_hat,
                     double* h_sketched_residual, double** fw_slot) {
  const int64_t dc = d + 1;
  const int rgrid = (int)((k + 31) / 32);  // lsq_residual_kernel: 32 rows per CTA
  // arena 2: FW (k x dc) | Gw (dc x dc) | G (d x d) | g (d) | r (k) | c (d) | y (2d) | part | out
  const size_t need = (size_t)k * dc + (size_t)dc * dc + (size_t)d * d + 4 * (size_t)d + (size_t)k + rgrid + 16;
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
  // Gram [FA Fb]^T [FA Fb] (dc x dc); G = leading d x d block, g = FA^T Fb
  SLRA_TRY(launch_gemm(cx, 1, 0, dc, dc, k, 1.0, FW, k, FW, k, 0.0, Gw, dc));
  SLRA_CUDA(cudaMemcpy2DAsync(G, 8 * d, Gw, 8 * dc, 8 * d, d, cudaMemcpyDeviceToDevice, st));
  SLRA_CUDA(cudaMemcpyAsync(g, Gw + (size_t)d * dc, 8 * d, cudaMemcpyDeviceToDevice, st));
  // rank tolerance from the largest column norm of FA
  double* hs = static_cast<double*>(cx->hsmall);
  SLRA_CUDA(cudaMemcpy2DAsync(hs, 8, Gw, 8 * (dc + 1), 8, (d < 500 ? d : 500), cudaMemcpyDeviceToHost, st));
  SLRA_CUDA(cudaStreamSynchronize(st));
  double dmax = 0.0;
  for (int64_t i = 0; i < (d < 500 ? d : 500); ++i) dmax = hs[i] > dmax ? hs[i] : dmax;
  const double tol2 = 1e-20 * dmax;
  const size_t smem = sizeof(double) * ((size_t)(d + 1) * kPW + (size_t)d + kPW);  // panel, diagonal, 1/L(j,j)
  SLRA_CUDA(cudaFuncSetAttribute(cholesky_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SLRA_TIMED(cx, "lsr_solve", cholesky_kernel<<<1, kLT, smem, st>>>(G, (int)d, tol2, d_status);)
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
  SLRA_CUDA(cudaMemcpyAsync(hs + 1, d_status, 4, cudaMemcpyDeviceToHost, st));
  SLRA_CUDA(cudaStreamSynchronize(st));
  if (*reinterpret_cast<int32_t*>(hs + 1)) return SLRA_ERR_SKETCH_RANK_FAILURE;
  if (h_sketched_residual) *h_sketched_residual = sqrt(hs[0]);
  return SLRA_OK;
}

}  // namespace slra_dev

extern "C" {

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

int slra_lsr_solve_sketched(slra_ctx ctx, const double* FW, int64_t ldfw, int64_t k, int64_t d, double* x_hat,
                            double* h_sketched_residual) {
  if (!ctx || !FW || ldfw != k || k <= d || d < 1) return SLRA_ERR_INVALID_ARGUMENT;
  if (d > 768) return SLRA_ERR_UNSUPPORTED;
  return lsr_solve(C(ctx), FW, k, d, x_hat, h_sketched_residual, nullptr);
}

}  // extern "C"
