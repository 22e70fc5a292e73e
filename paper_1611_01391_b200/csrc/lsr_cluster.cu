// K-d fast path of the sketched least-squares solve (sketch_solve,
// lsr.cpp:37-67) for d <= 256, in two kernels:
//
//  1. gram_tn_kernel — the augmented Gram [FA Fb]^T [FA Fb] (lower 64 x 64
//     tiles only) on FP64 DMMA, operands staged by a 3-stage cp.async ring
//     (64 columns x 32 rows of each operand per stage), split-K with a
//     deterministic fixed-order combine (gram_combine_kernel). Also the
//     general C = alpha X^T Y used by launch_gemm for TN products.
//
//  2. chol_cluster_kernel — ONE thread-block cluster of 8 CTAs (8 SMs):
//     CTA p holds the 32-column panel p of the augmented lower Gram in its
//     shared memory (rows 32p .. d, the last row being (FA^T Fb)^T), so the
//     256 x 257 factor lives in distributed shared memory. Right-looking:
//     a cluster barrier publishes panel p; every CTA q > p pulls the rows it
//     needs over DSMEM and updates its own panel. CTA p+1, whose panel is
//     next, updates its diagonal block first, then one warp factorises that
//     block in registers while the other warps update the rows below (the
//     critical path is the diagonal chain, not the update), then the rows
//     below are solved against it. The augmented row makes the forward solve
//     L y = FA^T Fb part of the factorisation; each CTA then inverts its
//     diagonal block (D_p = L_pp^-1) and the backward solve L^T x0 = y runs
//     panel by panel (x pushed to every CTA, per step a GEMV over the panel
//     and a 32 x 32 product with D_p^T). L and D go to global memory.
//  3. lsq_refine_kernel (full grid) — one pass over FW: r0 = Fb - FA x0,
//     per-CTA partials of c = FA^T r0 and ||r0||^2 (fixed order).
//  4. chol_refine_kernel (8-CTA cluster) — reloads its panel and D_p,
//     combines the partials, solves G delta = c (forward with partial sums
//     pushed over DSMEM, backward as above), x = x0 + delta and the sketched
//     residual ||FA x - Fb||^2 = ||r0||^2 - delta^T c (G delta = c).
//
// Pivot rules as the one-CTA kernel in lsr.cu (the rank floor 1e-20 max_j
// ||FA(:,j)||^2, 64 eps of the column's own squared norm, and the 1e-6
// well-conditioning test); any failure stops the cluster uniformly and the
// host runs the reference's ColPivHouseholderQR path.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace slra_dev {

// Phase timestamps of the cluster kernel (profiling builds only,
// -DSLRA_CHOL_PROF): thread 0 of CTA q records %globaltimer at mark m.
#ifdef SLRA_CHOL_PROF
__device__ unsigned long long g_chol_marks[8][64];
__device__ __forceinline__ void chol_mark(int q, int m) {
  if (threadIdx.x == 0 && m < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_chol_marks[q][m] = t;
  }
}
#define CHOL_MARK(q, m) chol_mark(q, m)
#else
#define CHOL_MARK(q, m) ((void)0)
#endif

// ------------------------------------------------------------ TN Gram / GEMM
namespace gt {
constexpr int NT = 256;
constexpr int BM = 64, BN = 64, BK = 32;
constexpr int LD = BK + 4;  // Xs[col][k]: fragment reads hit 16 distinct double slots
constexpr int NS = 3;
constexpr int STAGE = (BM + BN) * LD;  // doubles per stage
constexpr size_t SMEM = sizeof(double) * NS * STAGE;
}  // namespace gt

struct GramArgs {
  const double* X;
  int64_t ldx;
  const double* Y;
  int64_t ldy;
  int64_t m, n, K;  // C (m x n) = X^T Y, X: K x m, Y: K x n (column-major)
  int lower;        // only tiles with ti >= tj (X == Y, m == n)
  int tiles_n, ntiles;
  int64_t kchunk;  // rows of K per z-slice (multiple of BK)
  double* part;    // [z][tile][BM * BN] partial tiles
  // batched problems (blockIdx.z): X, Y, part, C advance by these strides
  int64_t sX = 0, sY = 0, sP = 0, sC = 0;
};

__device__ __forceinline__ void gt_cp16(double* smem, const double* g, int bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(g), "r"(bytes));
}

__device__ __forceinline__ void gt_tile_of(const GramArgs& a, int t, int& ti, int& tj) {
  if (a.lower) {
    ti = 0;
    while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
    tj = t - ti * (ti + 1) / 2;
  } else {
    ti = t / a.tiles_n;
    tj = t % a.tiles_n;
  }
}

// stage rows k0 .. k0+BK-1 of the X columns i0.. and the Y columns j0..
__device__ __forceinline__ void gt_stage(const GramArgs& a, int64_t i0, int64_t j0, int64_t k0, int64_t kend,
                                         double* st) {
  using namespace gt;
  double* Xs = st;
  double* Ys = st + BM * LD;
  // 16-byte chunks: 64 columns x 16 chunks per operand, 8 per thread
#pragma unroll
  for (int u = 0; u < (BM + BN) * (BK / 2) / NT; ++u) {
    const int e = threadIdx.x + u * NT;
    const bool isx = e < BM * (BK / 2);
    const int e2 = isx ? e : e - BM * (BK / 2);
    const int col = e2 >> 4, ch = e2 & 15;
    const int64_t kk = k0 + 2 * ch;
    const int64_t cc = (isx ? i0 : j0) + col;
    const int64_t lim = isx ? a.m : a.n;
    const double* base = isx ? a.X : a.Y;
    const int64_t ld = isx ? a.ldx : a.ldy;
    int bytes = 0;
    const double* src = base;
    if (cc < lim && kk < kend) {
      bytes = kk + 1 < kend ? 16 : 8;
      src = base + kk + cc * ld;
    }
    gt_cp16((isx ? Xs : Ys) + col * LD + 2 * ch, src, bytes);
  }
}

__global__ void __launch_bounds__(gt::NT, 2) gram_tn_kernel(GramArgs a) {
  using namespace gt;
  extern __shared__ __align__(16) double sm[];
  a.X += blockIdx.z * a.sX;
  a.Y += blockIdx.z * a.sY;
  a.part += blockIdx.z * a.sP;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;  // 32 x 16 per warp
  int ti, tj;
  gt_tile_of(a, blockIdx.x, ti, tj);
  const int64_t i0 = (int64_t)ti * BM, j0 = (int64_t)tj * BN;
  const int64_t kb = (int64_t)blockIdx.y * a.kchunk;
  const int64_t ke = kb + a.kchunk < a.K ? kb + a.kchunk : a.K;
  const int nsteps = kb < ke ? (int)((ke - kb + BK - 1) / BK) : 0;
  double acc[4][2][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
#pragma unroll
  for (int s = 0; s < NS - 1; ++s) {
    if (s < nsteps) gt_stage(a, i0, j0, kb + (int64_t)s * BK, ke, sm + s * STAGE);
    asm volatile("cp.async.commit_group;\n" ::);
  }
  for (int s = 0; s < nsteps; ++s) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(NS - 2));
    __syncthreads();
    // refill the slot consumed in the previous iteration
    if (s + NS - 1 < nsteps) gt_stage(a, i0, j0, kb + (int64_t)(s + NS - 1) * BK, ke, sm + ((s + NS - 1) % NS) * STAGE);
    asm volatile("cp.async.commit_group;\n" ::);
    const double* Xs = sm + (s % NS) * STAGE;
    const double* Ys = Xs + BM * LD;
#pragma unroll
    for (int kq = 0; kq < BK / 4; ++kq) {
      double af[4], bf[2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) af[mi] = Xs[(wm * 32 + mi * 8 + g) * LD + 4 * kq + t4];
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) bf[ni] = Ys[(wn * 16 + ni * 8 + g) * LD + 4 * kq + t4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  double* out = a.part + ((int64_t)blockIdx.y * a.ntiles + blockIdx.x) * (BM * BN);
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      const int r = wm * 32 + mi * 8 + g, c = wn * 16 + ni * 8 + 2 * t4;
      out[r + c * BM] = acc[mi][ni][0];
      out[r + (c + 1) * BM] = acc[mi][ni][1];
    }
}

// C = alpha sum_z part[z] + beta C over the computed tiles (slices in order)
__global__ void gram_combine_kernel(GramArgs a, int nz, double alpha, double beta, double* __restrict__ Cm,
                                    int64_t ldc) {
  using namespace gt;
  a.part += blockIdx.y * a.sP;
  Cm += blockIdx.y * a.sC;
  const int64_t total = (int64_t)a.ntiles * BM * BN;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(e / (BM * BN)), w = (int)(e % (BM * BN));
    int ti, tj;
    gt_tile_of(a, t, ti, tj);
    const int64_t r = (int64_t)ti * BM + (w % BM), c = (int64_t)tj * BN + (w / BM);
    if (r >= a.m || c >= a.n) continue;
    double s = 0.0;
    for (int z = 0; z < nz; ++z) s += a.part[(int64_t)z * total + e];
    double v = alpha * s;
    if (beta != 0.0) v += beta * Cm[r + c * ldc];
    Cm[r + c * ldc] = v;
  }
}

int launch_gram_tn_batched(Context* c, const char* fam, int nb, int64_t m, int64_t n, int64_t K, double alpha,
                           const double* X, int64_t ldx, int64_t sX, const double* Y, int64_t ldy, int64_t sY,
                           double beta, double* Cm, int64_t ldc, int64_t sC, int lower);

// C = alpha X^T Y + beta C (lower = 1: X == Y, only the lower triangle's
// tiles — every entry on or below the diagonal — are written).
// SLRA_ERR_UNSUPPORTED when the operands are not 16-byte aligned.
int launch_gram_tn(Context* c, const char* fam, int64_t m, int64_t n, int64_t K, double alpha, const double* X,
                   int64_t ldx, const double* Y, int64_t ldy, double beta, double* Cm, int64_t ldc, int lower) {
  return launch_gram_tn_batched(c, fam, 1, m, n, K, alpha, X, ldx, 0, Y, ldy, 0, beta, Cm, ldc, 0, lower);
}

// nb products of the same shape at fixed strides in one launch (grid z)
int launch_gram_tn_batched(Context* c, const char* fam, int nb, int64_t m, int64_t n, int64_t K, double alpha,
                           const double* X, int64_t ldx, int64_t sX, const double* Y, int64_t ldy, int64_t sY,
                           double beta, double* Cm, int64_t ldc, int64_t sC, int lower) {
  using namespace gt;
  if (m == 0 || n == 0 || nb == 0) return SLRA_OK;
  const bool aligned = ((uintptr_t)X % 16 == 0) && (ldx % 2 == 0) && ((uintptr_t)Y % 16 == 0) && (ldy % 2 == 0) &&
                       (sX % 2 == 0) && (sY % 2 == 0);
  if (!aligned || K < 1) return SLRA_ERR_UNSUPPORTED;
  const int tm = ceil_div(m, BM), tn_ = ceil_div(n, BN);
  const int ntiles = lower ? tm * (tm + 1) / 2 : tm * tn_;
  // split K so that the grid fills about two CTAs per SM, >= 4 k-steps each
  const int64_t ksteps = (K + BK - 1) / BK;
  int64_t nz = (2 * (int64_t)c->num_sms + (int64_t)ntiles * nb - 1) / ((int64_t)ntiles * nb);
  if (nz > ksteps / 4) nz = ksteps / 4;
  if (nz < 1) nz = 1;
  const int64_t kchunk = (ksteps + nz - 1) / nz * BK;
  nz = (K + kchunk - 1) / kchunk;
  const int64_t per = nz * ntiles * BM * BN;
  double* part = static_cast<double*>(workspace(c, sizeof(double) * per * nb));
  if (!part) return SLRA_ERR_CUDA;
  GramArgs a{X, ldx, Y, ldy, m, n, K, lower, tn_, ntiles, kchunk, part};
  a.sX = sX;
  a.sY = sY;
  a.sP = per;
  a.sC = sC;
  SLRA_CUDA(cudaFuncSetAttribute(gram_tn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
  SLRA_TIMED(c, fam, gram_tn_kernel<<<dim3(ntiles, (unsigned)nz, nb), NT, SMEM, c->stream>>>(a);)
  SLRA_CHECK_LAUNCH(c);
  int rg = ceil_div((int64_t)ntiles * BM * BN, 256);
  if (rg > c->num_sms * 4) rg = c->num_sms * 4;
  SLRA_TIMED(c, "gemm_reduce", gram_combine_kernel<<<dim3(rg, nb), 256, 0, c->stream>>>(a, (int)nz, alpha, beta, Cm, ldc);)
  SLRA_CHECK_LAUNCH(c);
  return SLRA_OK;
}

// ------------------------------------------------- cluster Cholesky + solve
namespace cc {
constexpr int NT = 256;
constexpr int NC = 8;    // CTAs per cluster = max panels
constexpr int PW = 32;   // panel width
constexpr int RMAX = NC * PW + 1;  // rows of panel 0 (augmented)
constexpr int LDMAX = (RMAX + 1) & ~1;
constexpr int LDD = PW + 1;  // D_p (32 x 32, ld 33)
// dynamic shared memory (doubles)
constexpr int OFF_P = 0;                  // own panel (ld = rows | 1)
constexpr int OFF_S = OFF_P + LDMAX * PW;  // staged rows of a published panel
constexpr int OFF_D = OFF_S + LDMAX * PW;  // D_p = L_pp^-1
constexpr int OFF_X = OFF_D + PW * LDD;    // x (every CTA keeps all of it)
constexpr int OFF_Y = OFF_X + RMAX + 1;    // y / delta
constexpr int OFF_A = OFF_Y + RMAX + 1;    // pushed partial sums (forward solve)
constexpr int OFF_C = OFF_A + PW;          // c of the own panel + ||r0||^2
constexpr int OFF_RD = OFF_C + PW + 2;     // 1 / L(j, j)
constexpr int OFF_GD = OFF_RD + PW;        // original diagonal of the own panel
constexpr int OFF_RED = OFF_GD + PW;       // 8 x 33 reduction scratch
constexpr int OFF_T = OFF_RED + 8 * 33;    // right-hand side of a panel step
constexpr int OFF_ST = OFF_T + PW;         // status ints: (fail, illc) per panel
constexpr int TOTAL = OFF_ST + NC + 1;  // + this CTA's own status word
constexpr size_t SMEM = sizeof(double) * TOTAL;
constexpr size_t SMEM_REFINE = sizeof(double) * OFF_S + sizeof(double) * (TOTAL - OFF_D);  // no staging area
constexpr int PANEL = LDMAX * PW;  // doubles per panel in the global copy
}  // namespace cc

struct CholArgs {
  const double* Gw;  // (d+1) x (d+1) augmented Gram, lower triangle valid, ld d+1
  int d;
  const double* FW;  // k x (d+1), ld k
  int64_t k;
  double tol_rel;   // rank floor relative to max_j ||FA(:,j)||^2
  double* x;        // d: x0 (K1), then x (K3)
  double* Lg;       // np panels (cc::PANEL doubles each) + np D blocks (PW * LDD each)
  const double* part;  // K2 partials: nparts x (d + 1) (c, ||r0||^2)
  int nparts;
  double* out;      // [0] sketched residual^2
  int32_t* status;  // [0] rank failure, [1] ill-conditioned (-> exact path)
};
// up to kMaxProb independent solves in one launch of each kernel (config 4's
// two samplers): cluster b / NC (K1, K3) or grid row blockIdx.y (K2) takes
// problem p[b]; the clusters run side by side on different SMs
constexpr int kMaxProb = 4;
struct CholArgsN {
  CholArgs p[kMaxProb];
};

// lane i of the calling warp ends with y_i of L11 y = t (FWD) or
// L11^T y = t: the 32-step shuffle chain (used to form D_p).
template <bool FWD>
__device__ __forceinline__ double warp_tri_solve(const double* P, int ldp, const double* rd, int pw, double t) {
  const int lane = threadIdx.x & 31;
  double l[cc::PW];
#pragma unroll
  for (int c = 0; c < cc::PW; ++c)
    l[c] = FWD ? load_sel(P + lane, (int64_t)c * ldp, c < lane && lane < pw)
               : load_sel(P + c, (int64_t)lane * ldp, c > lane && c < pw);
  const double r = lane < pw ? rd[lane] : 0.0;
  double y = lane < pw ? t : 0.0;
  if (FWD) {
#pragma unroll
    for (int c = 0; c < cc::PW; ++c) {
      if (lane == c) y *= r;
      const double yc = __shfl_sync(0xffffffffu, y, c);
      if (lane > c) y = fma(-l[c], yc, y);
    }
  } else {
#pragma unroll
    for (int c = cc::PW - 1; c >= 0; --c) {
      if (lane == c) y *= r;
      const double yc = __shfl_sync(0xffffffffu, y, c);
      if (lane < c) y = fma(-l[c], yc, y);
    }
  }
  return y;
}

// P(i, c) -= sum_t S(i, t) S(c, t) for panel rows i in [rb, re) (rb a
// multiple of 8), c < pw, i >= c, on FP64 DMMA (m8n8k4) by warps wid, wid +
// nw, ...: warp-level 8 x 32 row tiles, the B fragments (the staged diagonal
// rows, 32 x 32) held in registers for all of them.
__device__ __forceinline__ void dmma_update(double* P, const double* S, int ldp, int rb, int re, int pw, int wid,
                                            int nw) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  double bf[8][4];  // [k-step][n-tile]: B(k, n) = S(8 n + g, 4 k + t4)
#pragma unroll
  for (int k = 0; k < 8; ++k)
#pragma unroll
    for (int n = 0; n < 4; ++n) bf[k][n] = S[(8 * n + g) + (4 * k + t4) * ldp];
  const int ntiles = (re - rb + 7) >> 3;
  for (int mt = wid; mt < ntiles; mt += nw) {
    const int r = rb + 8 * mt + g;  // A(m, k) = S(row, 4 k + t4)
    double acc[4][2];
#pragma unroll
    for (int n = 0; n < 4; ++n) acc[n][0] = acc[n][1] = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double av = load_sel(S + (4 * k + t4) * ldp, r, r < re);
#pragma unroll
      for (int n = 0; n < 4; ++n) dmma_8x8x4(acc[n][0], acc[n][1], av, bf[k][n]);
    }
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * n + 2 * t4 + e;
        if (r < re && c < pw && r >= c) P[r + c * ldp] -= acc[n][e];
      }
  }
}

// S rows [i0, i1) (even bounds except an odd panel end, whose pad row is
// read) <- rows off + i of the published panel Pp (ld ldpp), 16-byte L2-only
// loads, eight in flight per thread, by threads th = 0 .. nth - 1
__device__ __forceinline__ void stage_rows(double* S, int ldp, const double* Pp, int ldpp, int off, int i0, int i1,
                                           int th, int nth) {
  const int hr = (i1 - i0 + 1) >> 1;  // row pairs per column
  for (int e0 = th; e0 < hr * cc::PW; e0 += nth * 8) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = min(e0 + u * nth, hr * cc::PW - 1);
      const int i2 = e % hr, c = e / hr;
      v[u] = __ldcg(reinterpret_cast<const double2*>(Pp + (off + i0 + 2 * i2) + (int64_t)c * ldpp));
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * nth;
      if (e < hr * cc::PW) *reinterpret_cast<double2*>(S + i0 + 2 * (e % hr) + (e / hr) * ldp) = v[u];
    }
  }
}

// Cholesky of the (fully updated) pw x pw diagonal block by warps 0-3 in a
// compact loop (this runs once per CTA: unrolled single-warp variants were
// bound by instruction fetch or by their serial instruction latency), while
// warps 4-7 stage and update the rows below. Thread (i = lane, w = warp < 4)
// holds A(i, w + 4 v), v < 8, in registers. Column j, once final, is
// published in M (32 x 33, kept: the factor is read from it at the end), and
// every thread applies A(i, c) += f_i A(c, j), f_i = -A(i, j) / A(j, j)
// (zero for i <= j) to all its entries unconditionally: entries of columns
// already published or above the diagonal take garbage, which is never read
// (the owner of column j+1 republishes only its unpublished columns). The
// pivot tests run after the loop on the published pivots (a failed pivot
// only poisons values that are then discarded). ~300 cycles per column step
// (one 128-thread named barrier). L(i, c) = M(i, c) / sqrt(M(c, c)); writes
// L11 and rd = 1 / L(j, j); returns fail | illc << 1.
__device__ int warp4_diag_factor(double* P, int ldp, int pw, const double* gd, double tol2, double* rd, double* M) {
  const int i = threadIdx.x & 31, w = threadIdx.x >> 5;  // w < 4
  constexpr int LM = cc::PW + 1;
  double a[8];
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    const int c = w + 4 * v;
    a[v] = (i < pw && c < pw && i >= c) ? P[i + c * ldp] : 0.0;
  }
  if (w == 0) M[i] = a[0];  // column 0
  asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll 1
  for (int j = 0; j < pw; ++j) {
    const double* cj = M + j * LM;
    const double piv = cj[j];
    const double rp = piv >= DBL_MIN ? fast_rcp(piv) : 1.0 / piv;
    const double f = i > j ? -cj[i] * rp : 0.0;
#pragma unroll
    for (int v = 0; v < 8; ++v) a[v] = fma(f, cj[w + 4 * v], a[v]);
    const int jn = j + 1;
    if (w == (jn & 3)) {
      const int vv = jn >> 2;
#pragma unroll
      for (int v = 0; v < 8; ++v)
        if (v >= vv) M[i + (w + 4 * v) * LM] = a[v];
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
  }
  int fail = 0, illc = 0;
  for (int c = 0; c < pw; ++c) {
    const double piv = M[c + c * LM], g0 = gd[c];
    if (!(piv > tol2) || !(piv > 64.0 * 2.220446049250313e-16 * g0)) fail = 1;
    if (!(piv > 1e-6 * g0)) illc = 1;
  }
  if (!fail) {
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const int c = w + 4 * v;
      if (i < pw && c < pw && i >= c) {
        const double pc = M[c + c * LM];
        const double r = pc >= DBL_MIN ? fast_rsqrt(pc) : 1.0 / sqrt(pc);
        P[i + c * ldp] = i == c ? pc * r : M[i + c * LM] * r;
        if (i == c) rd[c] = r;
      }
    }
  }
  return fail | (illc << 1);
}

// rows [pw, rows) of the own panel: L21 = A21 L11^-T, a thread per row
__device__ __forceinline__ void panel_trsm(double* P, int ldp, int pw, int rows, const double* rd) {
  for (int i = pw + threadIdx.x; i < rows; i += cc::NT) {
    double z[cc::PW];
#pragma unroll
    for (int c = 0; c < cc::PW; ++c) z[c] = load_sel(P + i, (int64_t)c * ldp, c < pw);
#pragma unroll
    for (int t = 0; t < cc::PW; ++t) {
      z[t] *= t < pw ? rd[t] : 0.0;
#pragma unroll
      for (int c = t + 1; c < cc::PW; ++c) z[c] = fma(-z[t], P[c + t * ldp], z[c]);
    }
#pragma unroll
    for (int c = 0; c < cc::PW; ++c)
      if (c < pw) P[i + c * ldp] = z[c];
  }
}

// the finished panel (ldp x 32, pads included) to its global slot, 16-byte stores
__device__ __forceinline__ void publish_panel(const double* P, int ldp, double* Lq) {
  const int n2 = ldp * cc::PW / 2;
  const double2* src = reinterpret_cast<const double2*>(P);
  double2* dst = reinterpret_cast<double2*>(Lq);
  for (int e = threadIdx.x; e < n2; e += cc::NT) __stcg(dst + e, src[e]);
}

// D = L11^-1 (lower, ld LDD): warp w forms columns w, w + 8, w + 16, w + 24
__device__ __forceinline__ void panel_diag_inverse(const double* P, int ldp, int pw, const double* rd, double* D) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = warp; c < cc::PW; c += cc::NT / 32) {
    const double y = warp_tri_solve<true>(P, ldp, rd, pw, lane == c ? 1.0 : 0.0);
    D[lane + c * cc::LDD] = (c < pw && lane < pw) ? y : 0.0;
  }
}

// One backward step on the own panel p: out_c = D_p^T (t_c - sum_i L(i, c) v_i)
// over the panel rows below the block (global rows r0 + i < d); `tin` is the
// right-hand side of the block (smem, PW), result pushed into v of every CTA.
__device__ __forceinline__ void backward_step(cg::cluster_group& cl, const double* P, int ldp, int pw, int rows,
                                              int r0, const double* D, double* v, const double* tin, double* red,
                                              double* tv) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  {
    double s0 = 0.0, s1 = 0.0;
    int i = pw + warp;
    for (; i + 8 < rows - 1; i += 16) {
      s0 = fma(P[i + lane * ldp], v[r0 + i], s0);
      s1 = fma(P[i + 8 + lane * ldp], v[r0 + i + 8], s1);
    }
    if (i < rows - 1) s0 = fma(P[i + lane * ldp], v[r0 + i], s0);
    red[warp * 33 + lane] = s0 + s1;
  }
  __syncthreads();
  if (warp == 0) {
    double t = lane < pw ? tin[lane] : 0.0;
#pragma unroll
    for (int w = 0; w < cc::NT / 32; ++w) t -= red[w * 33 + lane];
    tv[lane] = t;
  }
  __syncthreads();
  if (warp == 0) {
    // x_c = sum_{j >= c} D(j, c) t_j   (D^T is upper triangular)
    double x0 = 0.0, x1 = 0.0;
#pragma unroll
    for (int j = 0; j < cc::PW; j += 2) {
      x0 = fma(D[j + lane * cc::LDD], tv[j], x0);
      x1 = fma(D[j + 1 + lane * cc::LDD], tv[j + 1], x1);
    }
    const double xc = x0 + x1;
    if (lane < pw)
      for (int rk = 0; rk < cc::NC; ++rk) cl.map_shared_rank(v, rk)[r0 + lane] = xc;
  }
}

__global__ void __cluster_dims__(cc::NC, 1, 1) __launch_bounds__(cc::NT, 1) chol_cluster_kernel(CholArgsN args) {
  using namespace cc;
  const CholArgs a = args.p[blockIdx.x / NC];
  extern __shared__ __align__(16) double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int d = a.d, dc = d + 1;
  const int np = (d + PW - 1) / PW;
  const bool own = q < np;
  const int r0 = q * PW;
  const int pw = own ? (d - r0 < PW ? d - r0 : PW) : 0;
  const int rows = own ? dc - r0 : 0;  // panel rows r0 .. d (the last one is the augmented row)
  const int ldp = (rows + 1) & ~1;  // even: 16-byte aligned columns
  double* P = sm + OFF_P;
  double* S = sm + OFF_S;
  double* D = sm + OFF_D;
  double* xv = sm + OFF_X;
  double* rd = sm + OFF_RD;
  double* gd = sm + OFF_GD;
  double* red = sm + OFF_RED;
  double* tv = sm + OFF_T;
  int* st = reinterpret_cast<int*>(sm + OFF_ST);  // [0] fail [1] illc

  // rank floor from the largest squared column norm of FA (all d columns)
  double dm = 0.0;
  for (int j = tid; j < d; j += NT) dm = fmax(dm, a.Gw[j + (int64_t)j * dc]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
  if (lane == 0) red[warp] = dm;
  // every CTA of the cluster must have started before any DSMEM access:
  // arrive now, wait just before the first remote store (CTA 0: after its
  // first panel, so the wait costs nothing on the critical path)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
  // the own panel (lower part; zeros elsewhere), eight loads in flight
  if (own) {
    for (int e0 = tid; e0 < rows * PW; e0 += NT * 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * NT, i = e % rows, c = e / rows;
        v[u] = load_sel(a.Gw, (int64_t)(r0 + i) + (int64_t)(r0 + c) * dc, e < rows * PW && c < pw && i >= c);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * NT;
        if (e < rows * PW) P[(e % rows) + (e / rows) * ldp] = v[u];
      }
    }
    if (tid < PW) gd[tid] = tid < pw ? a.Gw[(r0 + tid) + (int64_t)(r0 + tid) * dc] : 1.0;
  }
  __syncthreads();
  double mx = 0.0;
  for (int w = 0; w < NT / 32; ++w) mx = fmax(mx, red[w]);
  const double tol2 = a.tol_rel * mx;
  CHOL_MARK(q, 0);
  if (q == 0) {
    int f = 0;
    if (warp < 4) {
      f = warp4_diag_factor(P, ldp, pw, gd, tol2, rd, D);
      if (tid == 0) st[2 * NC] = f;
    }
    __syncthreads();
    f = st[2 * NC];
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
    if (tid < NC) {  // the panel's status into every CTA's slot p (read locally after the barrier)
      int* rs = cl.map_shared_rank(st, tid);
      rs[2 * q] = f & 1;
      rs[2 * q + 1] = f >> 1;
    }
    __syncthreads();
    CHOL_MARK(7, 54);
    if (!f) panel_trsm(P, ldp, pw, rows, rd);
    __syncthreads();
    publish_panel(P, ldp, a.Lg);
  } else {
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
  }
  CHOL_MARK(q, 1);
  cl.sync();  // panel 0 published
  bool failed = false;
  for (int p = 0; p < np; ++p) {
    {
      const int f0 = st[2 * p], f1 = st[2 * p + 1];
      if (f0 | f1) {
        if (q == 0 && tid == 0) {
          a.status[0] = f0;
          a.status[1] = f1;
        }
        failed = true;
        break;  // cluster-uniform
      }
    }
    if (p == np - 1) break;
    if (own && q > p) {
      CHOL_MARK(q, 8 + 4 * p);
      // rows r0 .. d of panel p (its local rows r0 - 32 p ..) from the global
      // copy its owner wrote before the barrier (L2; one SM's shared memory
      // served to seven readers over DSMEM was the bottleneck)
      const double* Pp = a.Lg + (size_t)p * PANEL;
      const int ldpp = (dc - p * PW + 1) & ~1;
      const int off = r0 - p * PW;
      if (q == p + 1) {
        // the next panel (the critical path): its diagonal rows first, their
        // update, then warps 0-3 factorise the diagonal block while warps 4-7
        // stage and update the rows below; then the rows below are solved
        const int rd_end = rows < PW ? rows : PW;  // never past the panel's own ld
        stage_rows(S, ldp, Pp, ldpp, off, 0, rd_end, tid, NT);
        __syncthreads();
        CHOL_MARK(q, 9 + 4 * p);
        dmma_update(P, S, ldp, 0, pw, pw, warp, NT / 32);
        __syncthreads();
        CHOL_MARK(q, 10 + 4 * p);
        int f = 0;
        if (warp < 4) {
          f = warp4_diag_factor(P, ldp, pw, gd, tol2, rd, D);
          if (tid == 0) st[2 * NC] = f;
          CHOL_MARK(q, 48 + p);
        } else {
          stage_rows(S, ldp, Pp, ldpp, off, PW, rows, tid - 128, 128);
          asm volatile("bar.sync 2, 128;" ::: "memory");
          dmma_update(P, S, ldp, pw, rows, pw, warp - 4, 4);
        }
        __syncthreads();
        CHOL_MARK(q, 11 + 4 * p);
        f = st[2 * NC];
        if (tid < NC) {  // the panel's status into every CTA's slot q (read locally after the barrier)
          int* rs = cl.map_shared_rank(st, tid);
          rs[2 * q] = f & 1;
          rs[2 * q + 1] = f >> 1;
        }
        if (!f) panel_trsm(P, ldp, pw, rows, rd);
        __syncthreads();
        CHOL_MARK(q, 56 + p);
        publish_panel(P, ldp, a.Lg + (size_t)q * PANEL);
      } else {
        stage_rows(S, ldp, Pp, ldpp, off, 0, rows, tid, NT);
        __syncthreads();
        CHOL_MARK(q, 9 + 4 * p);
        dmma_update(P, S, ldp, 0, rows, pw, warp, NT / 32);
      }
      __syncthreads();
    }
    cl.sync();  // panel p + 1 published
  }

  if (!failed) {
    CHOL_MARK(q, 40);
    if (own) {
      panel_diag_inverse(P, ldp, pw, rd, D);
      if (tid < PW) tv[tid] = tid < pw ? P[(rows - 1) + tid * ldp] : 0.0;  // y (augmented row)
      __syncthreads();
    }
    // ---- x0 = L^-T y
    for (int p = np - 1; p >= 0; --p) {
      if (q == p) backward_step(cl, P, ldp, pw, rows, r0, D, xv, tv, red, tv + 0);
      cl.sync();
    }
    CHOL_MARK(q, 41);
    // L and D to global memory for the refinement solve; x0
    if (own) {
      double* Dq = a.Lg + (size_t)np * PANEL + (size_t)q * PW * LDD;
      for (int e = tid; e < PW * LDD; e += NT) Dq[e] = D[e];
    }
    if (q == 0) {
      for (int j = tid; j < d; j += NT) a.x[j] = xv[j];
      if (tid == 0) a.status[0] = a.status[1] = 0;
    }
  }
  cl.sync();  // no CTA leaves while others may still read its shared memory
  CHOL_MARK(q, 46);
}

// ---- r0 = Fb - FA x0 and per-CTA partials of c = FA^T r0, ||r0||^2 (K2)
constexpr int kRC = 32;  // rows per chunk
__global__ void __launch_bounds__(256) lsq_refine_kernel(CholArgsN args) {
  const CholArgs& pa = args.p[blockIdx.y];
  const double* __restrict__ FW = pa.FW;
  const int64_t k = pa.k;
  const int d = pa.d;
  const double* __restrict__ x = pa.x;
  const int32_t* __restrict__ status = pa.status;
  double* __restrict__ part = const_cast<double*>(pa.part);
  extern __shared__ double sm2[];
  double* xs = sm2;                   // d
  double* Ch = sm2 + d + 1;           // (d + 1) x (kRC + 1)
  __shared__ double red[8][33];
  __shared__ double rv[kRC];
  if (status[0] | status[1]) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int dc = d + 1;
  for (int j = tid; j < d; j += 256) xs[j] = x[j];
  __syncthreads();
  double cacc[2] = {0.0, 0.0};  // c_j for j = tid, tid + 256 (d <= 511)
  double rr = 0.0;
  for (int64_t i0 = (int64_t)blockIdx.x * kRC; i0 < k; i0 += (int64_t)gridDim.x * kRC) {
    const bool in = i0 + lane < k;
    const double* fw = FW + i0 + (in ? lane : 0);
    double part_ = 0.0;
    for (int j0 = warp; j0 < dc; j0 += 8 * 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = j0 + 8 * u;
        v[u] = load_sel(fw, (int64_t)j * k, in && j < dc);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = j0 + 8 * u;
        if (j < dc) {
          Ch[j * (kRC + 1) + lane] = v[u];
          part_ = j < d ? fma(v[u], xs[j], part_) : part_ - v[u];
        }
      }
    }
    red[warp][lane] = part_;
    __syncthreads();
    if (warp == 0) {
      double r = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) r -= red[w][lane];
      r = in ? r : 0.0;
      rv[lane] = r;
      rr = fma(r, r, rr);
    }
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = tid + 256 * h;
      if (j < d) {
        const double* cj = Ch + j * (kRC + 1);
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int i = 0; i < kRC; i += 2) {
          a0 = fma(cj[i], rv[i], a0);
          a1 = fma(cj[i + 1], rv[i + 1], a1);
        }
        cacc[h] += a0 + a1;
      }
    }
    __syncthreads();
  }
  double* pb = part + (int64_t)blockIdx.x * dc;
#pragma unroll
  for (int h = 0; h < 2; ++h)
    if (tid + 256 * h < d) pb[tid + 256 * h] = cacc[h];
  if (warp == 0) {
    rr = warp_sum(rr);
    if (lane == 0) pb[d] = rr;
  }
}

// ---- G delta = c on the cluster, x = x0 + delta (K3)
__global__ void __cluster_dims__(cc::NC, 1, 1) __launch_bounds__(cc::NT, 1) chol_refine_kernel(CholArgsN args) {
  using namespace cc;
  const CholArgs a = args.p[blockIdx.x / NC];
  extern __shared__ __align__(16) double sm[];
  cg::cluster_group cl = cg::this_cluster();
  if (a.status[0] | a.status[1]) return;  // uniform over the cluster (status is final)
  const int q = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int d = a.d, dc = d + 1;
  const int np = (d + PW - 1) / PW;
  const bool own = q < np;
  const int r0 = q * PW;
  const int pw = own ? (d - r0 < PW ? d - r0 : PW) : 0;
  const int rows = own ? dc - r0 : 0;
  const int ldp = (rows + 1) & ~1;  // even: 16-byte aligned columns
  // no staging area here: D and the vectors follow the panel directly
  double* P = sm;
  double* D = sm + OFF_S;
  double* base = D - OFF_D;  // so that base + OFF_X ... address the vectors
  double* xv = base + OFF_X;
  double* yv = base + OFF_Y;
  double* acc = base + OFF_A;
  double* cv = base + OFF_C;
  double* red = base + OFF_RED;
  double* tv = base + OFF_T;
  if (own) {
    const double* Lq = a.Lg + (size_t)q * PANEL;
    for (int e0 = tid; e0 < ldp * PW; e0 += NT * 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = load_sel(Lq, e0 + u * NT, e0 + u * NT < ldp * PW);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (e0 + u * NT < ldp * PW) P[e0 + u * NT] = v[u];
    }
    const double* Dq = a.Lg + (size_t)np * PANEL + (size_t)q * PW * LDD;
    for (int e = tid; e < PW * LDD; e += NT) D[e] = Dq[e];
    // c of the own panel from the K2 partials (fixed order)
    if (tid < PW + 1) {
      const int j = tid < PW ? r0 + tid : d;
      double s = 0.0;
      if (tid < pw || tid == PW)
        for (int b = 0; b < a.nparts; ++b) s += a.part[(int64_t)b * dc + j];
      cv[tid] = s;
    }
  }
  for (int j = tid; j < d; j += NT) xv[j] = a.x[j];
  if (tid < PW) acc[tid] = 0.0;
  __syncthreads();
  cl.sync();
  // forward: y_p = D_p (c_p - acc_p); push L(rows below, p) y_p to their owners
  for (int p = 0; p < np; ++p) {
    if (q == p) {
      if (warp == 0) {
        tv[lane] = lane < pw ? cv[lane] - acc[lane] : 0.0;
        __syncwarp();
        double y0 = 0.0, y1 = 0.0;
#pragma unroll
        for (int j = 0; j < PW; j += 2) {  // y_i = sum_{j <= i} D(i, j) t_j
          y0 = fma(D[lane + j * LDD], tv[j], y0);
          y1 = fma(D[lane + (j + 1) * LDD], tv[j + 1], y1);
        }
        const double y = lane < pw ? y0 + y1 : 0.0;
        __syncwarp();
        tv[lane] = y;
        yv[r0 + lane] = y;
      }
      __syncthreads();
      for (int i = pw + tid; i < rows - 1; i += NT) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int c = 0; c < PW; c += 2) {  // columns >= pw are zero
          s0 = fma(P[i + c * ldp], tv[c], s0);
          s1 = fma(P[i + (c + 1) * ldp], tv[c + 1], s1);
        }
        const int R = r0 + i;
        double* ra = cl.map_shared_rank(acc, R / PW);
        ra[R % PW] += s0 + s1;
      }
    }
    cl.sync();
  }
  // backward: delta = L^-T y
  double* tin = tv + 0;
  for (int p = np - 1; p >= 0; --p) {
    if (q == p) {
      if (tid < PW) tin[tid] = tid < pw ? yv[r0 + tid] : 0.0;
      __syncthreads();
      backward_step(cl, P, ldp, pw, rows, r0, D, yv, tin, red, tv);
    }
    cl.sync();
  }
  if (q == 0) {
    // x = x0 + delta; ||FA x - Fb||^2 = ||r0||^2 - delta^T c (sum of the
    // panels' c: every CTA's cv, gathered in rank order)
    double dc_ = 0.0;
    for (int j = tid; j < d; j += NT) {
      a.x[j] = xv[j] + yv[j];
      dc_ = fma(yv[j], cl.map_shared_rank(cv, j / PW)[j % PW], dc_);
    }
    dc_ = warp_sum(dc_);
    if (lane == 0) red[warp] = dc_;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < NT / 32; ++w) s += red[w];
      const double r2 = cv[PW] - s;
      a.out[0] = r2 > 0.0 ? r2 : 0.0;
    }
  }
  cl.sync();
}

// K1 + K2 + K3. Lg: workspace of lsr_cluster_ws_doubles(d) doubles.
size_t lsr_cluster_ws_doubles(int d, int64_t k, int num_sms) {
  const int np = (d + cc::PW - 1) / cc::PW;
  int64_t nparts = (k + kRC - 1) / kRC;
  if (nparts > 2 * num_sms) nparts = 2 * num_sms;
  return (size_t)np * cc::PANEL + (size_t)np * cc::PW * cc::LDD + (size_t)nparts * (d + 1) + 64;
}

// K1 + K2 + K3 for nprob <= kMaxProb independent solves of the same d and
// k (one launch each). Per problem: Gw, FW, x, ws (lsr_cluster_ws_doubles),
// out, status.
int launch_chol_cluster_batched(Context* c, int nprob, const double* const* Gw, int d, const double* const* FW,
                                int64_t k, double tol_rel, double* const* x, double* const* ws, double* const* out,
                                int32_t* const* status) {
  using namespace cc;
  if (d < 1 || d > NC * PW || nprob < 1 || nprob > kMaxProb) return SLRA_ERR_UNSUPPORTED;
  const int np = (d + PW - 1) / PW;
  int nparts = (int)((k + kRC - 1) / kRC);
  if (nparts > 2 * c->num_sms) nparts = 2 * c->num_sms;
  CholArgsN args{};
  for (int b = 0; b < nprob; ++b) {
    double* part = ws[b] + (size_t)np * PANEL + (size_t)np * PW * LDD;
    args.p[b] = CholArgs{Gw[b], d, FW[b], k, tol_rel, x[b], ws[b], part, nparts, out[b], status[b]};
  }
  SLRA_CUDA(cudaFuncSetAttribute(chol_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
  SLRA_TIMED(c, "lsr_solve", chol_cluster_kernel<<<NC * nprob, NT, SMEM, c->stream>>>(args);)
  SLRA_CHECK_LAUNCH(c);
  const size_t sm2 = sizeof(double) * ((size_t)d + 1 + (size_t)(d + 1) * (kRC + 1));
  SLRA_CUDA(cudaFuncSetAttribute(lsq_refine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
  SLRA_TIMED(c, "lsr_solve", lsq_refine_kernel<<<dim3(nparts, nprob), 256, sm2, c->stream>>>(args);)
  SLRA_CHECK_LAUNCH(c);
  SLRA_CUDA(cudaFuncSetAttribute(chol_refine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_REFINE));
  SLRA_TIMED(c, "lsr_solve", chol_refine_kernel<<<NC * nprob, NT, SMEM_REFINE, c->stream>>>(args);)
  SLRA_CHECK_LAUNCH(c);
  return SLRA_OK;
}

int launch_chol_cluster(Context* c, const double* Gw, int d, const double* FW, int64_t k, double tol_rel, double* x,
                        double* ws, double* out, int32_t* status) {
  return launch_chol_cluster_batched(c, 1, &Gw, d, &FW, k, tol_rel, &x, &ws, &out, &status);
}

}  // namespace slra_dev

#ifdef SLRA_CHOL_PROF
extern "C" int slra_debug_chol_marks(unsigned long long* h_out) {
  return cudaMemcpyFromSymbol(h_out, slra_dev::g_chol_marks, sizeof(unsigned long long) * 8 * 64) == cudaSuccess ? 0 : 1;
}
#endif
