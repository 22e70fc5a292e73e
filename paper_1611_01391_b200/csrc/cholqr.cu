// Shifted CholeskyQR3 (Fukaya, Kannan, Nakatsukasa, Yamamoto, Yanagisawa,
// "Shifted Cholesky QR for computing the QR factorization of ill-conditioned
// matrices", SISC 2020) for the tall-skinny sketch Y = M H of the range
// finder (lra.cpp:14-39, thin_qr linalg.cpp:67-79).
//
// Why here: Householder QR of a 4096 x 48 strip is a chain of 48 dependent
// column steps per tree level (latency-bound on one SM per leaf); CholeskyQR
// is three rounds of {Gram, an n x n Cholesky, a row-parallel triangular
// solve}. Pass 1 adds the shift s = 11 (m n + n (n + 1)) u ||Y||_F^2 so the
// Cholesky succeeds for cond(Y) up to ~1/u; passes 2-3 restore orthogonality
// to O(u). R = R3 R2 R1 has a positive diagonal — thin_qr's R(i,i) >= 0
// convention. Q spans the same space as Householder's Q; the range finder
// consumes only the top-r singular subspace of R, which is well conditioned
// here, so the result matches the oracle within tolerance. A Cholesky
// breakdown (cond(Y) beyond ~1/u, e.g. an exactly rank-deficient sketch) sets
// status[b] = 1 and the caller falls back to the Householder TSQR.
//
// Kernels per pass (templated on NP = n rounded up to a multiple of 8, so
// every loop bound is a compile-time constant — FP64 dependent latency is
// ~24 cycles here and index/predicate arithmetic was most of the issue
// slots): gram_partial_kernel (row chunks -> partial NP x NP Grams, no
// atomics), chol_small_kernel (sums the partials in a fixed order, shift,
// Cholesky padded with the identity beyond n, 1/R(i,i)), trsm_rows_kernel
// (Q = Y R^-1, a thread per row, right-looking in registers).
#include <cooperative_groups.h>

#include <cstdlib>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace slra_dev {

constexpr int kCQ = 256;
constexpr int kCQMax = 64;
constexpr int kGR = 128;  // rows per Gram chunk

// P_{b,k} = Y_b(chunk k, :)^T Y_b(chunk k, :) for chunk k = blockIdx.x
// (upper triangle, NP x NP with zero columns beyond n).
template <int NP>
__global__ void __launch_bounds__(kCQ) gram_partial_kernel(const double* __restrict__ Y, int64_t ldy, int64_t sY,
                                                           int64_t m, int n, double* __restrict__ P, int64_t sP,
                                                           const int32_t* __restrict__ status) {
  extern __shared__ __align__(16) double T[];  // chunk rows, ld kGR + 1 per column (odd: conflict-free)
  constexpr int ldt = kGR + 1;
  const int b = blockIdx.y, k = blockIdx.x, tid = threadIdx.x;
  if (status[b]) return;
  Y += b * sY;
  const int64_t r0 = (int64_t)k * kGR;
  const int rows = (int)((m - r0) < kGR ? (m - r0) : kGR);
#pragma unroll 4
  for (int e = tid; e < kGR * NP; e += kCQ) {
    const int i = e % kGR, c = e / kGR;
    T[i + c * ldt] = load_sel(Y, (r0 + i) + (int64_t)c * ldy, i < rows && c < n);
  }
  __syncthreads();
  double* out = P + b * sP + (int64_t)k * NP * NP;
  constexpr int NB = NP / 2;  // 2 x 2 output blocks: four independent FMA chains per thread
  for (int e = tid; e < NB * NB; e += kCQ) {
    const int bi = e % NB, bc = e / NB;
    if (bi > bc) continue;
    const int i0 = 2 * bi, c0 = 2 * bc;
    const double* a0 = T + i0 * ldt;
    const double* d0 = T + c0 * ldt;
    double s00 = 0.0, s01 = 0.0, s10 = 0.0, s11 = 0.0;
#pragma unroll 8
    for (int t = 0; t < kGR; ++t) {
      const double x0 = a0[t], x1 = a0[t + ldt], y0 = d0[t], y1 = d0[t + ldt];
      s00 = fma(x0, y0, s00);
      s01 = fma(x0, y1, s01);
      s10 = fma(x1, y0, s10);
      s11 = fma(x1, y1, s11);
    }
    out[i0 + c0 * NP] = s00;
    out[i0 + (c0 + 1) * NP] = s01;
    out[(i0 + 1) + c0 * NP] = s10;  // below the diagonal when bi == bc: unused
    out[(i0 + 1) + (c0 + 1) * NP] = s11;
  }
}

// Upper Cholesky factor R of G + shift*I (first n entries) padded with the
// identity beyond n, where G = the sum of the nchunk partial Grams (chunk
// order fixed); shift = shift_coef * trace(G). Thread (row ti, phase tc)
// owns L(ti, c) for c = tc, tc + 4, ...: each column step stages column j in
// registers, then writes (two barriers per step). Writes R (n x n, ld n),
// and 1/R(i,i) for all NP entries. A breakdown sets status[b] = 1.
template <int NP>
__global__ void __launch_bounds__(kCQ) chol_small_kernel(const double* __restrict__ P, int64_t sP, int nchunk, int n,
                                                         double shift_coef, double* __restrict__ R, int64_t sR,
                                                         double* __restrict__ rinv, int64_t sRi,
                                                         int32_t* __restrict__ status) {
  constexpr int ld = NP + 1;
  __shared__ double L[NP * ld];  // L(i, c) at i + c * ld, lower triangle
  __shared__ double red[40];
  __shared__ int fail;
  const int b = blockIdx.x, tid = threadIdx.x;
  if (status[b]) return;
  P += b * sP;
  R += b * sR;
  rinv += b * sRi;
  constexpr int NN = NP * NP;
  // upper-triangle entries only, every chunk's partial of an entry in flight
  // at once (the partials are L2 reads: this sum, not the factorisation, was
  // most of the kernel), added in chunk order
  constexpr int NU = NP * (NP + 1) / 2;
  for (int u = tid; u < NU; u += kCQ) {
    int c = (int)((sqrt(8.0 * u + 1.0) - 1.0) * 0.5);  // u = c (c + 1) / 2 + i, i <= c
    while ((c + 1) * (c + 2) / 2 <= u) ++c;
    while (c * (c + 1) / 2 > u) --c;
    const int i = u - c * (c + 1) / 2;
    const int e = i + c * NP;
    double s = 0.0;
    int k = 0;
    for (; k + 16 <= nchunk; k += 16) {
      double v[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) v[t] = P[(k + t) * NN + e];
#pragma unroll
      for (int t = 0; t < 16; ++t) s += v[t];
    }
    for (; k < nchunk; ++k) s += P[k * NN + e];
    L[c + i * ld] = s;  // lower: L(c, i) = G(i, c), c >= i
  }
  __syncthreads();
  double tr = 0.0;
  for (int i = tid; i < n; i += kCQ) tr += L[i + i * ld];
  tr = block_sum<kCQ>(tr, red);
  for (int i = tid; i < NP; i += kCQ) L[i + i * ld] = i < n ? L[i + i * ld] + shift_coef * tr : 1.0;
  if (tid == 0) fail = 0;
  __syncthreads();
  // Column-publishing right-looking factorisation (one barrier per column):
  // thread (i = tid % 64, g = tid / 64) holds A(i, g + 4 v) in registers;
  // column j, once final, sits in L(:, j) (published by its owner group at
  // the end of step j - 1) and every thread applies A(i, c) -= A(i, j) A(c, j)
  // / A(j, j) to all of its entries unconditionally — entries of published
  // columns and above the diagonal take garbage that is never read (the
  // owner of column j + 1 republishes only its unpublished columns). At the
  // end L(i, c) = A(i, c) / sqrt(A(c, c)).
  constexpr int kV = NP / 4;
  __shared__ double piv_s[NP];
  const int ti = tid & 63, tg = tid >> 6;
  double a[kV];
#pragma unroll
  for (int v = 0; v < kV; ++v) {
    const int c = tg + 4 * v;
    a[v] = (ti < NP && ti >= c) ? L[ti + c * ld] : 0.0;
  }
  for (int j = 0; j < NP; ++j) {
    const double* cj = L + j * ld;
    const double piv = cj[j];
    if (!(piv > 0.0)) {  // uniform: every thread read the same pivot
      if (tid == 0) fail = 1;
      break;
    }
    const double rp = piv >= DBL_MIN ? fast_rcp(piv) : 1.0 / piv;
    const double f = (ti > j && ti < NP) ? -cj[ti] * rp : 0.0;
#pragma unroll
    for (int v = 0; v < kV; ++v) a[v] = fma(f, cj[tg + 4 * v], a[v]);
    const int jn = j + 1;
    if (tg == (jn & 3) && ti < NP && jn < NP) {
      const int vv = jn >> 2;
#pragma unroll
      for (int v = 0; v < kV; ++v)
        if (v >= vv) L[ti + (tg + 4 * v) * ld] = a[v];
    }
    if (tid == 0) piv_s[j] = piv;
    __syncthreads();
  }
  if (fail) {
    if (tid == 0) status[b] = 1;
    return;
  }
  // R(i, c) = L(c, i) = A(c, i) / sqrt(A(i, i)) for i < c, sqrt(A(i, i)) on the diagonal
  for (int e = tid; e < n * n; e += kCQ) {
    const int i = e % n, c = e / n;
    const double pi = piv_s[i];
    const double r = fast_rsqrt(pi);
    R[e] = (i < c) ? L[c + i * ld] * r : (i == c ? pi * r : 0.0);
  }
  for (int i = tid; i < NP; i += kCQ) rinv[i] = fast_rsqrt(piv_s[i]);
}

// Q(i, :) = Y(i, :) R^-1 for every row i, one thread per row; problem
// blockIdx.y. R (n x n, ld n) is padded to NP x NP with the identity in
// shared memory; the row lives in registers and the substitution is
// right-looking (each final z(c) updates the later entries), so the
// dependent chain is one multiply + one FMA per column.
template <int NP>
__global__ void __launch_bounds__(128) trsm_rows_kernel(const double* __restrict__ Y, int64_t ldy, int64_t sY,
                                                        int64_t m, int n, const double* __restrict__ R, int64_t sR,
                                                        const double* __restrict__ rinv, int64_t sRi,
                                                        double* __restrict__ Q, int64_t ldq, int64_t sQ,
                                                        const int32_t* __restrict__ status) {
  __shared__ double Rs[NP * NP];
  __shared__ double ri[NP];
  const int b = blockIdx.y, tid = threadIdx.x;
  if (status[b]) return;
  Y += b * sY;
  Q += b * sQ;
  R += b * sR;
  rinv += b * sRi;
  for (int e = tid; e < NP * NP; e += 128) {
    const int r = e % NP, c = e / NP;
    Rs[e] = (r < n && c < n) ? R[r + c * n] : (r == c ? 1.0 : 0.0);
  }
  for (int c = tid; c < NP; c += 128) ri[c] = rinv[c];
  __syncthreads();
  const int64_t i = blockIdx.x * 128LL + tid;
  if (i >= m) return;
  double zr[NP];
#pragma unroll
  for (int c = 0; c < NP; ++c) zr[c] = load_sel(Y + i, (int64_t)c * ldy, c < n);
#pragma unroll
  for (int c = 0; c < NP; ++c) {
    const double z = zr[c] * ri[c];
    zr[c] = z;
#pragma unroll
    for (int c2 = c + 1; c2 < NP; ++c2) zr[c2] = fma(-z, Rs[c + c2 * NP], zr[c2]);
  }
#pragma unroll
  for (int c = 0; c < NP; ++c)
    if (c < n) Q[i + (int64_t)c * ldq] = zr[c];
}

// R = (R3 R2) R1 for upper-triangular n x n factors (ld n), problem
// blockIdx.x, operands staged in shared memory.
__global__ void __launch_bounds__(kCQ) trmm3_upper_kernel(const double* __restrict__ R1, const double* __restrict__ R2,
                                                          const double* __restrict__ R3, int64_t sIn, int n,
                                                          double* __restrict__ Rout, int64_t sOut, int64_t ldo,
                                                          const int32_t* __restrict__ status) {
  extern __shared__ __align__(16) double tm[];
  const int b = blockIdx.x, tid = threadIdx.x;
  if (status[b]) return;
  const int nn = n * n;
  double* A = tm;
  double* B = tm + nn;
  for (int e = tid; e < nn; e += kCQ) {
    A[e] = R3[b * sIn + e];
    B[e] = R2[b * sIn + e];
  }
  __syncthreads();
  constexpr int kPer = (kCQMax * kCQMax + kCQ - 1) / kCQ;
  double t3[kPer];
#pragma unroll
  for (int q = 0; q < kPer; ++q) {  // T = R3 R2 (upper)
    const int e = tid + q * kCQ;
    double acc = 0.0;
    if (e < nn) {
      const int i = e % n, c = e / n;
      for (int t = i; t <= c; ++t) acc = fma(A[i + t * n], B[t + c * n], acc);
    }
    t3[q] = acc;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int e = tid + q * kCQ;
    if (e < nn) {
      A[e] = t3[q];
      B[e] = R1[b * sIn + e];
    }
  }
  __syncthreads();
  for (int e = tid; e < nn; e += kCQ) {  // R = T R1
    const int i = e % n, c = e / n;
    double acc = 0.0;
    for (int t = i; t <= c; ++t) acc = fma(A[i + t * n], B[t + c * n], acc);
    Rout[b * sOut + i + (int64_t)c * ldo] = i <= c ? acc : 0.0;
  }
}


// ------------------------------------------------------------ fused cluster path
// The three passes in ONE launch when the sketch fits the shared memory of an
// 8-CTA thread-block cluster (config 2: 4096 x 48 -> 512 rows x 48 columns =
// 198 KB per CTA): CTA q keeps rows q RC .. (q + 1) RC - 1 of the problem
// resident for all three passes. Per pass: the chunk's Gram on DMMA (each
// warp runs every upper 8 x 8 tile over its share of the 4-row steps: one
// fragment load per 8 columns serves as A and B operand), a fixed-order sum
// over the warps, a fixed-order sum of the eight CTAs' partials over DSMEM
// (every CTA ends with the same bits), the 48-step Cholesky redundantly in
// every CTA (no broadcast of the factor), and the row-parallel triangular
// solve in place. Q leaves once, after pass 3; R = R3 (R2 R1) is formed along
// the way, an eighth of the entries per CTA.
#ifdef SLRA_CQC_PROF
#define CQC_MARK(i) do { if (tid == 0 && q == 0 && b == 0) pt[i] = clock64(); } while (0)
#else
#define CQC_MARK(i) do { } while (0)
#endif
namespace cqc {
// TMA bulk copies (cp.async.bulk) between the chunk's contiguous columns in
// global memory and shared memory; completion of the loads on an mbarrier
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
constexpr int NC = 8;
constexpr int NT = 256;
constexpr int kMaxSmem = 227 * 1024;
__host__ __device__ inline int chunk_rows(int64_t m) { return (int)((m + NC - 1) / NC); }
// leading dimension of the chunk: >= rows, = 4 (mod 16) so the DMMA fragment
// loads (lane (g, t) reads row k + t of column 8 I + g) hit 16 different banks
__host__ __device__ inline int chunk_ld(int rc) { return ((rc + 11) / 16) * 16 + 4; }
template <int NP>
struct Lay {
  static constexpr int LD = NP + 2;  // even: the solve reads pairs of R entries as double2
  static constexpr int NTILE = NP / 8;
  static constexpr int NUT = NTILE * (NTILE + 1) / 2;
  static constexpr int L_D = NP * LD;
  static constexpr int PU_D = NUT * 64;
  static constexpr int SMALL_D = 2 * NP + 40 + 2;  // pivots, 1/R(i,i), reduction scratch, fail flag, mbarrier
  static size_t bytes(int ldt) { return sizeof(double) * ((size_t)NP * ldt + L_D + PU_D + SMALL_D); }
};
}  // namespace cqc

template <int NP>
__global__ void __cluster_dims__(cqc::NC, 1, 1) __launch_bounds__(cqc::NT, 1)
    cholqr3_cluster_kernel(const double* __restrict__ Y, int64_t ldy, int64_t sY, int64_t m, int n,
                           double* __restrict__ Q, int64_t ldq, int64_t sQ, double* __restrict__ R, int64_t sR,
                           double* __restrict__ Rws, int64_t sRws, double shift_coef, int ldt,
                           int32_t* __restrict__ status) {
  using namespace cqc;
  using LY = Lay<NP>;
  constexpr int LD = LY::LD, NTILE = LY::NTILE, NUT = LY::NUT;
  extern __shared__ __align__(16) double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank();
  const int b = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  Y += b * sY;
  Q += b * sQ;
  R += b * sR;
  Rws += b * sRws;
  const int RC = chunk_rows(m);
  const int64_t r0 = (int64_t)q * RC;
  const int rows = (int)(m - r0 < 0 ? 0 : (m - r0 < RC ? m - r0 : RC));
  double* T = sm;                      // NP columns x ldt
  double* L = T + (size_t)NP * ldt;    // NP x LD
  double* PU = L + LY::L_D;            // this CTA's partial Gram, upper tiles in fragment order
  double* piv_s = PU + LY::PU_D;       // NP
  double* rinv = piv_s + NP;           // NP
  double* red = rinv + NP;             // 40
  int* fail = reinterpret_cast<int*>(red + 40);
#ifdef SLRA_CQC_PROF
  long long pt[32];
#endif
  CQC_MARK(0);
  // the chunk, zero beyond the problem (rows >= rows, columns >= n): one TMA
  // bulk copy per column when the alignment allows (16-byte source and size)
  uint64_t* mbar = reinterpret_cast<uint64_t*>(red + 41);
  const bool bulk_in = rows > 0 && (rows & 1) == 0 && (ldy & 1) == 0 && ((uintptr_t)(Y + r0) & 15) == 0;
  if (tid == 0) {
    *fail = 0;
    if (bulk_in) mbar_init(mbar, 1);
  }
  __syncthreads();
  if (bulk_in) {
    if (warp == 0) {
      if (lane == 0) mbar_arrive_expect_tx(mbar, (unsigned)(n * rows * 8));
      __syncwarp();
      for (int c = lane; c < n; c += 32)
        bulk_g2s(T + (size_t)c * ldt, Y + r0 + (int64_t)c * ldy, (unsigned)(rows * 8), mbar);
    }
    for (int c = warp; c < NP; c += NT / 32) {
      double* tc = T + (size_t)c * ldt;
      for (int i = (c < n ? rows : 0) + lane; i < ldt; i += 32) tc[i] = 0.0;
    }
    mbar_wait(mbar, 0);
  } else {
    for (int c = warp; c < NP; c += NT / 32) {
      const double* yc = Y + r0 + (int64_t)c * ldy;
      double* tc = T + (size_t)c * ldt;
      for (int i0 = lane; i0 < ldt; i0 += 32 * 8) {  // eight loads in flight per lane
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = load_sel(yc, (int64_t)(i0 + 32 * k), i0 + 32 * k < rows && c < n);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (i0 + 32 * k < ldt) tc[i0 + 32 * k] = v[k];
      }
    }
  }
  __syncthreads();
  CQC_MARK(1);
  const int ksteps = (RC + 3) / 4;
  for (int pass = 0; pass < 3; ++pass) {
    // ---- partial Gram of the chunk (upper tiles)
    double acc[NUT][2];
#pragma unroll
    for (int u = 0; u < NUT; ++u) acc[u][0] = acc[u][1] = 0.0;
    for (int ks = warp; ks < ksteps; ks += NT / 32) {
      const double* tk = T + 4 * ks + t + (size_t)g * ldt;
      double f[NTILE];
#pragma unroll
      for (int I = 0; I < NTILE; ++I) f[I] = tk[(size_t)(8 * I) * ldt];
      int u = 0;
#pragma unroll
      for (int I = 0; I < NTILE; ++I)
#pragma unroll
        for (int J = I; J < NTILE; ++J) {
          dmma_8x8x4(acc[u][0], acc[u][1], f[I], f[J]);
          ++u;
        }
    }
    CQC_MARK(2 + 8 * pass);
    // warps summed in warp order (lane (g, t) holds entries (g, 2t), (g, 2t + 1) of each tile)
    for (int w = 0; w < NT / 32; ++w) {
      if (warp == w) {
#pragma unroll
        for (int u = 0; u < NUT; ++u) {
          double2* dst = reinterpret_cast<double2*>(PU + u * 64 + 8 * g + 2 * t);
          double2 v = make_double2(acc[u][0], acc[u][1]);
          if (w > 0) {
            const double2 o = *dst;
            v.x += o.x;
            v.y += o.y;
          }
          *dst = v;
        }
      }
      __syncthreads();
    }
    CQC_MARK(3 + 8 * pass);
    cl.sync();  // every CTA's partial is complete
    CQC_MARK(4 + 8 * pass);
    // ---- G = sum over the CTAs in rank order -> L (lower storage: L(c, i) = G(i, c))
    {
      constexpr int DS_IT = (NUT * 64 + NT - 1) / NT;
      double v[DS_IT][NC];  // every remote load in flight before the first sum
#pragma unroll
      for (int it = 0; it < DS_IT; ++it) {
        const int e = tid + it * NT;
#pragma unroll
        for (int rk = 0; rk < NC; ++rk) v[it][rk] = e < NUT * 64 ? cl.map_shared_rank(PU, rk)[e] : 0.0;
      }
#pragma unroll
      for (int it = 0; it < DS_IT; ++it) {
        const int e = tid + it * NT;
        int u = e >> 6, I = 0;
        while (u >= NTILE - I && I < NTILE) {
          u -= NTILE - I;
          ++I;
        }
        const int J = I + u;
        const int i = 8 * I + ((e & 63) >> 3), c = 8 * J + (e & 7);
        double s = v[it][0];
#pragma unroll
        for (int rk = 1; rk < NC; ++rk) s += v[it][rk];
        if (e < NUT * 64 && i <= c) L[c + i * LD] = s;
      }
    }
    cl.sync();  // the partials may be overwritten (next pass); L is complete in this CTA
    CQC_MARK(5 + 8 * pass);
    double tr = 0.0;
    for (int i = tid; i < n; i += NT) tr += L[i + i * LD];
    tr = block_sum<NT>(tr, red);
    const double shift = pass == 0 ? shift_coef * tr : 0.0;
    for (int i = tid; i < NP; i += NT) L[i + i * LD] = i < n ? L[i + i * LD] + shift : 1.0;
    __syncthreads();
    CQC_MARK(6 + 8 * pass);
    // ---- Cholesky (chol_small_kernel's column-publishing loop), redundantly per CTA
    {
      constexpr int kV = NP / 4;
      const int ti = tid & 63, tg = tid >> 6;
      double a[kV];
#pragma unroll
      for (int v = 0; v < kV; ++v) {
        const int c = tg + 4 * v;
        a[v] = (ti < NP && ti >= c) ? L[ti + c * LD] : 0.0;
      }
      for (int j = 0; j < NP; ++j) {
        const double* cj = L + j * LD;
        const double piv = cj[j];
        if (!(piv > 0.0)) {  // uniform over the CTA and (same bits) over the cluster
          if (tid == 0) *fail = 1;
          break;
        }
        const double rp = piv >= DBL_MIN ? fast_rcp(piv) : 1.0 / piv;
        const double f = (ti > j && ti < NP) ? -cj[ti] * rp : 0.0;
#pragma unroll
        for (int v = 0; v < kV; ++v) a[v] = fma(f, cj[tg + 4 * v], a[v]);
        const int jn = j + 1;
        if (tg == (jn & 3) && ti < NP && jn < NP) {
          const int vv = jn >> 2;
#pragma unroll
          for (int v = 0; v < kV; ++v)
            if (v >= vv) L[ti + (tg + 4 * v) * LD] = a[v];
        }
        if (tid == 0) piv_s[j] = piv;
        __syncthreads();
      }
    }
    __syncthreads();
    CQC_MARK(7 + 8 * pass);
    if (*fail) {
      if (q == 0 && tid == 0) status[b] = 1;
      return;  // cluster-uniform; no DSMEM access is pending (second cl.sync above)
    }
    // R^T in place: L(c2, c) <- R(c, c2) = A(c2, c) / sqrt(A(c, c)) below the diagonal
    for (int i = tid; i < NP; i += NT) rinv[i] = fast_rsqrt(piv_s[i]);
    __syncthreads();
    for (int e = tid; e < NP * NP; e += NT) {
      const int c2 = e % NP, c = e / NP;
      if (c2 > c) L[c2 + c * LD] *= rinv[c];
    }
    // R = R3 (R2 R1), an eighth of the entries per CTA: the left factor is this
    // pass's R (in L), the right one (R1, then R2 R1) comes from global memory
    // (written before the two cluster barriers of this pass) staged packed
    // upper-triangular over the partial-Gram buffer, which is idle here
    const int nn = n * n;
    if (pass > 0) {
      const double* Gs = Rws + (int64_t)(pass - 1) * nn;
      for (int e = tid; e < nn; e += NT) {
        const int k = e % n, c = e / n;
        if (k <= c) PU[c * (c + 1) / 2 + k] = Gs[e];
      }
    }
    __syncthreads();
    if (pass == 0) {
      if (q == 0)
        for (int e = tid; e < nn; e += NT) {
          const int i = e % n, c = e / n;
          Rws[e] = (i < c) ? L[c + i * LD] : (i == c ? piv_s[i] * rinv[i] : 0.0);
        }
    } else {
      const int per = (nn + NC - 1) / NC;
      const int e1 = (q + 1) * per < nn ? (q + 1) * per : nn;
      double* out = pass == 1 ? Rws + nn : R;
      for (int e = q * per + tid; e < e1; e += NT) {
        const int i = e % n, c = e / n;
        double s = 0.0;
        if (i <= c) {
          const double* pc = PU + c * (c + 1) / 2;
          s = piv_s[i] * rinv[i] * pc[i];
          for (int k = i + 1; k <= c; ++k) s = fma(L[k + i * LD], pc[k], s);
        }
        out[e] = s;
      }
    }
    CQC_MARK(8 + 8 * pass);
    // ---- rows <- rows R^-1 in place (a thread per row, right-looking in registers)
    for (int i = tid; i < rows; i += NT) {
      double zr[NP];
#pragma unroll
      for (int c = 0; c < NP; ++c) zr[c] = T[i + (size_t)c * ldt];
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        const double z = zr[c] * rinv[c];
        zr[c] = z;
        const double* rc = L + c * LD;  // R(c, c2) at rc[c2], c2 > c
        int c2 = c + 1;
        if (c2 & 1) {
          if (c2 < NP) zr[c2] = fma(-z, rc[c2], zr[c2]);
          ++c2;
        }
#pragma unroll
        for (; c2 + 1 < NP; c2 += 2) {
          const double2 rr = *reinterpret_cast<const double2*>(rc + c2);
          zr[c2] = fma(-z, rr.x, zr[c2]);
          zr[c2 + 1] = fma(-z, rr.y, zr[c2 + 1]);
        }
      }
#pragma unroll
      for (int c = 0; c < NP; ++c) T[i + (size_t)c * ldt] = zr[c];
    }
    __syncthreads();
    CQC_MARK(9 + 8 * pass);
  }
  // ---- Q out (TMA bulk stores of the columns when aligned)
  const bool bulk_out = rows > 0 && (rows & 1) == 0 && (ldq & 1) == 0 && ((uintptr_t)(Q + r0) & 15) == 0;
  if (bulk_out) {
    if (warp == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the solve's generic writes before the async reads
      for (int c = lane; c < n; c += 32)
        bulk_s2g(Q + r0 + (int64_t)c * ldq, T + (size_t)c * ldt, (unsigned)(rows * 8));
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // the sources read; the writes land by grid end
    }
  } else {
    for (int c = warp; c < n; c += NT / 32) {
      double* qc = Q + r0 + (int64_t)c * ldq;
      const double* tc = T + (size_t)c * ldt;
#pragma unroll 8
      for (int i = lane; i < rows; i += 32) qc[i] = tc[i];
    }
  }
#ifdef SLRA_CQC_PROF
  __syncthreads();
  if (tid == 0 && b == 0 && q == 0) {
    pt[26] = clock64();
    printf("cqc load %lld |", pt[1] - pt[0]);
    for (int p = 0; p < 3; ++p)
      printf(" pass%d gram %lld wsum %lld clsync %lld dsum %lld shift %lld chol %lld rt %lld trsm %lld |", p,
             pt[2 + 8 * p] - (p ? pt[1 + 8 * p] : pt[1]), pt[3 + 8 * p] - pt[2 + 8 * p], pt[4 + 8 * p] - pt[3 + 8 * p],
             pt[5 + 8 * p] - pt[4 + 8 * p], pt[6 + 8 * p] - pt[5 + 8 * p], pt[7 + 8 * p] - pt[6 + 8 * p],
             pt[8 + 8 * p] - pt[7 + 8 * p], pt[9 + 8 * p] - pt[8 + 8 * p]);
    printf(" tail %lld total %lld\n", pt[26] - pt[25], pt[26] - pt[0]);
  }
#endif
}

// SLRA_NO_CLUSTER_CHOLQR=1: the multi-kernel path for every shape (tests of the fallback)
static bool cluster_path_disabled() {
  const char* e = getenv("SLRA_NO_CLUSTER_CHOLQR");
  return e && e[0] == '1';
}

template <int NP>
static bool cholqr3_cluster_fits(int64_t m, int n) {
  if (m > (int64_t)cqc::NC * 4096) return false;
  const int ldt = cqc::chunk_ld(cqc::chunk_rows(m));
  return cqc::Lay<NP>::bytes(ldt) <= (size_t)cqc::kMaxSmem;
}

template <int NP>
static int cholqr3_cluster(Context* cx, const double* Y, int64_t ldy, int64_t sY, int64_t m, int n, double* Q,
                           int64_t ldq, int64_t sQ, double* R, int64_t sR, int nb, double* ws, int64_t per,
                           int32_t* status) {
  const int ldt = cqc::chunk_ld(cqc::chunk_rows(m));
  const size_t smem = cqc::Lay<NP>::bytes(ldt);
  const double shift_coef = 11.0 * ((double)m * n + (double)n * (n + 1)) * (2.220446049250313e-16 / 2);  // u = eps/2
  SLRA_CUDA(cudaFuncSetAttribute(cholqr3_cluster_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SLRA_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t) * nb, cx->stream));
  SLRA_TIMED(cx, "cholqr_cluster",
             cholqr3_cluster_kernel<NP><<<dim3(cqc::NC, (unsigned)nb), cqc::NT, smem, cx->stream>>>(
                 Y, ldy, sY, m, n, Q, ldq, sQ, R, sR, ws, per, shift_coef, ldt, status);)
  SLRA_CHECK_LAUNCH(cx);
  return SLRA_OK;
}

static int64_t gram_chunks(int64_t m) { return (m + kGR - 1) / kGR; }

size_t cholqr3_workspace_doubles(int64_t m, int n) {
  return (size_t)m * n + (size_t)gram_chunks(m) * kCQMax * kCQMax + 3 * (size_t)n * n + kCQMax + 8;
}

template <int NP>
static int cholqr3_passes(Context* cx, const double* Y, int64_t ldy, int64_t sY, int64_t m, int n, double* Q,
                          int64_t ldq, int64_t sQ, double* R, int64_t ldr, int64_t sR, int nb, double* ws,
                          int32_t* status) {
  const int64_t per = (int64_t)cholqr3_workspace_doubles(m, n);
  const int64_t nn = (int64_t)n * n, nch = gram_chunks(m);
  if (cholqr3_cluster_fits<NP>(m, n) && !cluster_path_disabled())
    return cholqr3_cluster<NP>(cx, Y, ldy, sY, m, n, Q, ldq, sQ, R, sR, nb, ws, per, status);
  // per problem: T (m x n) | partial Grams (nch x NP x NP) | R1 | R2 | R3 | rinv (NP)
  double* T = ws;
  double* P = ws + m * n;
  double* R1 = P + nch * kCQMax * kCQMax;
  double* rinv = R1 + 3 * nn;
  const double shift_coef = 11.0 * ((double)m * n + (double)n * (n + 1)) * (2.220446049250313e-16 / 2);  // u = eps/2
  const size_t gsm_bytes = sizeof(double) * (size_t)(kGR + 1) * NP;
  SLRA_CUDA(cudaFuncSetAttribute(gram_partial_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)gsm_bytes));
  SLRA_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t) * nb, cx->stream));
  const double* src[3] = {Y, Q, T};
  const int64_t lds[3] = {ldy, ldq, m}, ss[3] = {sY, sQ, per};
  double* dst[3] = {Q, T, Q};
  const int64_t ldd[3] = {ldq, m, ldq}, sd[3] = {sQ, per, sQ};
  const dim3 gg((unsigned)nch, (unsigned)nb), tg((unsigned)((m + 127) / 128), (unsigned)nb);
  for (int pass = 0; pass < 3; ++pass) {
    double* Rk = R1 + pass * nn;
    SLRA_TIMED(cx, "cholqr_gram", gram_partial_kernel<NP><<<gg, kCQ, gsm_bytes, cx->stream>>>(
                                      src[pass], lds[pass], ss[pass], m, n, P, per, status);)
    SLRA_CHECK_LAUNCH(cx);
    SLRA_TIMED(cx, "cholqr_chol",
               chol_small_kernel<NP><<<nb, kCQ, 0, cx->stream>>>(P, per, (int)nch, n, pass == 0 ? shift_coef : 0.0,
                                                                 Rk, per, rinv, per, status);)
    SLRA_CHECK_LAUNCH(cx);
    SLRA_TIMED(cx, "cholqr_trsm",
               trsm_rows_kernel<NP><<<tg, 128, 0, cx->stream>>>(src[pass], lds[pass], ss[pass], m, n, Rk, per, rinv,
                                                                per, dst[pass], ldd[pass], sd[pass], status);)
    SLRA_CHECK_LAUNCH(cx);
  }
  const size_t msm_bytes = sizeof(double) * 2 * (size_t)nn;
  SLRA_CUDA(cudaFuncSetAttribute(trmm3_upper_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msm_bytes));
  SLRA_TIMED(cx, "cholqr_trmm", trmm3_upper_kernel<<<nb, kCQ, msm_bytes, cx->stream>>>(R1, R1 + nn, R1 + 2 * nn, per,
                                                                                        n, R, sR, ldr, status);)
  SLRA_CHECK_LAUNCH(cx);
  return SLRA_OK;
}

// Batched shifted CholeskyQR3 of nb problems Y_b (m x n, n <= 64): Q_b
// (ld ldq) and R_b (ld n) as thin_qr. ws: nb * cholqr3_workspace_doubles.
// status (device, nb ints) is zeroed here; status[b] != 0 marks a breakdown.
int launch_cholqr3_batched(Context* cx, const double* Y, int64_t ldy, int64_t sY, int64_t m, int n, double* Q,
                           int64_t ldq, int64_t sQ, double* R, int64_t ldr, int64_t sR, int nb, double* ws,
                           int32_t* status) {
  if (n < 1 || n > kCQMax || ldr != n || m < n) return SLRA_ERR_UNSUPPORTED;
  switch ((n + 7) / 8) {
    case 1: return cholqr3_passes<8>(cx, Y, ldy, sY, m, n, Q, ldq, sQ, R, ldr, sR, nb, ws, status);
    case 2: return cholqr3_passes<16>(cx, Y, ldy, sY, m, n, Q, ldq, sQ, R, ldr, sR, nb, ws, status);
    case 3: return cholqr3_passes<24>(cx, Y, ldy, sY, m, n, Q, ldq, sQ, R, ldr, sR, nb, ws, status);
    case 4: return cholqr3_passes<32>(cx, Y, ldy, sY, m, n, Q, ldq, sQ, R, ldr, sR, nb, ws, status);
    case 5: return cholqr3_passes<40>(cx, Y, ldy, sY, m, n, Q, ldq, sQ, R, ldr, sR, nb, ws, status);
    case 6: return cholqr3_passes<48>(cx, Y, ldy, sY, m, n, Q, ldq, sQ, R, ldr, sR, nb, ws, status);
    case 7: return cholqr3_passes<56>(cx, Y, ldy, sY, m, n, Q, ldq, sQ, R, ldr, sR, nb, ws, status);
    default: return cholqr3_passes<64>(cx, Y, ldy, sY, m, n, Q, ldq, sQ, R, ldr, sR, nb, ws, status);
  }
}

}  // namespace slra_dev
