// K-c: the FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) kernels.
//   * lowrank_residual: ||A - P Q||_F^2 and ||A||_F^2 in ONE pass over A —
//     P*Q tiles on the tensor pipe, subtract-square-reduce fused in the
//     epilogue, deterministic two-stage reduction. This is the reference's
//     cur_evaluate(M, c, Frobenius) = ||M - (C U) R||_F (cur.cpp:76-82,
//     linalg.cpp:139) and ||M - U V||_F of the range finder (lra.cpp:35-36),
//     with the m x n temporary never materialised.
//   * gemm: C = alpha op(A) op(B) + beta C for the small/skinny products of
//     the path (Eigen GEMMs at cur.cpp:76-78, lra.cpp:35-36, lsr.cpp:58).
#include "common.cuh"

namespace slra_dev {

constexpr int kRT = 256;       // threads per CTA (8 warps)
constexpr int kBM = 64;        // tile rows
constexpr int kBN = 64;        // tile cols
constexpr int kKC = 32;        // inner-dimension chunk staged in smem
constexpr int kLD = kBM + 4;   // smem leading dim: conflict-free fragment reads

// Warp layout: 2 (rows) x 4 (cols) warps, each a 32 x 16 sub-tile = 4 x 2
// m8n8 fragments.
struct ResidualArgs {
  const double* A;
  int64_t lda, m, n;
  const double* P;
  int64_t ldp;
  const double* Q;
  int64_t ldq;
  int64_t inner;
  // batching: problem b uses A + b*sA, P + b*sP, Q + b*sQ
  int64_t nprob, sA, sP, sQ;
  double* out;   // per-CTA partials (single problem) or per-problem results
  int per_problem;
};

__device__ __forceinline__ void stage_pq(const ResidualArgs& a, const double* P, const double* Q, int64_t i0,
                                         int64_t j0, int64_t k0, int kc, double* Ps, double* Qs) {
  // Ps[kk*kLD + i] = P(i0+i, k0+kk); Qs[kk*kLD + j] = Q(k0+kk, j0+j)
  for (int e = threadIdx.x; e < kKC * kBM; e += kRT) {
    const int i = e % kBM, kk = e / kBM;
    double v = 0.0;
    if (kk < kc && i0 + i < a.m) v = P[(i0 + i) + (k0 + kk) * a.ldp];
    Ps[kk * kLD + i] = v;
  }
  for (int e = threadIdx.x; e < kKC * kBN; e += kRT) {
    const int kk = e % kKC, j = e / kKC;
    double v = 0.0;
    if (kk < kc && j0 + j < a.n) v = Q[(k0 + kk) + (j0 + j) * a.ldq];
    Qs[kk * kLD + j] = v;
  }
}

__global__ void __launch_bounds__(kRT, 2) lowrank_residual_kernel(ResidualArgs a) {
  __shared__ double Ps[kKC * kLD];
  __shared__ double Qs[kKC * kLD];
  __shared__ double red[40];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, t4 = lane & 3;
  const int64_t tiles_m = (a.m + kBM - 1) / kBM, tiles_n = (a.n + kBN - 1) / kBN;
  const int64_t tiles = tiles_m * tiles_n;

  double rs = 0.0, ns = 0.0;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t prob = 0;
    const double* A = a.A + prob * a.sA;
    const double* P = a.P + prob * a.sP;
    const double* Q = a.Q + prob * a.sQ;
    const int64_t i0 = (tile % tiles_m) * kBM, j0 = (tile / tiles_m) * kBN;

    // Issue the 16 A loads of this lane first (latency overlaps the MMAs).
    double av[4][2][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t r = i0 + wm * 32 + mi * 8 + g;
          const int64_t cc = j0 + wn * 16 + ni * 8 + 2 * t4 + e;
          av[mi][ni][e] = (r < a.m && cc < a.n) ? __ldg(A + r + cc * a.lda) : 0.0;
        }

    double acc[4][2][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

    for (int64_t k0 = 0; k0 < a.inner; k0 += kKC) {
      const int kc = (int)((a.inner - k0) < kKC ? (a.inner - k0) : kKC);
      __syncthreads();
      stage_pq(a, P, Q, i0, j0, k0, kc, Ps, Qs);
      __syncthreads();
      const int kc4 = (kc + 3) & ~3;
      for (int kk = 0; kk < kc4; kk += 4) {
        double af[4], bf[2];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) af[mi] = Ps[(kk + t4) * kLD + wm * 32 + mi * 8 + g];
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) bf[ni] = Qs[(kk + t4) * kLD + wn * 16 + ni * 8 + g];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
      }
    }
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double x = av[mi][ni][e];
          const double d = x - acc[mi][ni][e];
          rs += d * d;
          ns += x * x;
        }

  }
  const double r1 = block_sum<kRT>(rs, red);
  const double n1 = block_sum<kRT>(ns, red);
  if (threadIdx.x == 0) {
    a.out[2 * blockIdx.x] = r1;
    a.out[2 * blockIdx.x + 1] = n1;
  }
}

// Per-problem mode needs each problem's tiles on one CTA: iterate problems.
__global__ void __launch_bounds__(kRT, 2) lowrank_residual_batched_kernel(ResidualArgs a) {
  __shared__ double Ps[kKC * kLD];
  __shared__ double Qs[kKC * kLD];
  __shared__ double red[40];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, t4 = lane & 3;
  const int64_t tiles_m = (a.m + kBM - 1) / kBM, tiles_n = (a.n + kBN - 1) / kBN;
  const int64_t tiles = tiles_m * tiles_n;
  for (int64_t prob = blockIdx.x; prob < a.nprob; prob += gridDim.x) {
    const double* A = a.A + prob * a.sA;
    const double* P = a.P + prob * a.sP;
    const double* Q = a.Q + prob * a.sQ;
    double rs = 0.0, ns = 0.0;
    for (int64_t tile = 0; tile < tiles; ++tile) {
      const int64_t i0 = (tile % tiles_m) * kBM, j0 = (tile / tiles_m) * kBN;
      double av[4][2][2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int64_t r = i0 + wm * 32 + mi * 8 + g;
            const int64_t cc = j0 + wn * 16 + ni * 8 + 2 * t4 + e;
            av[mi][ni][e] = (r < a.m && cc < a.n) ? __ldg(A + r + cc * a.lda) : 0.0;
          }
      double acc[4][2][2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
      for (int64_t k0 = 0; k0 < a.inner; k0 += kKC) {
        const int kc = (int)((a.inner - k0) < kKC ? (a.inner - k0) : kKC);
        __syncthreads();
        stage_pq(a, P, Q, i0, j0, k0, kc, Ps, Qs);
        __syncthreads();
        const int kc4 = (kc + 3) & ~3;
        for (int kk = 0; kk < kc4; kk += 4) {
          double af[4], bf[2];
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) af[mi] = Ps[(kk + t4) * kLD + wm * 32 + mi * 8 + g];
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) bf[ni] = Qs[(kk + t4) * kLD + wn * 16 + ni * 8 + g];
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
        }
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double x = av[mi][ni][e];
            const double d = x - acc[mi][ni][e];
            rs += d * d;
            ns += x * x;
          }
    }
    const double r1 = block_sum<kRT>(rs, red);
    const double n1 = block_sum<kRT>(ns, red);
    if (threadIdx.x == 0) {
      a.out[2 * prob] = r1;
      a.out[2 * prob + 1] = n1;
    }
  }
}

// Fixed-order reduction of per-CTA (resid, norm) partial pairs.
__global__ void reduce_pairs_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double red[40];
  double r = 0.0, s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    r += part[2 * i];
    s += part[2 * i + 1];
  }
  r = block_sum<256>(r, red);
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) {
    out[0] = r;
    out[1] = s;
  }
}

int launch_residual_stream(Context* c, const double* A, int64_t lda, int64_t m, int64_t n, const double* P,
                           int64_t ldp, const double* Q, int64_t ldq, int64_t inner, double* d_out);
int launch_tn_skinny(Context* c, const char* fam, int64_t r, int64_t n, int64_t K, double alpha, const double* W,
                     int64_t ldw, const double* B, int64_t ldb, double* Cm, int64_t ldc);

int launch_lowrank_residual(Context* c, const double* A, int64_t lda, int64_t m, int64_t n, const double* P,
                            int64_t ldp, const double* Q, int64_t ldq, int64_t inner, double* d_out) {
  // pipelined streaming kernel when the operands suit it (stream_dmma.cu)
  const int st = launch_residual_stream(c, A, lda, m, n, P, ldp, Q, ldq, inner, d_out);
  if (st != SLRA_ERR_UNSUPPORTED) return st;
  ResidualArgs a{A, lda, m, n, P, ldp, Q, ldq, inner, 1, 0, 0, 0, nullptr, 0};
  const int64_t tiles = ((m + kBM - 1) / kBM) * ((n + kBN - 1) / kBN);
  int grid = c->num_sms * 2;
  if (tiles < grid) grid = (int)(tiles > 0 ? tiles : 1);
  double* part = partials(c, 2 * grid);
  if (!part) return SLRA_ERR_CUDA;
  a.out = part;
  SLRA_TIMED(c, "residual", lowrank_residual_kernel<<<grid, kRT, 0, c->stream>>>(a);)
  SLRA_CHECK_LAUNCH(c);
  SLRA_TIMED(c, "residual_reduce", reduce_pairs_kernel<<<1, 256, 0, c->stream>>>(part, grid, d_out);)
  SLRA_CHECK_LAUNCH(c);
  return SLRA_OK;
}

int launch_lowrank_residual_batched(Context* c, const double* A, int64_t lda, int64_t sA, int64_t m, int64_t n,
                                    const double* P, int64_t ldp, int64_t sP, const double* Q, int64_t ldq,
                                    int64_t sQ, int64_t inner, int64_t nprob, double* d_out_pairs) {
  ResidualArgs a{A, lda, m, n, P, ldp, Q, ldq, inner, nprob, sA, sP, sQ, d_out_pairs, 1};
  int grid = c->num_sms * 2;
  if (nprob < grid) grid = (int)nprob;
  SLRA_TIMED(c, "residual_batched", lowrank_residual_batched_kernel<<<grid, kRT, 0, c->stream>>>(a);)
  SLRA_CHECK_LAUNCH(c);
  return SLRA_OK;
}

// ---------------------------------------------------------------- GEMM
constexpr int kGK = 16;  // k-tile

struct GemmArgs {
  int ta, tb;
  int64_t m, n, k;
  double alpha, beta;
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* Cm;
  int64_t ldc;
  int64_t ksplit;   // k range per z-slice
  double* partial;  // split-K partial outputs (m x n per slice, ld = m) or null
};

__device__ __forceinline__ double ldA(const GemmArgs& g, int64_t i, int64_t kk) {
  if (i >= g.m || kk >= g.k) return 0.0;
  return g.ta ? __ldg(g.A + kk + i * g.lda) : __ldg(g.A + i + kk * g.lda);
}
__device__ __forceinline__ double ldB(const GemmArgs& g, int64_t kk, int64_t j) {
  if (j >= g.n || kk >= g.k) return 0.0;
  return g.tb ? __ldg(g.B + j + kk * g.ldb) : __ldg(g.B + kk + j * g.ldb);
}

__global__ void __launch_bounds__(kRT) gemm_kernel(GemmArgs g) {
  __shared__ double As[kGK * kLD];
  __shared__ double Bs[kGK * kLD];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  const int gq = lane >> 2, t4 = lane & 3;
  const int64_t i0 = (int64_t)blockIdx.x * kBM, j0 = (int64_t)blockIdx.y * kBN;
  const int64_t kb = (int64_t)blockIdx.z * g.ksplit;
  int64_t ke = kb + g.ksplit;
  if (ke > g.k) ke = g.k;

  double acc[4][2][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

  // Each thread stages 4 A and 4 B elements per k-tile (64x16 each).
  double ra[4], rb[4];
  auto fetch = [&](int64_t k0) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = threadIdx.x + u * kRT;
      int i, kk;
      if (g.ta) { kk = e % kGK; i = e / kGK; } else { i = e % kBM; kk = e / kBM; }
      ra[u] = (k0 + kk < ke) ? ldA(g, i0 + i, k0 + kk) : 0.0;
      int j, kb2;
      if (g.tb) { j = e % kBN; kb2 = e / kBN; } else { kb2 = e % kGK; j = e / kGK; }
      rb[u] = (k0 + kb2 < ke) ? ldB(g, k0 + kb2, j0 + j) : 0.0;
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = threadIdx.x + u * kRT;
      int i, kk;
      if (g.ta) { kk = e % kGK; i = e / kGK; } else { i = e % kBM; kk = e / kBM; }
      As[kk * kLD + i] = ra[u];
      int j, kb2;
      if (g.tb) { j = e % kBN; kb2 = e / kBN; } else { kb2 = e % kGK; j = e / kGK; }
      Bs[kb2 * kLD + j] = rb[u];
    }
  };
  if (kb < ke) fetch(kb);
  for (int64_t k0 = kb; k0 < ke; k0 += kGK) {
    __syncthreads();
    store();
    __syncthreads();
    if (k0 + kGK < ke) fetch(k0 + kGK);
#pragma unroll
    for (int kk = 0; kk < kGK; kk += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) af[mi] = As[(kk + t4) * kLD + wm * 32 + mi * 8 + gq];
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) bf[ni] = Bs[(kk + t4) * kLD + wn * 16 + ni * 8 + gq];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
  }
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t r = i0 + wm * 32 + mi * 8 + gq;
        const int64_t cc = j0 + wn * 16 + ni * 8 + 2 * t4 + e;
        if (r < g.m && cc < g.n) {
          if (g.partial) {
            g.partial[(int64_t)blockIdx.z * g.m * g.n + r + cc * g.m] = acc[mi][ni][e];
          } else {
            double v = g.alpha * acc[mi][ni][e];
            if (g.beta != 0.0) v += g.beta * g.Cm[r + cc * g.ldc];
            g.Cm[r + cc * g.ldc] = v;
          }
        }
      }
}

// Deterministic split-K combine: slices summed in order.
__global__ void splitk_reduce_kernel(const double* __restrict__ part, int64_t m, int64_t n, int nz, double alpha,
                                     double beta, double* __restrict__ Cm, int64_t ldc) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < nz; ++z) s += part[z * total + e];
    const int64_t r = e % m, cc = e / m;
    double v = alpha * s;
    if (beta != 0.0) v += beta * Cm[r + cc * ldc];
    Cm[r + cc * ldc] = v;
  }
}

int launch_gemm_fam(Context* c, const char* fam, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
                int64_t lda, const double* B, int64_t ldb, double beta, double* Cm, int64_t ldc) {
  if (m == 0 || n == 0) return SLRA_OK;
  if (ta == 1 && tb == 0 && beta == 0.0 && m <= 64 && k >= 256) {
    // skinny W^T B over a tall K (range finder V = U^+ M): streaming kernel
    const int st = launch_tn_skinny(c, fam, m, n, k, alpha, A, lda, B, ldb, Cm, ldc);
    if (st != SLRA_ERR_UNSUPPORTED) return st;
  }
  GemmArgs g{ta, tb, m, n, k, alpha, beta, A, lda, B, ldb, Cm, ldc, k, nullptr};
  const int gx = ceil_div(m, kBM), gy = ceil_div(n, kBN);
  int nz = 1;
  const int64_t tiles = (int64_t)gx * gy;
  if (tiles < c->num_sms && k >= 512) {
    nz = (int)((2 * c->num_sms + tiles - 1) / tiles);
    const int64_t maxz = k / 256;
    if (nz > maxz) nz = (int)maxz;
    if (nz < 1) nz = 1;
  }
  if (nz > 1) {
    int64_t ks = (k + nz - 1) / nz;
    ks = (ks + kGK - 1) / kGK * kGK;
    nz = (int)((k + ks - 1) / ks);
    g.ksplit = ks;
    double* part = static_cast<double*>(workspace(c, sizeof(double) * m * n * nz));
    if (!part) return SLRA_ERR_CUDA;
    g.partial = part;
    SLRA_TIMED(c, fam, gemm_kernel<<<dim3(gx, gy, nz), kRT, 0, c->stream>>>(g);)
    SLRA_CHECK_LAUNCH(c);
    int rg = ceil_div(m * n, 256);
    if (rg > c->num_sms * 8) rg = c->num_sms * 8;
    SLRA_TIMED(c, "gemm_reduce", splitk_reduce_kernel<<<rg, 256, 0, c->stream>>>(part, m, n, nz, alpha, beta, Cm, ldc);)
    SLRA_CHECK_LAUNCH(c);
    return SLRA_OK;
  }
  SLRA_TIMED(c, fam, gemm_kernel<<<dim3(gx, gy, 1), kRT, 0, c->stream>>>(g);)
  SLRA_CHECK_LAUNCH(c);
  return SLRA_OK;
}

int launch_gemm(Context* c, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
                int64_t lda, const double* B, int64_t ldb, double beta, double* Cm, int64_t ldc) {
  return launch_gemm_fam(c, "gemm", ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, Cm, ldc);
}

}  // namespace slra_dev

using namespace slra_dev;

extern "C" {

int slra_lowrank_residual(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t n, const double* P,
                          int64_t ldp, const double* Q, int64_t ldq, int64_t inner, double* d_out) {
  if (!ctx || lda < m || m < 0 || n < 0 || inner < 0 || (inner > 0 && (ldp < m || ldq < inner)))
    return SLRA_ERR_INVALID_ARGUMENT;
  return launch_lowrank_residual(C(ctx), A, lda, m, n, P, ldp, Q, ldq, inner, d_out);
}

int slra_gemm(slra_ctx ctx, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
              int64_t lda, const double* B, int64_t ldb, double beta, double* Cm, int64_t ldc) {
  if (!ctx || m < 0 || n < 0 || k < 0 || ldc < m) return SLRA_ERR_INVALID_ARGUMENT;
  if ((!ta && lda < m) || (ta && lda < k) || (!tb && ldb < k) || (tb && ldb < n)) return SLRA_ERR_INVALID_ARGUMENT;
  return launch_gemm(C(ctx), ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, Cm, ldc);
}

}  // extern "C"
