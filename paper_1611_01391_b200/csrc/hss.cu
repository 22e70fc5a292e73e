// HSS construction (Svd strategy) and the HSS matrix-vector product on the
// device — /root/reference/proj/src/hss.cpp:58-96 (approx_block, Svd
// branch), :143-185 (build_node / build_hss), :193-212 (hss_matvec).
//
// Packed level-major layout (slra_cuda.h): at level l the 2^(l+1)
// off-diagonal blocks have pairwise-disjoint row ranges that tile [0, n), and
// likewise their column ranges, so every level's generators pack into two
// n x r matrices with no offsets table:
//   F_l (n x r, ld n):  F_l(row0_b + i, a) = F_b(i, a)
//   HT_l (n x r, ld n): HT_l(col0_b + j, a) = H_b(a, j)      (H_b^T)
// and the leaves into D (n x leaf, ld n): D(i, j) = M(i, leaf0(i) + j).
// Block b = 2 t + {0: upper, 1: lower} of node t at level l; rank[l][b].
//
// The Svd strategy draws nothing from the Rng, so every block of every level
// is independent: all SVDs are launched back to back (batched per level and
// side), one host sync reads the singular values, the reference's rank rule
// runs on the host, and one kernel per level writes the factors.
#include <cmath>
#include <vector>

#include "common.cuh"

namespace slra_dev {

int launch_svd_small_batched(Context* cx, const double* A, int64_t lda, int64_t sA, int m, int n, double* S,
                             int64_t lds, int64_t sS, double* sigma, int64_t sSig, double* T, int64_t ldt, int64_t sT,
                             int nb, double deflate);
size_t svd_large_workspace_doubles(int64_t m, int64_t n, int nb);
int launch_svd_large_batched(Context* cx, const double* A, int64_t lda, int64_t sA, int m, int n, int nb,
                             double* S, int64_t lds, int64_t sS, double* sigma, int64_t sSig, double* T, int64_t ldt,
                             int64_t sT, double* ws);

namespace {

constexpr int kHT = 256;

// D(i, j) = M(i, (i / leaf) * leaf + j)
__global__ void hss_leaves_kernel(const double* __restrict__ M, int64_t ldm, int64_t n, int64_t leaf,
                                  double* __restrict__ D) {
  const int64_t total = n * leaf;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % n, j = e / n;
    D[e] = M[i + ((i / leaf) * leaf + j) * ldm];
  }
}

// Level l factors from the per-block SVDs (S_b half x half, sigma_b, T_b):
// F_l(row0 + i, a) = S_b(i, a) sigma_b[a], HT_l(col0 + j, a) = T_b(j, a) for
// a < rank_b (hss.cpp:93-94), zero for rank_b <= a < r.
__global__ void hss_emit_svd_kernel(const double* __restrict__ Sb, const double* __restrict__ sig,
                                    const double* __restrict__ Tb, int64_t half, int nblk, int64_t r,
                                    const int64_t* __restrict__ rank, double* __restrict__ F,
                                    double* __restrict__ HT, int64_t n) {
  const int64_t total = n * r;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % n, a = e / n;
    // row i of F_l belongs to block b_row; column i of H_l to block b_col
    const int64_t t = i / (2 * half), w = i % (2 * half);
    const int64_t b_row = 2 * t + (w < half ? 0 : 1);  // upper block holds the node's first half rows
    const int64_t b_col = 2 * t + (w < half ? 1 : 0);  // lower block holds the node's first half columns
    const int64_t ii = w % half;
    const int64_t hh = half * half;
    F[e] = a < rank[b_row] ? Sb[b_row * hh + ii + a * half] * sig[b_row * half + a] : 0.0;
    HT[e] = a < rank[b_col] ? Tb[b_col * hh + ii + a * half] : 0.0;
  }
}

// t[l][b][a] = sum_j H_b(a, j) x(col0_b + j) = sum_j HT_l(col0_b + j, a) x(col0_b + j)
// one warp per (l, b, a)
__global__ void hss_project_kernel(const double* __restrict__ HT, const int64_t* __restrict__ rank,
                                   const double* __restrict__ x, int64_t n, int L, int64_t r,
                                   double* __restrict__ tv) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nblk_all = ((int64_t)2 << L) - 2;
  if (wid >= nblk_all * r) return;
  const int64_t g = wid / r, a = wid % r;  // g: level-major block id
  int l = 0;
  int64_t base = 0;
  while (base + ((int64_t)2 << l) <= g) {
    base += (int64_t)2 << l;
    ++l;
  }
  const int64_t b = g - base, t = b >> 1;
  const int64_t size = n >> l, half = size >> 1;  // n divisible by 2^L
  const int64_t col0 = t * size + ((b & 1) ? 0 : half);
  double s = 0.0;
  if (a < rank[g]) {
    const double* h = HT + (int64_t)l * n * r + a * n + col0;
    for (int64_t j = lane; j < half; j += 32) s = fma(h[j], x[col0 + j], s);
    s = warp_sum(s);
  }
  if (lane == 0) tv[g * r + a] = s;
}

// y_i = D(i, :) x(leaf block) + sum_l F_l(i, :) t[l][b(i, l)] in the
// reference's order (leaves first, then the blocks by level: hss.cpp:196-209).
__global__ void hss_apply_kernel(const double* __restrict__ D, const double* __restrict__ F,
                                 const int64_t* __restrict__ rank, const double* __restrict__ tv,
                                 const double* __restrict__ x, int64_t n, int L, int64_t leaf, int64_t r,
                                 double* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l0 = (i / leaf) * leaf;
    double acc = 0.0;
    for (int64_t j = 0; j < leaf; ++j) acc = fma(D[i + j * n], x[l0 + j], acc);
    int64_t base = 0;
    for (int l = 0; l < L; ++l) {
      const int64_t size = n >> l, half = size >> 1;
      const int64_t t = i / size, w = i % size;
      const int64_t g = base + 2 * t + (w < half ? 0 : 1);
      const int64_t rk = rank[g];
      if (rk > 0) {
        const double* f = F + (int64_t)l * n * r + i;
        const double* tt = tv + g * r;
        double s = 0.0;
        for (int64_t a = 0; a < rk; ++a) s = fma(f[a * n], tt[a], s);
        acc += s;
      }
      base += (int64_t)2 << l;
    }
    y[i] = acc;
  }
}

bool hss_shape_ok(int64_t n, int L, int64_t r) {
  if (n < 2 || L < 1 || L > 30 || r < 0) return false;
  const int64_t blocks = (int64_t)1 << L;
  return n % blocks == 0 && n / blocks >= r;
}

}  // namespace

int launch_hss_matvec(Context* cx, int64_t n, int L, int64_t r, const double* D, const double* F, const double* HT,
                      const int64_t* rank, const double* x, double* y, double* tv) {
  const int64_t leaf = n >> L;
  const int64_t nblk = ((int64_t)2 << L) - 2;
  if (r > 0) {
    const int64_t warps = nblk * r;
    SLRA_TIMED(cx, "hss_matvec", hss_project_kernel<<<(unsigned)ceil_div(warps * 32, kHT), kHT, 0, cx->stream>>>(
                                     HT, rank, x, n, L, r, tv);)
    SLRA_CHECK_LAUNCH(cx);
  }
  int64_t g = ceil_div(n, kHT);
  if (g > cx->num_sms * 8) g = cx->num_sms * 8;
  SLRA_TIMED(cx, "hss_matvec", hss_apply_kernel<<<(unsigned)g, kHT, 0, cx->stream>>>(D, F, rank, tv, x, n, L, leaf,
                                                                                      r > 0 ? r : 1, y);)
  SLRA_CHECK_LAUNCH(cx);
  return SLRA_OK;
}

}  // namespace slra_dev

using namespace slra_dev;

extern "C" {

int slra_hss_leaves(slra_ctx ctx, const double* M, int64_t ldm, int64_t n, int L, double* D) {
  if (!ctx || ldm < n || !hss_shape_ok(n, L, 0)) return SLRA_ERR_INVALID_ARGUMENT;
  Context* cx = C(ctx);
  const int64_t leaf = n >> L;
  int64_t g = ceil_div(n * leaf, 256);
  if (g > cx->num_sms * 8) g = cx->num_sms * 8;
  SLRA_TIMED(cx, "hss_build", hss_leaves_kernel<<<(unsigned)g, 256, 0, cx->stream>>>(M, ldm, n, leaf, D);)
  SLRA_CHECK_LAUNCH(cx);
  return SLRA_OK;
}

int slra_hss_build_svd(slra_ctx ctx, const double* M, int64_t ldm, int64_t n, int L, int64_t r, double tol,
                       double* D, double* F, double* HT, int64_t* h_rank, int32_t* h_overflow) {
  if (!ctx || ldm < n || !hss_shape_ok(n, L, r) || !(tol >= 0.0)) return SLRA_ERR_INVALID_ARGUMENT;
  Context* cx = C(ctx);
  SLRA_TRY(slra_hss_leaves(ctx, M, ldm, n, L, D));
  // per level: 2^(l+1) blocks of half x half -> S, sigma, T (level-major)
  std::vector<size_t> off_s(L), off_sig(L);
  size_t tot = 0, big_ws = 0;
  for (int l = 0; l < L; ++l) {
    const int64_t half = (n >> l) >> 1, nb = (int64_t)2 << l;
    off_s[l] = tot;
    tot += 2 * (size_t)nb * half * half;  // S and T
    off_sig[l] = tot;
    tot += (size_t)nb * half;
    if (half > 64) {
      const size_t w = svd_large_workspace_doubles(half, half, (int)(nb / 2));
      if (w > big_ws) big_ws = w;
    }
  }
  const size_t nblk_all = ((size_t)2 << L) - 2;
  double* buf = static_cast<double*>(arena(cx, 11, sizeof(double) * (tot + big_ws + nblk_all + 64)));
  if (!buf) return SLRA_ERR_CUDA;
  double* bigw = buf + tot;
  int64_t* drank = reinterpret_cast<int64_t*>(bigw + big_ws);
  for (int l = 0; l < L; ++l) {
    const int64_t size = n >> l, half = size >> 1, nodes = (int64_t)1 << l, nb = 2 * nodes;
    const int64_t hh = half * half;
    double* S = buf + off_s[l];
    double* T = S + (size_t)nb * hh;
    double* sig = buf + off_sig[l];
    const int64_t stride = size * (ldm + 1);  // node t -> node t + 1 along the diagonal
    for (int side = 0; side < 2; ++side) {     // 0: upper (rows first half, cols second half)
      const double* A0 = M + (side == 0 ? half * ldm : half);
      // blocks of one side are b = 2 t + side: output stride 2 hh, sigma stride 2 half
      double* Sb = S + side * hh;
      double* Tb = T + side * hh;
      double* sb = sig + side * half;
      if (half <= 64) {
        SLRA_TRY(launch_svd_small_batched(cx, A0, ldm, stride, (int)half, (int)half, Sb, half, 2 * hh, sb, 2 * half,
                                          Tb, half, 2 * hh, (int)nodes, 0.0));
      } else {
        SLRA_TRY(launch_svd_large_batched(cx, A0, ldm, stride, (int)half, (int)half, (int)nodes, Sb, half, 2 * hh, sb,
                                          2 * half, Tb, half, 2 * hh, bigw));
      }
    }
  }
  // rank rule (hss.cpp:71-92) on the singular values: smallest rho <= min(r, half)
  // whose discarded tail meets tol * ||sigma||, else r with the overflow flag
  std::vector<double> hs(tot);
  SLRA_CUDA(cudaMemcpyAsync(hs.data(), buf, sizeof(double) * tot, cudaMemcpyDeviceToHost, cx->stream));
  SLRA_CUDA(cudaStreamSynchronize(cx->stream));
  std::vector<int64_t> ranks(nblk_all);
  size_t g = 0;
  for (int l = 0; l < L; ++l) {
    const int64_t half = (n >> l) >> 1, nb = (int64_t)2 << l;
    for (int64_t b = 0; b < nb; ++b, ++g) {
      const double* s = hs.data() + off_sig[l] + b * half;
      auto tail = [&](int64_t rho) {
        if (rho >= half) return 0.0;
        double q = 0.0;
        for (int64_t j = rho; j < half; ++j) q += s[j] * s[j];
        return std::sqrt(q);
      };
      const double total = tail(0);
      int64_t rho = 0;
      bool over = false;
      if (total > 0) {
        const int64_t cap = r < half ? r : half;
        rho = cap;
        for (int64_t cand = 0; cand <= cap; ++cand)
          if (tail(cand) <= tol * total) {
            rho = cand;
            break;
          }
        over = tail(rho) > tol * total;
      }
      ranks[g] = rho;
      if (h_rank) h_rank[g] = rho;
      if (h_overflow) h_overflow[g] = over ? 1 : 0;
    }
  }
  SLRA_CUDA(cudaMemcpyAsync(drank, ranks.data(), sizeof(int64_t) * nblk_all, cudaMemcpyHostToDevice, cx->stream));
  size_t base = 0;
  for (int l = 0; l < L; ++l) {
    const int64_t half = (n >> l) >> 1, nb = (int64_t)2 << l;
    const int64_t hh = half * half;
    double* S = buf + off_s[l];
    int64_t gr = ceil_div(n * r, 256);
    if (gr > cx->num_sms * 8) gr = cx->num_sms * 8;
    // S_b at S + b hh? blocks were written at side offsets: b = 2 t + side -> S + (2 t + side) hh
    SLRA_TIMED(cx, "hss_build", hss_emit_svd_kernel<<<(unsigned)gr, 256, 0, cx->stream>>>(
                                    S, buf + off_sig[l], S + (size_t)nb * hh, half, (int)nb, r, drank + base,
                                    F + (size_t)l * n * r, HT + (size_t)l * n * r, n);)
    SLRA_CHECK_LAUNCH(cx);
    base += nb;
  }
  // the host vector above must outlive the async copy
  SLRA_CUDA(cudaStreamSynchronize(cx->stream));
  return SLRA_OK;
}

int slra_hss_matvec(slra_ctx ctx, int64_t n, int L, int64_t r, const double* D, const double* F, const double* HT,
                    const int64_t* rank, const double* x, double* y) {
  if (!ctx || !hss_shape_ok(n, L, r)) return SLRA_ERR_INVALID_ARGUMENT;
  Context* cx = C(ctx);
  const size_t nblk_all = ((size_t)2 << L) - 2;
  double* tv = static_cast<double*>(workspace(cx, sizeof(double) * (nblk_all * (size_t)(r > 0 ? r : 1) + 8)));
  if (!tv) return SLRA_ERR_CUDA;
  return launch_hss_matvec(cx, n, L, r, D, F, HT, rank, x, y, tv);
}

}  // extern "C"

namespace slra_dev {
namespace {

// out(i, j) = [M(i, j) -] HSS(i, j): the leaf entry, or row i of the level-l
// generator F_l times row j of HT_l, where l is the level whose node holds
// i and j in opposite halves (hss.cpp:214-221).
__global__ void hss_reconstruct_kernel(const double* __restrict__ D, const double* __restrict__ F,
                                       const double* __restrict__ HT, const int64_t* __restrict__ rank, int64_t n,
                                       int L, int64_t r, const double* __restrict__ M, int64_t ldm,
                                       double* __restrict__ out, int64_t ldo) {
  const int64_t leaf = n >> L;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % n, j = e / n;
    double v = 0.0;
    if (i / leaf == j / leaf) {
      v = D[i + (j - (i / leaf) * leaf) * n];
    } else {
      int64_t base = 0;
      for (int l = 0; l < L; ++l) {
        const int64_t size = n >> l, half = size >> 1;
        if (i / size == j / size) {
          const bool iu = (i % size) < half, ju = (j % size) < half;
          if (iu != ju) {
            const int64_t g = base + 2 * (i / size) + (iu ? 0 : 1);
            const double* f = F + (int64_t)l * n * r;
            const double* h = HT + (int64_t)l * n * r;
            for (int64_t a = 0; a < rank[g]; ++a) v = fma(f[i + a * n], h[j + a * n], v);
            break;
          }
        }
        base += (int64_t)2 << l;
      }
    }
    out[i + j * ldo] = M ? M[i + j * ldm] - v : v;
  }
}

}  // namespace
}  // namespace slra_dev

extern "C" {

int slra_hss_reconstruct(slra_ctx ctx, int64_t n, int L, int64_t r, const double* D, const double* F,
                         const double* HT, const int64_t* rank, const double* M, int64_t ldm, double* out,
                         int64_t ldo) {
  if (!ctx || !hss_shape_ok(n, L, r) || ldo < n || (M && ldm < n)) return SLRA_ERR_INVALID_ARGUMENT;
  Context* cx = C(ctx);
  int64_t g = ceil_div(n * n, 256);
  if (g > cx->num_sms * 8) g = cx->num_sms * 8;
  SLRA_TIMED(cx, "hss_reconstruct", hss_reconstruct_kernel<<<(unsigned)g, 256, 0, cx->stream>>>(
                                        D, F, HT, rank, n, L, r > 0 ? r : 1, M, ldm, out, ldo);)
  SLRA_CHECK_LAUNCH(cx);
  return SLRA_OK;
}

}  // extern "C"
