// K-a: gathers (EntryOracle::rows_of/cols_of/block, testgen.cpp:11-30;
// select_rows/cols/block, linalg.cpp:35-52) and compiled sketch plans
// (SparseCirculantOp sketch.cpp:215-282, ah_recurse sketch.cpp:98-107,
// Permutation/SignDiagonal/SubIdentity/Product/ColumnSlice composites).
// Pure data movement plus exact +-1 arithmetic: every result is bit-exact
// against the reference's full-operator application.
#include "common.cuh"

namespace slra_dev {

constexpr int kNT = 256;

// ---------------------------------------------------------------- gathers
// Columns are contiguous in column-major storage: 16-byte vector loads when
// both sides are 16-byte aligned (lda, ldc even and base pointers aligned).
__global__ void __launch_bounds__(kNT) gather_cols_vec_kernel(const double* __restrict__ A, int64_t lda,
                                                              int64_t m, const int64_t* __restrict__ J,
                                                              double* __restrict__ Cm, int64_t ldc) {
  const int64_t t = blockIdx.y;
  const double2* src = reinterpret_cast<const double2*>(A + J[t] * lda);
  double2* dst = reinterpret_cast<double2*>(Cm + t * ldc);
  const int64_t m2 = m >> 1;
  for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < m2; i += (int64_t)gridDim.x * kNT)
    dst[i] = __ldg(src + i);
  if ((m & 1) && blockIdx.x == 0 && threadIdx.x == 0) Cm[t * ldc + m - 1] = A[J[t] * lda + m - 1];
}

__global__ void __launch_bounds__(kNT) gather_cols_kernel(const double* __restrict__ A, int64_t lda, int64_t m,
                                                          const int64_t* __restrict__ J,
                                                          double* __restrict__ Cm, int64_t ldc) {
  const int64_t t = blockIdx.y;
  const double* src = A + J[t] * lda;
  for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < m; i += (int64_t)gridDim.x * kNT)
    Cm[t * ldc + i] = __ldg(src + i);
}

// R(t, j) = A(I[t], j): consecutive threads walk t so the stores coalesce;
// each load is a separate 32-byte sector of the column-major input.
__global__ void __launch_bounds__(kNT) gather_rows_kernel(const double* __restrict__ A, int64_t lda, int64_t n,
                                                          const int64_t* __restrict__ I, int64_t k,
                                                          double* __restrict__ R, int64_t ldr) {
  const int64_t total = k * n;
  for (int64_t e = blockIdx.x * (int64_t)kNT + threadIdx.x; e < total; e += (int64_t)gridDim.x * kNT) {
    const int64_t t = e % k, j = e / k;
    R[t + j * ldr] = __ldg(A + I[t] + j * lda);
  }
}

// RT(j, t) = A(I[t], j): the row strip of the C-A sweep (cur.cpp:215-217)
// written straight as the n x k tall matrix R^T that select_rows_spanning
// factorises; consecutive threads walk j so the stores coalesce.
__global__ void __launch_bounds__(kNT) gather_rows_t_kernel(const double* __restrict__ A, int64_t lda, int64_t n,
                                                            const int64_t* __restrict__ I, int64_t k,
                                                            double* __restrict__ RT, int64_t ldrt) {
  const int64_t total = k * n;
  for (int64_t e = blockIdx.x * (int64_t)kNT + threadIdx.x; e < total; e += (int64_t)gridDim.x * kNT) {
    const int64_t j = e % n, t = e / n;
    RT[j + t * ldrt] = __ldg(A + I[t] + j * lda);
  }
}

__global__ void __launch_bounds__(kNT) gather_block_kernel(const double* __restrict__ A, int64_t lda,
                                                           const int64_t* __restrict__ I, int64_t k,
                                                           const int64_t* __restrict__ J, int64_t l,
                                                           double* __restrict__ G, int64_t ldg) {
  const int64_t total = k * l;
  for (int64_t e = blockIdx.x * (int64_t)kNT + threadIdx.x; e < total; e += (int64_t)gridDim.x * kNT) {
    const int64_t s = e % k, t = e / k;
    G[s + t * ldg] = __ldg(A + I[s] + J[t] * lda);
  }
}

// ---------------------------------------------------------------- sketch plans
// Combine `W` signed leaves in the reference's evaluation order.
template <int W, int TREE>
__device__ __forceinline__ double combine(const double (&z)[W], int q) {
  if (TREE == SLRA_TREE_LIST) {
    double acc = z[0];
#pragma unroll
    for (int s = 1; s < W; ++s) acc = acc + z[s];
    return acc;
  } else {
    // ah_recurse: level with half-size h pairs (i, i+h) inside blocks of 2h,
    // top = a + b, bottom = a - b; outermost level first.
    double y[W];
#pragma unroll
    for (int s = 0; s < W; ++s) y[s] = z[s];
#pragma unroll
    for (int len = W; len > 1; len >>= 1) {
      const int h = len >> 1;
#pragma unroll
      for (int base = 0; base < W; base += len)
#pragma unroll
        for (int i = 0; i < h; ++i) {
          const double a = y[base + i], b = y[base + i + h];
          y[base + i] = a + b;
          y[base + i + h] = a - b;
        }
    }
    double out = 0;
#pragma unroll
    for (int s = 0; s < W; ++s)
      if (s == q) out = y[s];
    return out;
  }
}

// out(:, t) = combine_s coef[t,s] * A(:, src[t,s]); one block column per t.
template <int W, int TREE>
__global__ void __launch_bounds__(kNT) sketch_cols_kernel(const double* __restrict__ A, int64_t lda, int64_t m,
                                                          const int64_t* __restrict__ src,
                                                          const double* __restrict__ coef,
                                                          const int32_t* __restrict__ qv,
                                                          double* __restrict__ out, int64_t ldo) {
  const int64_t t = blockIdx.y;
  __shared__ const double* cols[W];
  __shared__ double cf[W];
  if (threadIdx.x < W) {
    cols[threadIdx.x] = A + src[t * W + threadIdx.x] * lda;
    cf[threadIdx.x] = coef[t * W + threadIdx.x];
  }
  __syncthreads();
  const int q = TREE == SLRA_TREE_FWHT ? qv[t] : 0;
  for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < m; i += (int64_t)gridDim.x * kNT) {
    double z[W];
#pragma unroll
    for (int s = 0; s < W; ++s) z[s] = cf[s] * __ldg(cols[s] + i);
    out[t * ldo + i] = combine<W, TREE>(z, q);
  }
}

// Generic width (list order only), for plans wider than the templated set.
__global__ void __launch_bounds__(kNT) sketch_cols_list_kernel(const double* __restrict__ A, int64_t lda,
                                                               int64_t m, const int64_t* __restrict__ src,
                                                               const double* __restrict__ coef, int64_t w,
                                                               double* __restrict__ out, int64_t ldo) {
  const int64_t t = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < m; i += (int64_t)gridDim.x * kNT) {
    double acc = coef[t * w] * A[src[t * w] * lda + i];
    for (int64_t s = 1; s < w; ++s) acc = acc + coef[t * w + s] * A[src[t * w + s] * lda + i];
    out[t * ldo + i] = acc;
  }
}

// out(t, :) = combine_s coef[t,s] * W(src[t,s], :); thread per (t, j),
// t fastest so stores coalesce.
// columns per thread of sketch_rows_kernel (kJB * Wd gathers in flight)
__host__ __device__ constexpr int sr_jb(int wd) { return wd <= 2 ? 8 : (wd <= 4 ? 4 : (wd <= 8 ? 2 : 1)); }

template <int Wd, int TREE>
__global__ void __launch_bounds__(kNT) sketch_rows_kernel(const double* __restrict__ Wm, int64_t ldw,
                                                          int64_t ncols, const int64_t* __restrict__ src,
                                                          const double* __restrict__ coef,
                                                          const int32_t* __restrict__ qv, int64_t k,
                                                          double* __restrict__ out, int64_t ldo) {
  // a thread per output row t and kJB consecutive columns: the plan entries
  // of the row are read once and all kJB * Wd gathers are in flight together
  // (the rows are scattered sectors; one load per thread per iteration left
  // the kernel latency-bound); no 64-bit index division
  constexpr int kJB = sr_jb(Wd);
  const int64_t t = blockIdx.x * (int64_t)kNT + threadIdx.x;
  if (t >= k) return;
  const int64_t j0 = (int64_t)blockIdx.y * kJB;
  int64_t sr[Wd];
  double cf[Wd];
#pragma unroll
  for (int s = 0; s < Wd; ++s) {
    sr[s] = src[t * Wd + s];
    cf[s] = coef[t * Wd + s];
  }
  const int qt = TREE == SLRA_TREE_FWHT ? qv[t] : 0;
  double z[kJB][Wd];
#pragma unroll
  for (int u = 0; u < kJB; ++u) {
    const int64_t j = j0 + u < ncols ? j0 + u : j0;
#pragma unroll
    for (int s = 0; s < Wd; ++s) z[u][s] = __ldg(Wm + sr[s] + j * ldw);
  }
#pragma unroll
  for (int u = 0; u < kJB; ++u) {
    if (j0 + u < ncols) {
      double zz[Wd];
#pragma unroll
      for (int s = 0; s < Wd; ++s) zz[s] = cf[s] * z[u][s];
      out[t + (j0 + u) * ldo] = combine<Wd, TREE>(zz, qt);
    }
  }
}

__global__ void __launch_bounds__(kNT) sketch_rows_list_kernel(const double* __restrict__ Wm, int64_t ldw,
                                                               int64_t ncols, const int64_t* __restrict__ src,
                                                               const double* __restrict__ coef, int64_t w,
                                                               int64_t k, double* __restrict__ out, int64_t ldo) {
  const int64_t total = k * ncols;
  for (int64_t e = blockIdx.x * (int64_t)kNT + threadIdx.x; e < total; e += (int64_t)gridDim.x * kNT) {
    const int64_t t = e % k, j = e / k;
    double acc = coef[t * w] * Wm[src[t * w] + j * ldw];
    for (int64_t s = 1; s < w; ++s) acc = acc + coef[t * w + s] * Wm[src[t * w + s] + j * ldw];
    out[t + j * ldo] = acc;
  }
}

// Row-sharded form of the LIST-order sketch (width 1 = gather): this rank
// holds rows [row0, row0 + mloc) of W; terms whose source row lives on
// another rank are skipped, so summing the per-rank outputs (NCCL
// allreduce) reproduces the full combination — bit-exactly for width <= 2,
// where every output is one or two terms plus exact zeros. transpose = 1
// writes out(j, t) (ncols x k) instead of out(t, j).
__global__ void __launch_bounds__(kNT) sketch_rows_shard_kernel(const double* __restrict__ Wm, int64_t ldw,
                                                                int64_t row0, int64_t mloc, int64_t ncols,
                                                                const int64_t* __restrict__ src,
                                                                const double* __restrict__ coef, int64_t w,
                                                                int64_t k, double* __restrict__ out, int64_t ldo,
                                                                int transpose) {
  const int64_t total = k * ncols;
  for (int64_t e = blockIdx.x * (int64_t)kNT + threadIdx.x; e < total; e += (int64_t)gridDim.x * kNT) {
    const int64_t t = transpose ? e / ncols : e % k, j = transpose ? e % ncols : e / k;
    double acc = 0.0;
    bool first = true;
    for (int64_t s = 0; s < w; ++s) {
      const int64_t r = src[t * w + s] - row0;
      if (r < 0 || r >= mloc) continue;
      const double term = coef[t * w + s] * __ldg(Wm + r + j * ldw);
      acc = first ? term : acc + term;
      first = false;
    }
    out[transpose ? j + t * ldo : t + j * ldo] = acc;
  }
}

static int grid_1d(const Context* c, int64_t work) {
  const int64_t per = kNT * 4;
  int64_t g = (work + per - 1) / per;
  const int64_t cap = (int64_t)c->num_sms * 16;
  if (g > cap) g = cap;
  return static_cast<int>(g < 1 ? 1 : g);
}

int launch_sketch_cols(Context* c, const double* A, int64_t lda, int64_t m, const int64_t* src,
                       const double* coef, const int32_t* q, int64_t width, int tree, int64_t l, double* out,
                       int64_t ldo) {
  int gx = ceil_div(m, kNT);
  const int cap = (int)((int64_t)c->num_sms * 8 / (l > 0 ? l : 1)) + 1;
  if (gx > cap) gx = cap;
  dim3 grid(gx < 1 ? 1 : gx, static_cast<unsigned>(l));
  cudaStream_t s = c->stream;
  if (tree == SLRA_TREE_FWHT) {
    switch (width) {
      case 1: sketch_cols_kernel<1, SLRA_TREE_FWHT><<<grid, kNT, 0, s>>>(A, lda, m, src, coef, q, out, ldo); break;
      case 2: sketch_cols_kernel<2, SLRA_TREE_FWHT><<<grid, kNT, 0, s>>>(A, lda, m, src, coef, q, out, ldo); break;
      case 4: sketch_cols_kernel<4, SLRA_TREE_FWHT><<<grid, kNT, 0, s>>>(A, lda, m, src, coef, q, out, ldo); break;
      case 8: sketch_cols_kernel<8, SLRA_TREE_FWHT><<<grid, kNT, 0, s>>>(A, lda, m, src, coef, q, out, ldo); break;
      case 16: sketch_cols_kernel<16, SLRA_TREE_FWHT><<<grid, kNT, 0, s>>>(A, lda, m, src, coef, q, out, ldo); break;
      default: return SLRA_ERR_UNSUPPORTED;
    }
  } else {
    switch (width) {
      case 1: sketch_cols_kernel<1, SLRA_TREE_LIST><<<grid, kNT, 0, s>>>(A, lda, m, src, coef, q, out, ldo); break;
      case 2: sketch_cols_kernel<2, SLRA_TREE_LIST><<<grid, kNT, 0, s>>>(A, lda, m, src, coef, q, out, ldo); break;
      case 3: sketch_cols_kernel<3, SLRA_TREE_LIST><<<grid, kNT, 0, s>>>(A, lda, m, src, coef, q, out, ldo); break;
      case 4: sketch_cols_kernel<4, SLRA_TREE_LIST><<<grid, kNT, 0, s>>>(A, lda, m, src, coef, q, out, ldo); break;
      case 8: sketch_cols_kernel<8, SLRA_TREE_LIST><<<grid, kNT, 0, s>>>(A, lda, m, src, coef, q, out, ldo); break;
      default: sketch_cols_list_kernel<<<grid, kNT, 0, s>>>(A, lda, m, src, coef, width, out, ldo); break;
    }
  }
  SLRA_CHECK_LAUNCH(c);
  return SLRA_OK;
}

int launch_gather_cols(Context* c, const double* A, int64_t lda, int64_t m, const int64_t* J, int64_t l,
                       double* Cm, int64_t ldc) {
  if (l == 0 || m == 0) return SLRA_OK;
  const bool vec = (lda % 2 == 0) && (ldc % 2 == 0) && ((uintptr_t)A % 16 == 0) && ((uintptr_t)Cm % 16 == 0);
  int gx = ceil_div(vec ? (m + 1) / 2 : m, kNT);
  const int cap = c->num_sms * 8 / (int)l + 1;
  if (gx > cap) gx = cap;
  dim3 grid(gx < 1 ? 1 : gx, static_cast<unsigned>(l));
  if (vec)
    SLRA_TIMED(c, "gather", gather_cols_vec_kernel<<<grid, kNT, 0, c->stream>>>(A, lda, m, J, Cm, ldc);)
  else
    SLRA_TIMED(c, "gather", gather_cols_kernel<<<grid, kNT, 0, c->stream>>>(A, lda, m, J, Cm, ldc);)
  SLRA_CHECK_LAUNCH(c);
  return SLRA_OK;
}

int launch_gather_rows(Context* c, const double* A, int64_t lda, int64_t n, const int64_t* I, int64_t k, double* R,
                       int64_t ldr) {
  if (k == 0 || n == 0) return SLRA_OK;
  SLRA_TIMED(c, "gather", gather_rows_kernel<<<grid_1d(c, k * n), kNT, 0, c->stream>>>(A, lda, n, I, k, R, ldr);)
  SLRA_CHECK_LAUNCH(c);
  return SLRA_OK;
}

int launch_gather_rows_t(Context* c, const double* A, int64_t lda, int64_t n, const int64_t* I, int64_t k,
                         double* RT, int64_t ldrt) {
  if (k == 0 || n == 0) return SLRA_OK;
  SLRA_TIMED(c, "gather", gather_rows_t_kernel<<<grid_1d(c, k * n), kNT, 0, c->stream>>>(A, lda, n, I, k, RT, ldrt);)
  SLRA_CHECK_LAUNCH(c);
  return SLRA_OK;
}

int launch_gather_block(Context* c, const double* A, int64_t lda, const int64_t* I, int64_t k, const int64_t* J,
                        int64_t l, double* G, int64_t ldg) {
  if (k == 0 || l == 0) return SLRA_OK;
  SLRA_TIMED(c, "gather", gather_block_kernel<<<grid_1d(c, k * l), kNT, 0, c->stream>>>(A, lda, I, k, J, l, G, ldg);)
  SLRA_CHECK_LAUNCH(c);
  return SLRA_OK;
}

int launch_sketch_rows(Context* c, const double* Wm, int64_t ldw, int64_t ncols, const int64_t* src,
                       const double* coef, const int32_t* q, int64_t width, int tree, int64_t k, double* out,
                       int64_t ldo) {
  const int g = grid_1d(c, k * ncols);
  cudaStream_t s = c->stream;
  if (tree == SLRA_TREE_FWHT) {
    KernelTimer kt(c, "sketch");
    switch (width) {
      case 1: sketch_rows_kernel<1, SLRA_TREE_FWHT><<<dim3(ceil_div(k, kNT), ceil_div(ncols, sr_jb(1))), kNT, 0, s>>>(Wm, ldw, ncols, src, coef, q, k, out, ldo); break;
      case 2: sketch_rows_kernel<2, SLRA_TREE_FWHT><<<dim3(ceil_div(k, kNT), ceil_div(ncols, sr_jb(2))), kNT, 0, s>>>(Wm, ldw, ncols, src, coef, q, k, out, ldo); break;
      case 4: sketch_rows_kernel<4, SLRA_TREE_FWHT><<<dim3(ceil_div(k, kNT), ceil_div(ncols, sr_jb(4))), kNT, 0, s>>>(Wm, ldw, ncols, src, coef, q, k, out, ldo); break;
      case 8: sketch_rows_kernel<8, SLRA_TREE_FWHT><<<dim3(ceil_div(k, kNT), ceil_div(ncols, sr_jb(8))), kNT, 0, s>>>(Wm, ldw, ncols, src, coef, q, k, out, ldo); break;
      case 16: sketch_rows_kernel<16, SLRA_TREE_FWHT><<<dim3(ceil_div(k, kNT), ceil_div(ncols, sr_jb(16))), kNT, 0, s>>>(Wm, ldw, ncols, src, coef, q, k, out, ldo); break;
      default: return SLRA_ERR_UNSUPPORTED;
    }
  } else {
    KernelTimer kt(c, "sketch");
    switch (width) {
      case 1: sketch_rows_kernel<1, SLRA_TREE_LIST><<<dim3(ceil_div(k, kNT), ceil_div(ncols, sr_jb(1))), kNT, 0, s>>>(Wm, ldw, ncols, src, coef, q, k, out, ldo); break;
      case 2: sketch_rows_kernel<2, SLRA_TREE_LIST><<<dim3(ceil_div(k, kNT), ceil_div(ncols, sr_jb(2))), kNT, 0, s>>>(Wm, ldw, ncols, src, coef, q, k, out, ldo); break;
      case 3: sketch_rows_kernel<3, SLRA_TREE_LIST><<<dim3(ceil_div(k, kNT), ceil_div(ncols, sr_jb(3))), kNT, 0, s>>>(Wm, ldw, ncols, src, coef, q, k, out, ldo); break;
      case 4: sketch_rows_kernel<4, SLRA_TREE_LIST><<<dim3(ceil_div(k, kNT), ceil_div(ncols, sr_jb(4))), kNT, 0, s>>>(Wm, ldw, ncols, src, coef, q, k, out, ldo); break;
      default: sketch_rows_list_kernel<<<g, kNT, 0, s>>>(Wm, ldw, ncols, src, coef, width, k, out, ldo); break;
    }
  }
  SLRA_CHECK_LAUNCH(c);
  return SLRA_OK;
}

}  // namespace slra_dev

using namespace slra_dev;

extern "C" {

int slra_gather_rows(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t n, const int64_t* I, int64_t k,
                     double* R, int64_t ldr) {
  if (!ctx || lda < m || ldr < k || k < 0 || n < 0) return SLRA_ERR_INVALID_ARGUMENT;
  return launch_gather_rows(C(ctx), A, lda, n, I, k, R, ldr);
}

int slra_gather_cols(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t n, const int64_t* J, int64_t l,
                     double* Cm, int64_t ldc) {
  (void)n;
  if (!ctx || lda < m || ldc < m || l < 0) return SLRA_ERR_INVALID_ARGUMENT;
  return launch_gather_cols(C(ctx), A, lda, m, J, l, Cm, ldc);
}

int slra_gather_block(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t n, const int64_t* I, int64_t k,
                      const int64_t* J, int64_t l, double* G, int64_t ldg) {
  (void)n;
  if (!ctx || lda < m || ldg < k) return SLRA_ERR_INVALID_ARGUMENT;
  return launch_gather_block(C(ctx), A, lda, I, k, J, l, G, ldg);
}

int slra_sketch_cols(slra_ctx ctx, const double* A, int64_t lda, int64_t m, int64_t n, const int64_t* src,
                     const double* coef, const int32_t* q, int64_t width, int tree, int64_t l, double* out,
                     int64_t ldo) {
  (void)n;
  if (!ctx || lda < m || ldo < m || width < 1 || l < 0) return SLRA_ERR_INVALID_ARGUMENT;
  if (tree == SLRA_TREE_FWHT && (width & (width - 1))) return SLRA_ERR_INVALID_ARGUMENT;
  if (l == 0 || m == 0) return SLRA_OK;
  return launch_sketch_cols(C(ctx), A, lda, m, src, coef, q, width, tree, l, out, ldo);
}

int slra_sketch_rows(slra_ctx ctx, const double* Wm, int64_t ldw, int64_t m, int64_t ncols, const int64_t* src,
                     const double* coef, const int32_t* q, int64_t width, int tree, int64_t k, double* out,
                     int64_t ldo) {
  if (!ctx || ldw < m || ldo < k || width < 1 || k < 0) return SLRA_ERR_INVALID_ARGUMENT;
  if (tree == SLRA_TREE_FWHT && (width & (width - 1))) return SLRA_ERR_INVALID_ARGUMENT;
  if (k == 0 || ncols == 0) return SLRA_OK;
  return launch_sketch_rows(C(ctx), Wm, ldw, ncols, src, coef, q, width, tree, k, out, ldo);
}

int slra_sketch_rows_shard(slra_ctx ctx, const double* Wm, int64_t ldw, int64_t row0, int64_t mloc, int64_t ncols,
                           const int64_t* src, const double* coef, int64_t width, int64_t k, double* out,
                           int64_t ldo, int transpose) {
  if (!ctx || ldw < mloc || mloc < 0 || row0 < 0 || width < 1 || k < 0 || ncols < 0) return SLRA_ERR_INVALID_ARGUMENT;
  if (ldo < (transpose ? ncols : k)) return SLRA_ERR_INVALID_ARGUMENT;
  if (k == 0 || ncols == 0) return SLRA_OK;
  Context* c = C(ctx);
  SLRA_TIMED(c, "sketch", sketch_rows_shard_kernel<<<grid_1d(c, k * ncols), kNT, 0, c->stream>>>(
                              Wm, ldw, row0, mloc, ncols, src, coef, width, k, out, ldo, transpose);)
  SLRA_CHECK_LAUNCH(c);
  return SLRA_OK;
}

}  // extern "C"
