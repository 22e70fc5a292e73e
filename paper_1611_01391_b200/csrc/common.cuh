// Shared device/runtime helpers for the sm_100a kernels behind slra_cuda.h.
#pragma once

#include <nvtx3/nvToolsExt.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cfloat>
#include <cmath>
#include <mutex>
#include <string>
#include <vector>

#include "slra_cuda.h"

namespace slra_dev {

// Jacobi rotation (c, s) from the pair's Gram entries a = |x|^2, b = |y|^2,
// g = x.y: t = sign(d) 2g / (|d| + sqrt(d^2 + 4g^2)), d = b - a, c = 1 /
// sqrt(1 + t^2), s = c t. Only the orthogonality of the rotation matters for
// the one-sided Jacobi result (sigma are the final column norms, checked by
// the orthogonality threshold); the angle itself may be off by the hardware
// seed's ~2^-22, which the next sweep absorbs. So t comes from the MUFU
// rsqrt / rcp seeds (rsqrt.approx.f64, rcp.approx.ftz.f64: one instruction
// each instead of the IEEE sqrt and division sequences), while c is refined
// to full precision (two Newton steps) so that c^2 + s^2 = 1 to rounding.
__device__ __forceinline__ double mufu_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__device__ __forceinline__ double mufu_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
// Full-precision (<= ~1 ulp, not correctly rounded) reciprocal and square
// root from the MUFU seeds with Newton steps: a handful of dependent DFMAs
// instead of the IEEE division / sqrt sequences (with their slow-path
// branches). For the reflector and norm chains of the small factorisations,
// whose results are compared with the oracle by value, not by bits. x must be
// finite; fast_rcp needs |x| in the normal range.
__device__ __forceinline__ double fast_rcp(double x) {
  double y = mufu_rcp(x);
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ double fast_rsqrt(double x) {  // x > 0, normal
  double y = mufu_rsqrt(x);
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  return y * fma(-hx * y, y, 1.5);
}
__device__ __forceinline__ double fast_sqrt(double x) {
  double y = mufu_rsqrt(x);
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  const double s = x * y;
  const double r = fma(0.5 * y, fma(-s, s, x), s);
  return x > 0.0 ? r : x;  // sqrt(0) = 0 (rsqrt(0) = inf)
}
// Householder reflector scalars of makeHouseholder (c0 the pivot entry, tail the
// squared norm of the entries below it, tail > DBL_MIN): beta = -sgn sqrt(v),
// rden = 1 / (c0 - beta) = sgn / (|c0| + sqrt(v)), tau = (beta - c0) / beta =
// 1 + |c0| / sqrt(v), v = c0^2 + tail — arranged for the shortest dependent
// chain (one cubic step from each MUFU seed, no corrected sqrt and no division
// on the way to rden; FP64 dependent latency is ~35-40 cycles and a reflector
// sits on the critical path of every pivot). ~1 ulp, not correctly rounded.
__device__ __forceinline__ void fast_reflector(double c0, double tail, double& beta, double& rden, double& tau) {
  const double v = fma(c0, c0, tail), ac = fabs(c0);
  const double y0 = mufu_rsqrt(v);
  const double e = fma(-(v * y0), y0, 1.0);
  const double y = fma(y0, e * fma(0.375, e, 0.5), y0);
  const double den = fma(v, y, ac);
  const double r0 = mufu_rcp(den);
  const double er = fma(-den, r0, 1.0);
  rden = copysign(fma(r0, fma(er, er, er), r0), c0 >= 0.0 ? 1.0 : -1.0);
  const double sq = v * y;
  const double sqc = fma(0.5 * y, fma(-sq, sq, v), sq);
  beta = c0 >= 0.0 ? -sqc : sqc;
  tau = fma(ac, y, 1.0);
}
__device__ __forceinline__ void jacobi_rotation(double a, double b, double g, double& cs, double& sn) {
  const double d = b - a, g2 = 2.0 * g;
  const double h = fma(d, d, g2 * g2);
  if (!(h < 0.125 * DBL_MAX) || h < DBL_MIN) {
    // overflowing (column norms above ~1e154; 4 h is formed below) or subnormal Gram entries: the
    // IEEE sqrt / divide (the MUFU seeds would give inf * 0 or flush to zero)
    const double t = (g2 * g2 < 1e-17 * (d * d)) ? g2 / (2.0 * d) : copysign(1.0, d) * g2 / (fabs(d) + sqrt(h));
    cs = 1.0 / sqrt(fma(t, t, 1.0));
    sn = cs * t;
    return;
  }
  // c = w / sqrt(2 s w), s = sign(d) g2 / sqrt(2 s w) with s = sqrt(h), w = |d| + s
  // (t = g2 / w, 1 + t^2 = 2 s / w): both square roots from the MUFU seed (the
  // angle is then off by ~2^-22, as before), and the pair (c, s) renormalised to
  // c^2 + s^2 = 1 by the second-order series of rsqrt(1 + e), e = c^2 + s^2 - 1
  // ~ 2^-21 (e^3 is below the rounding): 13 dependent operations instead of 17
  // (FP64 dependent latency is what a Jacobi round is made of).
  const double s = h * mufu_rsqrt(h);
  const double w = fabs(d) + s;
  const double rz = mufu_rsqrt(2.0 * s * w);
  const double c0 = w * rz, s0 = copysign(g2, d * g2) * rz;
  const double e = fma(c0, c0, fma(s0, s0, -1.0));
  const double f = fma(e, fma(0.375, e, -0.5), 1.0);
  cs = c0 * f;
  sn = s0 * f;
}

// ------------------------------------------------------------------ context
constexpr int kArenaSlots = 14;

struct Context {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  bool owns_stream = false;
  // copy streams + events of the host-streamed batched C-A (created on first use)
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev[6] = {};
  int64_t launches = 0;
  // growable scratch (device) and pinned host scratch
  void* ws = nullptr;
  size_t ws_bytes = 0;
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  // per-CTA partial sums of the two-stage reductions
  double* partials = nullptr;
  int partials_cap = 0;
  // small persistent device scratch (statuses, ranks, flags): 4096 bytes
  void* dsmall = nullptr;
  // pinned host mirror of dsmall for status read-back
  void* hsmall = nullptr;
  // independent growable device arenas for multi-kernel orchestrations
  // (0: range finder, 1: cur residual, 2: lsr, 3: svd, 4: large C-A, 5: factored residual,
  //  6: wide-svd transpose, 7: tall maxvol/select, 8: pinv, 9: premult / two-stage truncate,
  //  10: large (multi-CTA Jacobi) svd, 11: hss, 12: host-streamed batched C-A,
  //  13: exact (column-pivoted QR) least squares)
  void* arena[kArenaSlots] = {};
  size_t arena_bytes[kArenaSlots] = {};
  // opt-in per-kernel-family timing (CUDA events on the context stream)
  bool timing = false;
  struct Rec {
    const char* family;
    cudaEvent_t start, stop;
  };
  std::vector<Rec> records;
  std::vector<cudaEvent_t> event_pool;
};

cudaEvent_t pooled_event(Context* c);

// Records start/stop events around one kernel launch when timing is on, and
// always an NVTX range named after the kernel family (header-only NVTX3: a
// no-op unless a profiler injects itself, e.g. ncu --nvtx / nsys).
struct KernelTimer {
  Context* c;
  const char* family;
  cudaEvent_t start = nullptr;
  KernelTimer(Context* ctx, const char* fam) : c(ctx), family(fam) {
    nvtxRangePushA(fam);
    if (c->timing) {
      start = pooled_event(c);
      cudaEventRecord(start, c->stream);
    }
  }
  ~KernelTimer() {
    if (start) {
      cudaEvent_t stop = pooled_event(c);
      cudaEventRecord(stop, c->stream);
      c->records.push_back({family, start, stop});
    }
    nvtxRangePop();
  }
};

#define SLRA_TIMED(ctx, fam, ...)                  \
  {                                                \
    slra_dev::KernelTimer _slra_kt((ctx), (fam));  \
    __VA_ARGS__                                    \
  }

void set_last_error(const std::string& s);
int cuda_status(cudaError_t e, const char* where);
// Scratch of at least `bytes` (device). Synchronizes the stream when it grows.
void* workspace(Context* c, size_t bytes);
void* pinned_scratch(Context* c, size_t bytes);
double* partials(Context* c, int n);
void* arena(Context* c, int slot, size_t bytes);

#define SLRA_CHECK_LAUNCH(ctx)                                          \
  do {                                                                  \
    (ctx)->launches++;                                                  \
    cudaError_t _e = cudaGetLastError();                                \
    if (_e != cudaSuccess) return slra_dev::cuda_status(_e, __func__);  \
  } while (0)

#define SLRA_CUDA(call)                                                 \
  do {                                                                  \
    cudaError_t _e = (call);                                            \
    if (_e != cudaSuccess) return slra_dev::cuda_status(_e, #call);     \
  } while (0)

#define SLRA_TRY(expr)              \
  do {                              \
    int _s = (expr);                \
    if (_s != SLRA_OK) return _s;   \
  } while (0)

inline Context* C(slra_ctx c) { return reinterpret_cast<Context*>(c); }

// ------------------------------------------------------------------ device helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum, result broadcast to every thread. `red` >= 33 doubles of smem.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double t = lane < NT / 32 ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

// Argmax key: larger value wins; ties -> smaller index (Eigen maxCoeff keeps
// the first maximum in traversal order).
struct ArgMax {
  double v;
  int64_t i;
};
__device__ __forceinline__ ArgMax argmax_merge(ArgMax a, ArgMax b) {
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}
__device__ __forceinline__ ArgMax warp_argmax(ArgMax a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgMax b;
    b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
    b.i = __shfl_xor_sync(0xffffffffu, a.i, o);
    a = argmax_merge(a, b);
  }
  return a;
}
// Block argmax broadcast to all threads; `rv` >= 33 doubles, `ri` >= 33 int64.
template <int NT>
__device__ __forceinline__ ArgMax block_argmax(ArgMax a, double* rv, int64_t* ri) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  a = warp_argmax(a);
  __syncthreads();
  if (lane == 0) {
    rv[warp] = a.v;
    ri[warp] = a.i;
  }
  __syncthreads();
  if (warp == 0) {
    ArgMax t;
    t.v = lane < NT / 32 ? rv[lane] : -1.0;
    t.i = lane < NT / 32 ? ri[lane] : INT64_MAX;
    t = warp_argmax(t);
    if (lane == 0) {
      rv[32] = t.v;
      ri[32] = t.i;
    }
  }
  __syncthreads();
  ArgMax out;
  out.v = rv[32];
  out.i = ri[32];
  return out;
}

// FP64 tensor-core MMA (sm_80+ mma.sync; SASS DMMA.8x8x4 on sm_100a).
// A 8x4 row: a = A[lane>>2][lane&3]; B 4x8 col: b = B[lane&3][lane>>2];
// C 8x8: c0,c1 = C[lane>>2][2*(lane&3) + {0,1}].
// Load p[ok ? i : 0] unconditionally and select afterwards: a guarded load
// (`ok ? p[i] : 0`) compiles to a branch around each load, which serialises
// a batch of loads on their full latency; this form keeps them all in flight.
// p[0] must be a valid address.
template <typename T>
__device__ __forceinline__ T load_sel(const T* p, int64_t i, bool ok) {
  const T v = p[ok ? i : 0];
  return ok ? v : T(0);
}

// m16n8k16 FP64 MMA (8x the work of m8n8k4 per PTX instruction; on sm_100a
// ptxas lowers it to a sequence of DMMA.8x8x4 — the SASS has no wider FP64
// MMA — so the gain is fewer issued instructions, not a wider unit).
// Fragments (g = lane >> 2, t = lane & 3), from the PTX f64 m16n8k16 layout
// (as in CuTe's SM90_16x8x16_F64F64F64F64_TN traits):
//   a[v] = A[g + 8 (v & 1)][t + 4 (v >> 1)]      v = 0..7  (A 16 x 16, row)
//   b[v] = B[t + 4 v][g]                          v = 0..3  (B 16 x 8, col)
//   c[v] = C[g + 8 (v >> 1)][2 t + (v & 1)]       v = 0..3  (C 16 x 8)
__device__ __forceinline__ void dmma_16x8x16(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
        "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

// Phase timing of the CTA-resident kernels (profiling builds only,
// -DSLRA_PHASE_PROF): thread 0 adds the clock64 cycles since its previous
// mark to g_phase_cycles[id]. Marks sit right after block barriers, so the
// intervals are the block's critical path per phase.
#ifdef SLRA_PHASE_PROF
__device__ unsigned long long g_phase_cycles[32];
__device__ __forceinline__ void prof_mark(int id) {
  __shared__ long long t_last;
  if (threadIdx.x == 0) {
    const long long now = clock64();
    if (id >= 0) atomicAdd(&g_phase_cycles[id], (unsigned long long)(now - t_last));
    t_last = now;
  }
}
#define SLRA_PROF(id) ::slra_dev::prof_mark(id)
#else
#define SLRA_PROF(id) ((void)0)
#endif

}  // namespace slra_dev
