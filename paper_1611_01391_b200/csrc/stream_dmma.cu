// Streaming FP64 tensor-core kernels for the two HBM-sized products of the
// hot path (both read A once, FLOP:byte ~8 at inner dimension 32, i.e. just
// above the B200 FP64 ridge of 37.2 TF/s / 6.55 TB/s ~ 5.7):
//
//   residual_stream:  sum (A - P Q)^2 and sum A^2 over A (m x n), P m x r,
//                     Q r x n, r <= 32  — cur_evaluate(M, c, Frobenius)
//                     (cur.cpp:80-82) and ||M - U V||_F (lra.cpp:35-36).
//   tn_skinny:        C = W^T B (r x n, r <= 64) — V = U^+ M / U^T M of the
//                     range finder (lra.cpp:35-36).
//
// Both stage their tiles with cp.async (16-byte, zero-filled at the edges)
// into double-buffered shared memory so the next tile streams in while the
// current one runs on DMMA (mma.sync.m8n8k4.f64), and both reduce
// deterministically (fixed per-CTA partials, fixed-order final sum).
#include "common.cuh"

namespace slra_dev {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---------------------------------------------------------------- residual
// Each CTA walks a contiguous range of 128 x 32 tiles of A, row block by
// row block. Each warp owns 16 rows of the block, and its P fragments (16
// rows x 32 inner, the whole m16n8k16 A operand for every tile of the row
// block) stay in REGISTERS, so per tile only the A tile and the 32 x 32 Q
// tile stream through shared memory (cp.async, NS stages in flight). Two
// CTAs per SM: one CTA's MMAs run while the other sits in its epilogue or
// barrier (ncu: with one CTA per SM the DMMA pipe idled through every
// epilogue, 52 % active).
namespace rs {
constexpr int NT = 256;        // 8 warps, 16 * MI rows each
constexpr int MI = 1;          // m16 blocks per warp
constexpr int TM = 8 * 16 * MI;  // tile rows (row block)
#ifndef SLRA_RS_TN
#define SLRA_RS_TN 32
#endif
#ifndef SLRA_RS_NS
#define SLRA_RS_NS 2
#endif
constexpr int TN = SLRA_RS_TN; // tile cols
constexpr int NI = TN / 8;     // n8 fragments per tile
constexpr int KP = 32;         // inner dimension (padded)
constexpr int LDV = KP + 4;    // Vs[col][k]: conflict-free B fragment reads
constexpr int LDM = TM + 2;    // Ms[col][row]: conflict-free epilogue reads
constexpr int V_D = TN * LDV;  // doubles per Q stage
constexpr int M_D = TN * LDM;  // doubles per A stage
constexpr int NS = SLRA_RS_NS; // stages (NS - 1 tiles in flight behind the current one)
constexpr size_t SMEM = sizeof(double) * NS * (V_D + M_D);
}  // namespace rs

struct StreamResidualArgs {
  const double* A;
  int64_t lda, m, n;
  const double* P;
  int64_t ldp;
  const double* Q;
  int64_t ldq;
  int inner;
  double* part;  // 2 per CTA
  // Cauchy FunctionOracle (config 3: A_ij = 1/(x_i - y_j), one IEEE
  // division): the A tiles are evaluated instead of loaded (null: dense)
  const double* cx = nullptr;
  const double* cy = nullptr;
};

template <bool CAU>
__device__ __forceinline__ void rs_stage(const StreamResidualArgs& a, int64_t i0, int64_t j0, double* Vs,
                                         double* Ms) {
  using namespace rs;
  const int tid = threadIdx.x;
  if constexpr (CAU) {
    // evaluated A tile: the same values the materialised matrix holds
#pragma unroll 4
    for (int e = tid; e < TN * (TM / 2); e += NT) {
      const int col = e / (TM / 2), ch = e % (TM / 2);
      const int64_t r = i0 + 2 * ch, cc = j0 + col;
      const bool cin = cc < a.n;
      const double yc = cin ? __ldg(a.cy + cc) : 0.0;
      const double v0 = (cin && r < a.m) ? __ddiv_rn(1.0, __dsub_rn(__ldg(a.cx + r), yc)) : 0.0;
      const double v1 = (cin && r + 1 < a.m) ? __ddiv_rn(1.0, __dsub_rn(__ldg(a.cx + r + 1), yc)) : 0.0;
      *reinterpret_cast<double2*>(Ms + col * LDM + 2 * ch) = make_double2(v0, v1);
    }
  }
  // A tile: TN columns x TM rows in 16-byte chunks of 2 rows (a column is
  // 2 KB contiguous in HBM)
#pragma unroll 4
  for (int e = tid; e < (CAU ? 0 : TN * (TM / 2)); e += NT) {
    const int col = e / (TM / 2), ch = e % (TM / 2);
    const int64_t r = i0 + 2 * ch, cc = j0 + col;
    int bytes = 0;
    const double* src = a.A;
    if (cc < a.n && r < a.m) {
      bytes = (r + 1 < a.m) ? 16 : 8;
      src = a.A + r + cc * a.lda;
    }
    cp_async16(Ms + col * LDM + 2 * ch, src, bytes);
  }
  // Q tile: per column the inner entries are contiguous
  for (int e = tid; e < TN * (KP / 2); e += NT) {
    const int col = e / (KP / 2), ch = e % (KP / 2);
    const int k = 2 * ch;
    const int64_t cc = j0 + col;
    int bytes = 0;
    const double* src = a.Q;
    if (cc < a.n && k < a.inner) {
      bytes = (k + 1 < a.inner) ? 16 : 8;
      src = a.Q + k + cc * a.ldq;
    }
    cp_async16(Vs + col * LDV + k, src, bytes);
  }
}

template <bool CAU>
__device__ __forceinline__ void residual_stream_body(const StreamResidualArgs& a) {
  using namespace rs;
  extern __shared__ __align__(16) double smem[];
#define VB(s) (smem + (s) * V_D)
#define MB(s) (smem + NS * V_D + (s) * M_D)
  __shared__ double red[40];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int64_t tiles_m = (a.m + TM - 1) / TM, tiles_n = (a.n + TN - 1) / TN;
  const int64_t tiles = tiles_m * tiles_n;
  // contiguous tile range per CTA, row-block major (the P fragments change
  // only when the range crosses into the next row block)
  const int64_t t0 = tiles * blockIdx.x / gridDim.x, t1 = tiles * (blockIdx.x + 1) / gridDim.x;
  const int nkk = (a.inner + 15) >> 4;  // k16 steps (0, 1 or 2)
  double rsum = 0.0, nsum = 0.0;
#pragma unroll
  for (int s = 0; s < NS - 1; ++s) {
    const int64_t t = t0 + s;
    if (t < t1) rs_stage<CAU>(a, (t / tiles_n) * TM, (t % tiles_n) * TN, VB(s), MB(s));
    cp_async_commit();
  }
  double af[MI][2][8];  // [m16 block][k16 step][fragment]
  int64_t rb_loaded = -1;
  int slot = 0;
  for (int64_t t = t0; t < t1; ++t) {
    // tile t landed (NS - 2 newer groups may still fly); after the barrier
    // every warp is past tile t - 1, so its slot can take tile t + NS - 1
    // (prefetched below, behind this tile's DMMAs): one barrier per tile
    cp_async_wait<NS - 2>();
    __syncthreads();
    const int64_t rb = t / tiles_n;
    if (rb != rb_loaded) {  // P fragments of this warp's 32 rows (zero outside P)
      rb_loaded = rb;
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int kk = 0; kk < 2; ++kk)
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            const int64_t row = rb * TM + warp * 16 * MI + mi * 16 + g + 8 * (v & 1);
            const int k = kk * 16 + t4 + 4 * (v >> 1);
            af[mi][kk][v] = (row < a.m && k < a.inner) ? __ldg(a.P + row + (int64_t)k * a.ldp) : 0.0;
          }
    }
    const double* Vs = VB(slot);
    const double* Ms = MB(slot) + warp * 16 * MI;
    double acc[MI][NI][4];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
      for (int ni = 0; ni < NI; ++ni)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[mi][ni][v] = 0.0;
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      if (kk < nkk) {
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          double bf[4];
#pragma unroll
          for (int v = 0; v < 4; ++v) bf[v] = Vs[(ni * 8 + g) * LDV + kk * 16 + t4 + 4 * v];
#pragma unroll
          for (int mi = 0; mi < MI; ++mi) dmma_16x8x16(acc[mi][ni], af[mi][kk], bf);
        }
      }
    }
    {  // prefetch tile t + NS - 1 while the DMMAs above drain (issued after them in program order)
      const int64_t tp = t + NS - 1;
      const int sp = (slot + NS - 1) % NS;
      if (tp < t1) rs_stage<CAU>(a, (tp / tiles_n) * TM, (tp % tiles_n) * TN, VB(sp), MB(sp));
      cp_async_commit();
    }
    double r0 = 0.0, r1 = 0.0, n0 = 0.0, n1 = 0.0;  // short chains (FP64 FMA latency)
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
      for (int ni = 0; ni < NI; ++ni)
#pragma unroll
        for (int v = 0; v < 4; v += 2) {
          const int row = mi * 16 + g + 8 * (v >> 1), col = ni * 8 + 2 * t4;
          const double x0 = Ms[col * LDM + row], x1 = Ms[(col + 1) * LDM + row];  // zero outside A
          const double d0 = x0 - acc[mi][ni][v], d1 = x1 - acc[mi][ni][v + 1];
          r0 = fma(d0, d0, r0);
          r1 = fma(d1, d1, r1);
          n0 = fma(x0, x0, n0);
          n1 = fma(x1, x1, n1);
        }
    rsum += r0 + r1;
    nsum += n0 + n1;
    slot = (slot + 1) % NS;
  }
  cp_async_wait<0>();
#undef VB
#undef MB
  rsum = block_sum<NT>(rsum, red);
  nsum = block_sum<NT>(nsum, red);
  if (threadIdx.x == 0) {
    a.part[2 * blockIdx.x] = rsum;
    a.part[2 * blockIdx.x + 1] = nsum;
  }
}

__global__ void __launch_bounds__(rs::NT, 2) residual_stream_kernel(StreamResidualArgs a) {
  residual_stream_body<false>(a);
}
__global__ void __launch_bounds__(rs::NT, 2) cauchy_residual_stream_kernel(StreamResidualArgs a) {
  residual_stream_body<true>(a);
}

__global__ void reduce_pairs2_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
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

// Returns SLRA_ERR_UNSUPPORTED when the shape/alignment does not suit the
// streaming kernel (caller falls back to the generic one).
int launch_residual_stream(Context* c, const double* A, int64_t lda, int64_t m, int64_t n, const double* P,
                           int64_t ldp, const double* Q, int64_t ldq, int64_t inner, double* d_out) {
  const bool aligned = ((uintptr_t)A % 16 == 0) && (lda % 2 == 0) && (inner == 0 || (((uintptr_t)P % 16 == 0) &&
                       (ldp % 2 == 0) && ((uintptr_t)Q % 16 == 0) && (ldq % 2 == 0)));
  if (!aligned || inner > rs::KP || m < 1 || n < 1) return SLRA_ERR_UNSUPPORTED;
  const int64_t tiles = ((m + rs::TM - 1) / rs::TM) * ((n + rs::TN - 1) / rs::TN);
  int grid = 2 * c->num_sms;  // two co-resident CTAs per SM: their epilogues and barriers interleave
  if (tiles < grid) grid = (int)tiles;
  double* part = partials(c, 2 * grid);
  if (!part) return SLRA_ERR_CUDA;
  StreamResidualArgs a{A, lda, m, n, inner ? P : A, inner ? ldp : 2, inner ? Q : A, inner ? ldq : 2, (int)inner,
                       part};
  SLRA_CUDA(cudaFuncSetAttribute(residual_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rs::SMEM));
  SLRA_TIMED(c, "residual", residual_stream_kernel<<<grid, rs::NT, rs::SMEM, c->stream>>>(a);)
  SLRA_CHECK_LAUNCH(c);
  SLRA_TIMED(c, "residual_reduce", reduce_pairs2_kernel<<<1, 256, 0, c->stream>>>(part, grid, d_out);)
  SLRA_CHECK_LAUNCH(c);
  return SLRA_OK;
}

// ||A - P Q||^2 and ||A||^2 for the Cauchy block A_ij = 1/(x_i - y_j) (m x n).
int launch_residual_stream_cauchy(Context* c, const double* x, const double* y, int64_t m, int64_t n,
                                  const double* P, int64_t ldp, const double* Q, int64_t ldq, int64_t inner,
                                  double* d_out) {
  const bool aligned = inner == 0 || (((uintptr_t)P % 16 == 0) && (ldp % 2 == 0) && ((uintptr_t)Q % 16 == 0) &&
                                      (ldq % 2 == 0));
  if (!aligned || inner > rs::KP || m < 1 || n < 1) return SLRA_ERR_UNSUPPORTED;
  const int64_t tiles = ((m + rs::TM - 1) / rs::TM) * ((n + rs::TN - 1) / rs::TN);
  int grid = 2 * c->num_sms;
  if (tiles < grid) grid = (int)tiles;
  double* part = partials(c, 2 * grid);
  if (!part) return SLRA_ERR_CUDA;
  StreamResidualArgs a{x, 2, m, n, inner ? P : x, inner ? ldp : 2, inner ? Q : x, inner ? ldq : 2, (int)inner, part,
                       x, y};
  SLRA_CUDA(cudaFuncSetAttribute(cauchy_residual_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)rs::SMEM));
  SLRA_TIMED(c, "residual", cauchy_residual_stream_kernel<<<grid, rs::NT, rs::SMEM, c->stream>>>(a);)
  SLRA_CHECK_LAUNCH(c);
  SLRA_TIMED(c, "residual_reduce", reduce_pairs2_kernel<<<1, 256, 0, c->stream>>>(part, grid, d_out);)
  SLRA_CHECK_LAUNCH(c);
  return SLRA_OK;
}

// ---------------------------------------------------------------- C = W^T B
// W (K x r, ld ldw), B (K x n, ld ldb), C (r x n, ld ldc), r <= 56.
// CTA = 64 output columns x one K-slice; warp w owns columns 8 w .. 8 w + 7
// for ALL r rows (RF 8 x 8 fragments: 2 RF accumulator registers), so there
// is no cross-warp reduction and the register footprint is small enough for
// two co-resident CTAs per SM (one CTA's DMMAs run while the other waits on
// its barrier or its loads). K streams through a cp.async ring of TK-row
// stages (one barrier per stage); per 4-row step a warp loads RF + 1
// fragments for RF DMMAs. The K dimension is split stream-K style (below).
namespace tn {
constexpr int NT = 256;
#ifndef SLRA_TN_TK
#define SLRA_TN_TK 64
#endif
#ifndef SLRA_TN_NS
#define SLRA_TN_NS 2
#endif
#ifndef SLRA_TN_CTAS
#define SLRA_TN_CTAS 2
#endif
constexpr int TK = SLRA_TN_TK; // K rows per stage
constexpr int TN = 64;         // output columns per CTA
constexpr int NS = SLRA_TN_NS; // stages
constexpr int CTAS = SLRA_TN_CTAS;  // co-resident CTAs per SM the launch is sized for
constexpr int LDB = TK + 4;    // [col][k]: fragment loads hit 16 different banks per half-warp
constexpr int B_D = TN * LDB;
inline size_t smem_bytes(int RF) { return sizeof(double) * NS * (size_t)(RF * 8 * LDB + B_D); }
}  // namespace tn

struct TnArgs {
  const double* W;
  int64_t ldw;
  const double* B;
  int64_t ldb;
  int64_t K, n;
  int r;
  int S;         // stages per column tile (ceil(K / TK))
  int64_t U;     // stage units in all: column tiles x S
  double* part;  // partial blocks: [piece][r x n] (ld r)
};
// Stream-K split: the flattened (column tile, stage) units are cut into
// gridDim.x equal contiguous ranges — every CTA runs the same number of
// stages (+-1) whatever n and K are, so there is no partial last wave. A
// range that crosses a tile boundary ends one partial block and starts the
// next; the piece index of a segment is its CTA's distance from the first
// CTA that touches the tile, so the combine adds the pieces of a tile in CTA
// order (deterministic).
__host__ __device__ inline int64_t tn_first_unit(int64_t i, int64_t U, int64_t G) { return i * U / G; }
__host__ __device__ inline int64_t tn_owner(int64_t u, int64_t U, int64_t G) { return ((u + 1) * G - 1) / U; }

template <int RF>
__device__ __forceinline__ void tn_stage(const TnArgs& a, int64_t k0, int64_t j0, int64_t kend, double* Ws,
                                         double* Bs) {
  using namespace tn;
  const int tid = threadIdx.x;
  // W^T tile: Ws[q][k] (W is column-major K x r: a column's rows are contiguous)
  for (int e = tid; e < RF * 8 * (TK / 2); e += NT) {
    const int q = e / (TK / 2), ch = e % (TK / 2);
    const int64_t k = k0 + 2 * ch;
    int bytes = 0;
    const double* src = a.W;
    if (q < a.r && k < kend) {
      bytes = (k + 1 < kend) ? 16 : 8;
      src = a.W + k + (int64_t)q * a.ldw;
    }
    cp_async16(Ws + q * LDB + 2 * ch, src, bytes);
  }
#pragma unroll
  for (int e = tid; e < TN * (TK / 2); e += NT) {
    const int col = e / (TK / 2), ch = e % (TK / 2);
    const int64_t k = k0 + 2 * ch, cc = j0 + col;
    int bytes = 0;
    const double* src = a.B;
    if (cc < a.n && k < kend) {
      bytes = (k + 1 < kend) ? 16 : 8;
      src = a.B + k + cc * a.ldb;
    }
    cp_async16(Bs + col * LDB + 2 * ch, src, bytes);
  }
}

template <int RF>  // RF = r rounded up to 8, in fragments of 8 (1..7)
__global__ void __launch_bounds__(tn::NT, tn::CTAS) tn_skinny_kernel(TnArgs a) {
  using namespace tn;
  extern __shared__ __align__(16) double smem[];
  constexpr int W_D = RF * 8 * LDB;
#define WB(b) (smem + (b) * (W_D + B_D))
#define BB(b) (smem + (b) * (W_D + B_D) + W_D)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int64_t G = gridDim.x;
  int64_t u = tn_first_unit(blockIdx.x, a.U, G);
  const int64_t u1 = tn_first_unit(blockIdx.x + 1, a.U, G);
  while (u < u1) {
    const int64_t jt = u / a.S;
    const int sa = (int)(u - jt * a.S);
    const int nst = (int)((u1 - u) < (a.S - sa) ? (u1 - u) : (a.S - sa));
    const int64_t j0 = jt * TN, kb = (int64_t)sa * TK, ke = a.K;
    double acc[RF][2];
#pragma unroll
    for (int mi = 0; mi < RF; ++mi) acc[mi][0] = acc[mi][1] = 0.0;
#pragma unroll
    for (int s = 0; s < NS - 1; ++s) {
      if (s < nst) tn_stage<RF>(a, kb + (int64_t)s * TK, j0, ke, WB(s), BB(s));
      cp_async_commit();
    }
    int slot = 0;
    for (int st = 0; st < nst; ++st) {
      // stage st landed (NS - 2 newer groups may still fly); after the barrier
      // every warp is past stage st - 1, whose slot takes stage st + NS - 1
      cp_async_wait<NS - 2>();
      __syncthreads();
      {
        const int sn = st + NS - 1;
        const int sp = (slot + NS - 1) % NS;
        if (sn < nst) tn_stage<RF>(a, kb + (int64_t)sn * TK, j0, ke, WB(sp), BB(sp));
        cp_async_commit();
      }
      const double* Ws = WB(slot) + g * LDB + t4;
      const double* Bs = BB(slot) + (warp * 8 + g) * LDB + t4;
#pragma unroll
      for (int s = 0; s < TK / 4; ++s) {
        double af[RF];
        const double bf = Bs[4 * s];
#pragma unroll
        for (int mi = 0; mi < RF; ++mi) af[mi] = Ws[mi * 8 * LDB + 4 * s];
#pragma unroll
        for (int mi = 0; mi < RF; ++mi) dmma_8x8x4(acc[mi][0], acc[mi][1], af[mi], bf);
      }
      slot = (slot + 1) % NS;
    }
    cp_async_wait<0>();
    // lane (g, t4) holds C(8 mi + g, 8 warp + 2 t4 + e) of this segment
    const int64_t piece = (int64_t)blockIdx.x - tn_owner(jt * a.S, a.U, G);
    double* out = a.part + piece * a.r * a.n;
#pragma unroll
    for (int mi = 0; mi < RF; ++mi)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int row = mi * 8 + g;
        const int64_t cc = j0 + warp * 8 + 2 * t4 + e;
        if (row < a.r && cc < a.n) out[row + cc * a.r] = acc[mi][e];
      }
    u += nst;
    __syncthreads();  // every warp is done with the ring before the next segment refills it
  }
#undef WB
#undef BB
}

// C = alpha * (sum of the pieces of each column tile, in CTA order). Block
// (q, jt) takes a quarter (16 columns) of column tile jt: the piece count is
// computed once per block and every piece's load is in flight before the sum.
__global__ void __launch_bounds__(256) streamk_sum_kernel(const double* __restrict__ part, int r, int64_t n, int S,
                                                          int64_t U, int64_t G, double alpha,
                                                          double* __restrict__ Cm, int64_t ldc) {
  const int64_t jt = blockIdx.y;
  const int cnt = (int)(tn_owner(jt * S + S - 1, U, G) - tn_owner(jt * S, U, G)) + 1;
  const int64_t total = (int64_t)r * n;
  const int64_t c0 = jt * tn::TN + blockIdx.x * 16;
  for (int e = threadIdx.x; e < 16 * r; e += 256) {
    const int col = e / r, row = e - col * r;
    const int64_t cc = c0 + col;
    if (cc >= n) continue;
    const double* p = part + row + cc * r;
    double s = 0.0;
    int z = 0;
    for (; z + 4 <= cnt; z += 4) {
      const double v0 = p[z * total], v1 = p[(z + 1) * total], v2 = p[(z + 2) * total], v3 = p[(z + 3) * total];
      s = ((s + v0) + v1) + v2 + v3;
    }
    for (; z < cnt; ++z) s += p[z * total];
    Cm[row + cc * ldc] = alpha * s;
  }
}

// C (r x n) = alpha * W^T B. Returns SLRA_ERR_UNSUPPORTED when unsuitable.
int launch_tn_skinny(Context* c, const char* fam, int64_t r, int64_t n, int64_t K, double alpha, const double* W,
                     int64_t ldw, const double* B, int64_t ldb, double* Cm, int64_t ldc) {
  const bool aligned = ((uintptr_t)W % 16 == 0) && (ldw % 2 == 0) && ((uintptr_t)B % 16 == 0) && (ldb % 2 == 0);
  if (!aligned || r < 1 || r > 56 || K < 256) return SLRA_ERR_UNSUPPORTED;  // r > 56 would spill
  const int gx = ceil_div(n, tn::TN);
  if (gx > 65535) return SLRA_ERR_UNSUPPORTED;  // the combine's grid.y (caller falls back to the generic GEMM)
  const int S = ceil_div(K, tn::TK);
  const int64_t U = (int64_t)gx * S;
  const int64_t slots = (int64_t)tn::CTAS * c->num_sms;
  const int64_t G = U < slots ? U : slots;
  int pmax = 1;  // most pieces of one column tile
  for (int64_t jt = 0; jt < gx; ++jt) {
    const int cnt = (int)(tn_owner(jt * S + S - 1, U, G) - tn_owner(jt * S, U, G)) + 1;
    if (cnt > pmax) pmax = cnt;
  }
  double* part = static_cast<double*>(workspace(c, sizeof(double) * r * n * pmax));
  if (!part) return SLRA_ERR_CUDA;
  TnArgs a{W, ldw, B, ldb, K, n, (int)r, S, U, part};
  const int RF = (int)((r + 7) / 8);
  const size_t smem = tn::smem_bytes(RF);
  dim3 grid((unsigned)G);
#define SLRA_TN_CASE(RFV)                                                                                     \
  case RFV:                                                                                                   \
    SLRA_CUDA(cudaFuncSetAttribute(tn_skinny_kernel<RFV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    SLRA_TIMED(c, fam, tn_skinny_kernel<RFV><<<grid, tn::NT, smem, c->stream>>>(a);)                        \
    break;
  switch (RF) {
    SLRA_TN_CASE(1)
    SLRA_TN_CASE(2)
    SLRA_TN_CASE(3)
    SLRA_TN_CASE(4)
    SLRA_TN_CASE(5)
    SLRA_TN_CASE(6)
    SLRA_TN_CASE(7)
    default: return SLRA_ERR_UNSUPPORTED;
  }
#undef SLRA_TN_CASE
  SLRA_CHECK_LAUNCH(c);
  SLRA_TIMED(c, "gemm_reduce", streamk_sum_kernel<<<dim3(4, (unsigned)gx), 256, 0, c->stream>>>(part, (int)r, n, S, U,
                                                                                              G, alpha, Cm, ldc);)
  SLRA_CHECK_LAUNCH(c);
  return SLRA_OK;
}

}  // namespace slra_dev
