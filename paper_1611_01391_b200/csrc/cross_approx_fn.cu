// The FunctionOracle build of the C-A block kernel (oracle.hpp:43-54,
// cur.cpp:201-255): the config-5 log-kernel blocks K_ij = 0.5 log(dx^2 +
// dy^2) evaluated from their points wherever the algorithm reads an entry
// (the strips, the generator, the residual's full pass), so the blocks are
// never materialised. The same kernel source as cross_approx.cu with the
// entry reads behind an accessor; compiled as its own translation unit so
// that the dense kernel's code generation (register allocation of its long,
// latency-bound body) is untouched: templating the dense kernel on the same
// accessor measurably slowed its strip QR phase (437 K -> 520 K cycles per
// block). Entries are bit-identical to slra_gen_log_kernel_blocks', so the
// results are the dense path's exactly (tests/test_gpu_config5.py).
// (from cross_approx.cu) K-b / K-n: Cross-Approximation with maxvol pivoting and the CUR nucleus,
// CTA-resident. One thread block runs the whole of cross_approx
// (cur.cpp:201-255) for one problem whose strips fit in shared memory:
//   per loop:  R = A(I,:) -> J = select_rows_spanning(R^T, l)   (cur.cpp:215-224)
//              C = A(:,J) -> I = select_rows_spanning(C, k)      (cur.cpp:227-236)
//   then primitive_cur(A, I, J, r) (cur.cpp:137-162) and the residual
//   factors P = C T_r Sigma_r^-1 (m x r), Q = S_r^T R (r x n), so that
//   C U R = P Q and ||A - C U R||_F runs with inner dimension r.
// A grid of such blocks is the batched superfast-multipole workload
// (config 5; hss.cpp:47-55 pattern) with no inter-block communication.
#include <algorithm>

#include "dense_cta.cuh"
#include "blocked_qr.cuh"
#include "select_regs.cuh"

namespace slra_dev {
namespace logk {  // the FunctionOracle (log-kernel) build of the C-A block kernel

constexpr int kCT = 256;

struct CaParams {
  const double* A;
  int64_t lda, stride;
  int m, n, r, k, l, loops;
  double h;
  const int64_t* init_rows;  // nprob x k
  int64_t* I_out;            // nprob x k
  int64_t* J_out;            // nprob x l
  double* nucleus;           // nprob x (l*k), ld l
  int64_t* r_out;            // nprob
  int32_t* status;           // nprob
  int64_t* trace_rows;       // (2*loops) x k   (problem 0 only, nullable)
  int64_t* trace_cols;       // (2*loops) x l
  double* trace_vol;         // 2*loops
  double* P;                 // nprob x (m * rq), ld m   (nullable)
  double* Q;                 // nprob x (rq * n), ld rq
  int rq;                    // min(k, l)
  int mode;                  // 0 = cross_approx, 1 = primitive_cur only (I,J given in I_out/J_out)
  double* Tsig_out = nullptr;  // problem 0: T_r Sigma_r^-1 (l x r, ld l), nullable
  double* Sr_out = nullptr;    // problem 0: S_r (k x r, ld k), nullable
  double* pairs = nullptr;     // nprob x 2: fused (||B - CUR||^2, ||B||^2) (nullable; needs m, n % 8 == 0)
  // log-kernel blocks evaluated on the fly instead of A (FunctionOracle,
  // oracle.hpp:43-54): per-block points, nprob x m (px, py) and nprob x n (qx, qy)
  const double* px = nullptr;
  const double* py = nullptr;
  const double* qx = nullptr;
  const double* qy = nullptr;
};

// Entry access of the C-A block kernel (the reference's EntryOracle): a
// dense column-major block (DenseOracle), or the config-5 log kernel
// K_ij = 0.5 log(dx^2 + dy^2) evaluated where the algorithm reads an entry
// (FunctionOracle) — the strips, the generator and the residual's full pass
// — from the block's points, with the products and the sum rounded
// separately exactly as slra_gen_log_kernel_blocks materialises them (the
// two forms give bit-identical entries, hence identical selections).
struct DenseEntries {
  static constexpr bool kDense = true;
  const double* A;
  int64_t lda;
  __device__ __forceinline__ double get(int i, int j) const { return __ldg(A + i + (int64_t)j * lda); }
};
__device__ __noinline__ double log_kernel_entry(double pxi, double pyi, double qxj, double qyj) {
  const double dx = __dsub_rn(pxi, qxj);
  const double dy = __dsub_rn(pyi, qyj);
  return 0.5 * log(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
}
struct LogEntries {
  static constexpr bool kDense = false;
  const double* px;
  const double* py;
  const double* qx;
  const double* qy;
  __device__ __forceinline__ double get(int i, int j) const {
    return log_kernel_entry(__ldg(px + i), __ldg(py + i), __ldg(qx + j), __ldg(qy + j));
  }
};

// Shared-memory plan of one C-A block. Only S is strip-sized (mm x c): it
// holds the gathered strip, its basis Q and then B = Q G^-1 in place, and at
// the end the staged C / R^T strips of the residual factors. Everything else
// is c x c or mm-vectors, so a 256 x 256 block with k = l = 32 needs ~110 KB
// and two blocks share an SM (the kernel is latency bound: two resident CTAs
// hide each other's dependent chains).
struct CaSmem {
  double *S, *W, *R, *Gt, *V, *tau, *v, *nu, *nd, *rn, *sigma, *sgn, *rv, *Tm, *Sm, *volv;
  int *p2r, *r2p, *Icur, *Jcur, *perm, *order, *flag, *tmpidx;
  int64_t* ri;
  uint64_t* mbar;  // the bulk-copy (TMA) barrier of the column-strip staging
};

__host__ __device__ inline size_t ca_even(size_t d) { return (d + 1) & ~(size_t)1; }
__host__ __device__ inline size_t ca_max(size_t a, size_t b) { return a > b ? a : b; }

// every region starts 16-byte aligned (the selection reads v as double2)
__host__ __device__ inline size_t ca_smem_bytes(int m, int n, int k, int l) {
  const int mm = m > n ? m : n, c = k > l ? k : l;
  // S (mm c + c), W / Gt / V ((c+1) c each), tau / sigma / sgn (c), v (64),
  // nu / nd / rn (mm each), rv 40, volv 8 + slack 2c
  const int cw = c > 32 ? c : 32;  // W / Gt / V: also the selection's RMAX x r R (RMAX <= 32)
  const size_t nn = c <= 32 ? 5 * (size_t)c * c + c : (size_t)c * c;  // the nucleus' c x c buffers
  const size_t ns = ca_max((size_t)mm * ((c + 3) & ~3) + c, nn);
  size_t d = ca_even(ns) + 3 * ca_even((size_t)(cw + 1) * cw) + 3 * ca_even(c) + 64 +
             3 * ca_even(mm > 16 ? mm : 16) + 40 + 8 + ca_even(2 * (size_t)c);
  size_t i = 2 * (size_t)mm + 5 * (size_t)c + 8;
  return d * 8 + 34 * 8 + i * 4 + 64;
}

__device__ CaSmem ca_carve(char* base, int m, int n, int k, int l) {
  const int mm = m > n ? m : n, c = k > l ? k : l;
  CaSmem s;
  double* d = reinterpret_cast<double*>(base);
  // the strip; the fused residual's Q fragments (n x 4 ceil(r/4)); the
  // preconditioned nucleus' U_w, J_w, left / right vectors and rotations (5 c x c)
  s.S = d; d += ca_even(ca_max((size_t)mm * ((c + 3) & ~3) + c, c <= 32 ? 5 * (size_t)c * c + c : (size_t)c * c));
  const int cw = c > 32 ? c : 32;
  s.W = d; d += ca_even((size_t)(cw + 1) * cw);  // the nucleus' Jacobi operand (ld p | 1, p <= c)
  s.R = nullptr;
  s.Gt = d; d += ca_even((size_t)(cw + 1) * cw);  // maxvol QR (ld rq | 1) / the selection's R (ld RMAX)
  s.V = d; d += ca_even((size_t)(cw + 1) * cw);  // room for ld = q | 1
  // the nucleus factors T_r Sigma_r^-1 and S_r are written after
  // cta_svd_finish, when the Jacobi operands V and W are dead
  s.Tm = s.V;
  s.Sm = s.W;
  s.tau = d; d += ca_even(c);
  s.v = d; d += 64;  // the selection's reflector: RMAX entries
  s.sigma = d; d += ca_even(c);
  s.sgn = d; d += ca_even(c);
  const int mv = mm > 16 ? mm : 16;  // nu doubles as the selection's argmax slots
  s.nu = d; d += ca_even(mv);
  s.nd = d; d += ca_even(mv);
  s.rn = d; d += ca_even(mv);
  s.rv = d; d += 40;
  s.volv = d; d += 8;
  d += ca_even(2 * (size_t)c);  // slack
  s.ri = reinterpret_cast<int64_t*>(d);
  s.mbar = reinterpret_cast<uint64_t*>(s.ri + 33);
  int* ip = reinterpret_cast<int*>(s.ri + 34);
  s.p2r = ip; ip += mm;
  s.r2p = ip; ip += mm;
  s.Icur = ip; ip += c;
  s.Jcur = ip; ip += c;
  s.perm = ip; ip += c;
  s.order = ip; ip += c;
  s.tmpidx = ip; ip += c;
  s.flag = ip;
  return s;
}

// ---- TMA bulk copies (cp.async.bulk) for the contiguous column strips
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
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

// S (len x nidx, ld len) <- the strip A(idx, :)^T (rows_strip) or A(:, idx):
// a thread per strip row, eight independent global loads in flight before
// the shared-memory stores (no per-element integer division)
template <int NT, class E>
__device__ void stage_strip(double* S, const E& ent, bool rows_strip, const int* idx, int nidx, int len,
                            uint64_t* mbar = nullptr, unsigned* phase = nullptr) {
  if constexpr (!E::kDense) {
    // evaluated entries: a thread per strip row, the point of the row once
    for (int i = threadIdx.x; i < len; i += NT)
      for (int t = 0; t < nidx; ++t) S[i + t * len] = rows_strip ? ent.get(idx[t], i) : ent.get(i, idx[t]);
    return;
  } else {
  const double* A = ent.A;
  const int64_t lda = ent.lda;
  if (!rows_strip && mbar && nidx <= 32 && (len & 1) == 0 && (lda & 1) == 0 && ((uintptr_t)A & 15) == 0) {
    // column strip: nidx contiguous columns of len doubles -> one TMA bulk
    // copy each (warp 0's lanes issue them), completion on the mbarrier.
    // The callers' block barrier precedes this; the proxy fence orders the
    // earlier generic accesses to S before the async-proxy writes.
    if (threadIdx.x < 32) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (threadIdx.x == 0) mbar_arrive_expect_tx(mbar, (unsigned)(nidx * len * 8));
      __syncwarp();
      if (threadIdx.x < nidx)
        bulk_g2s(S + threadIdx.x * len, A + (int64_t)idx[threadIdx.x] * lda, (unsigned)(len * 8), mbar);
    }
    mbar_wait(mbar, *phase);
    *phase ^= 1u;
    return;
  }
  for (int i = threadIdx.x; i < len; i += NT) {
    for (int t0 = 0; t0 < nidx; t0 += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int t = t0 + u < nidx ? t0 + u : nidx - 1;
        v[u] = rows_strip ? __ldg(A + idx[t] + (int64_t)i * lda) : __ldg(A + i + (int64_t)idx[t] * lda);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (t0 + u < nidx) S[i + (t0 + u) * len] = v[u];
    }
  }
  }
}

// select_rows_spanning(strip, count, h) where strip (len x nidx) is gathered
// from A: rows_strip -> strip = A(idx_in, :)^T (len = n), else A(:, idx_in).
template <int NT, int CMAX, class E>
__device__ int select_strip(CaSmem& s, const E& ent, bool rows_strip, const int* idx_in, int nidx, int len, int count,
                            double h, int* idx_out, double* vol_out, unsigned* phase = nullptr) {
  const int tid = threadIdx.x;
  // gather (each element of the strip is an entry read of the oracle)
  // 2-D loops (no integer division per element), unrolled so that several
  // independent global loads are in flight before the shared-memory stores
  stage_strip<NT>(s.S, ent, rows_strip, idx_in, nidx, len, phase ? s.mbar : nullptr, phase);
  __syncthreads();
  SLRA_PROF(1);
  // ONE len x nidx array carries the strip, its basis Q (in place) and then
  // B = Q G^-1 (in place): the pivot order is taken with the working copy in
  // registers, and the volume |det Q[idx, :]| is tracked through the swaps.
  // The pivot phase's reflectors are those of maxvol round 0's ColPivQR(G^T)
  // (G = Q(I, :)), so round 0 continues from them instead of refactorising.
  if (nidx <= 32 && NT == 256) {
    // blocked Householder (8-column panels, DMMA trailing updates and
    // block-reflector Q formation); scratch: the W / Gt / V regions
    cta_blocked_qr_q<NT>(s.S, len, len, nidx, s.tau, s.W, s.rv);
  } else {
    cta_thin_qr_inplace<NT, CMAX>(s.S, len, len, nidx, s.tau, s.rv);
  }
  SLRA_PROF(3);
  const int rq = count < nidx ? count : nidx;
  if (count > rq) {  // the padding branch needs the basis row norms (cur.cpp:125-134)
    for (int i = tid; i < len; i += NT) {
      double acc = 0.0;
      for (int j = 0; j < nidx; ++j) acc += s.S[i + j * len] * s.S[i + j * len];
      s.rn[i] = sqrt(acc);
    }
  }
  double vol = 0.0;
  if (rq <= 32) {
    // pivoted-QR initialisation, maxvol round 0 and the swaps with the basis
    // rows in registers (select_regs.cuh)
    const SelScratch ss{s.nu, s.p2r, s.v, s.Gt, rq <= 16 ? 16 : 32, s.sigma, s.rv, s.tau, s.flag};
    const int st = rq <= 16 ? cta_select_regs<NT, 16>(s.S, len, len, rq, h, 4 * rq, s.tmpidx, ss)
                            : cta_select_regs<NT, 32>(s.S, len, len, rq, h, 4 * rq, s.tmpidx, ss);
    if (st != SLRA_OK) return st;
    vol = s.tau[1];
  } else {
    if constexpr (CMAX > 32)
      cta_colpiv_init_regs<NT, 64>(s.S, len, len, rq, s.nu, s.nd, s.p2r, s.r2p, s.v, s.tau, s.rv, s.ri, s.tmpidx,
                                   s.S, s.Gt, rq | 1, s.sigma);
    __syncthreads();
    // Gt with an odd leading dimension: warp_colpiv_qr gives each lane a
    // column, and ld = rq (even) put all 32 lanes on the same shared bank
    const int st = cta_maxvol_swaps<NT>(s.S, len, len, rq, h, 4 * rq, s.tmpidx, s.S, len, s.Gt, rq | 1, s.perm,
                                        s.tau, s.nu, s.nd, s.rv, s.ri, s.flag, s.volv, s.r2p, s.sigma);
    if (st != SLRA_OK) return st;
    __syncthreads();
    vol = *s.volv;
  }
  __syncthreads();
  for (int t = tid; t < rq; t += NT) idx_out[t] = s.tmpidx[t];
  __syncthreads();
  if (count > rq) {
    // pad with the largest remaining rows of the basis (cur.cpp:125-134);
    // equal norms: lower index first.
    for (int t = rq; t < count; ++t) {
      ArgMax a{-1.0, INT64_MAX};
      for (int i = tid; i < len; i += NT) {
        bool used = false;
        for (int u = 0; u < t; ++u) used |= (idx_out[u] == i);
        if (!used) a = argmax_merge(a, ArgMax{s.rn[i], i});
      }
      a = block_argmax<NT>(a, s.rv, s.ri);
      if (tid == 0) idx_out[t] = (int)a.i;
      __syncthreads();
    }
  }
  // volume proxy |det Q[idx,:]| (cur.cpp:192-197), only when square
  if (vol_out) {
    // |det Q[idx, :]| = the swap loop's tracked volume (round-0 QR of G times
    // the pivot magnitudes of the swaps)
    if (tid == 0) *vol_out = count == nidx ? vol : 0.0;
    __syncthreads();
  }
  return SLRA_OK;
}

// primitive_cur nucleus from G = A(I, J) (k x l). Writes r, nucleus (l x k)
// and the factors Tm = T_r Sigma_r^-1 (l x r, ld l) and Sm = S_r (k x r, ld k)
// into smem. Returns status.
template <int NT, int CMAX, class E>
__device__ int cta_nucleus(CaSmem& s, const E& ent, const int* I, int k, const int* J, int l, int r_req, int* r_out) {
  const int tid = threadIdx.x;
  const bool tall = k > l;  // square generators take the transposed (faster) path
  const int p = tall ? k : l, q = tall ? l : k;
  const double* Sl;  // left vectors of G (k x q)
  const double* Tr;  // right vectors of G (l x q)
  int ldsl, ldtr;
  if (k == l && k <= 32) {
    // Square generator, QR-preconditioned one-sided Jacobi (Drmac-Veselic):
    // G Pi = Q R (column-pivoted Householder, Eigen's rules), then Jacobi on
    // the rows of R (R^T Jv = U_w Sigma): the rows of R are graded, so the
    // sweeps settle in about half as many rounds as on G itself. Then
    // G = (Q Jv) Sigma (Pi U_w)^T: left vectors Q Jv (the reflectors applied
    // to Jv), right vectors Pi U_w (a row permutation).
    const int n = k, ld = n | 1;
    for (int e = tid; e < n * n; e += NT) {
      const int a = e % n, b = e / n;
      s.W[a + b * ld] = ent.get(I[a], J[b]);
    }
    __syncthreads();
    SLRA_PROF(9);
    for (int e = tid; e < n * ld; e += NT) s.Gt[e] = 0.0;  // R^T: zeros above its diagonal
    __syncthreads();
    // G Pi = Q R by one warp (columns in registers): R^T into Gt, the
    // reflectors into V (the G copy in W is not needed afterwards)
    if (tid < 32) warp_colpiv_regs(s.W, ld, n, s.Gt, ld, s.V, ld, s.tau, s.perm, s.v);
    __syncthreads();
    // Rows of R below 1e-15 of the largest row norm are dropped: they move
    // every singular value by less than 1e-15 sqrt(n) sigma_1 — below the
    // Jacobi's own absolute accuracy on the small ones, and nine orders under
    // the 1e-10 rank cut — and the Jacobi then runs on nr <= n columns.
    if (tid < 32) {
      const int lane = tid;
      double rn = 0.0;
      if (lane < n)
        for (int j = lane; j < n; ++j) rn = fma(s.Gt[j + lane * ld], s.Gt[j + lane * ld], rn);
      const double mx = __shfl_sync(0xffffffffu, rn, 0);  // row 0 carries the largest pivot
      double rmax = rn;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
      (void)mx;
      const unsigned keep = __ballot_sync(0xffffffffu, lane < n && rn > 1e-30 * rmax);
      if (lane == 0) s.flag[4] = keep ? 32 - __clz(keep) : 1;
    }
    __syncthreads();
    const int nr = s.flag[4];
    // QLP: the second, unpivoted QR R_top^T = Q1 R1 (one warp; V1 over Gt,
    // tau1 in rv), then the Jacobi on W = R1^T (nr x nr): on the twice
    // QR-reduced factor the sweeps settle in ~4 instead of ~6.5
    // (Drmac-Veselic), on columns of length nr instead of n.
    double* Jrot = s.S + 3 * n * n;  // nr x nr rotations (ld ld), consumed by svd_finish
    for (int e = tid; e < n * ld; e += NT) s.W[e] = 0.0;
    __syncthreads();
    if (tid < 32) warp_house_regs(s.Gt, ld, n, nr, s.W, ld, s.rv, s.v);
    __syncthreads();
    cta_jacobi<NT, CMAX>(s.W, ld, nr, nr, Jrot, ld, s.flag, 1e-10 / sqrt((double)nr));
    SLRA_PROF(10);
#ifdef SLRA_PHASE_PROF
    if (tid == 0) {
      atomicAdd(&g_phase_cycles[20], (unsigned long long)s.flag[2]);
      atomicAdd(&g_phase_cycles[21], (unsigned long long)nr);
    }
#endif
    // R1^T Jw = Uw Sigma  =>  G = (Q [Uw; 0]) Sigma (Pi Q1 [Jw; 0])^T
    double* Uw = s.S;               // nr x nr, ld n
    double* Jw = s.S + n * n;       // nr x nr, ld n
    double* Lv = s.S + 2 * n * n;   // left vectors of G: Q [Uw; 0]  (n x nr, ld n)
    double* Rv = s.S + 3 * n * n;   // right vectors of G: Pi Q1 [Jw; 0]
    cta_svd_finish<NT>(s.W, ld, nr, nr, Jrot, ld, s.sigma, s.order, Uw, n, Jw, n, s.sgn);
    for (int i = nr + tid; i < n; i += NT) s.sigma[i] = 0.0;
    {
      const int lane = tid & 31, warp = tid >> 5;
      // a warp per column, a lane per row: the reflectors applied backwards
      for (int j = warp; j < 2 * nr; j += NT / 32) {
        const bool left = j < nr;
        const int jj = left ? j : j - nr;
        double y = lane < nr ? (left ? Uw : Jw)[lane + jj * n] : 0.0;
        if (left) {
          for (int kk = n - 1; kk >= 0; --kk) {  // Q = H_0 ... H_{n-1} (G Pi = Q R)
            const double v = lane < n ? s.V[lane + kk * ld] : 0.0;  // unit head, zeros above
            const double w = warp_sum(v * y);
            y = fma(-s.tau[kk] * w, v, y);
          }
          if (lane < n) Lv[lane + jj * n] = y;
        } else {
          for (int kk = nr - 1; kk >= 0; --kk) {  // Q1 = H1_0 ... H1_{nr-1}
            const double v = lane < n ? s.Gt[lane + kk * ld] : 0.0;
            const double w = warp_sum(v * y);
            y = fma(-s.rv[kk] * w, v, y);
          }
          if (lane < n) Rv[s.perm[lane] + jj * n] = y;  // (Jrot, under Rv, is consumed)
        }
      }
    }
    __syncthreads();
    // the sign rule on the left vectors of G (linalg.cpp:87-96)
    for (int t = tid >> 5; t < nr; t += NT / 32) {
      const int lane = tid & 31;
      ArgMax a{-1.0, INT64_MAX};
      for (int i = lane; i < n; i += 32) a = argmax_merge(a, ArgMax{fabs(Lv[i + t * n]), i});
      a = warp_argmax(a);
      const double f = (Lv[a.i + t * n] < 0.0) ? -1.0 : 1.0;
      __syncwarp();
      for (int i = lane; i < n; i += 32) {
        Lv[i + t * n] *= f;
        Rv[i + t * n] *= f;
      }
    }
    __syncthreads();
    Sl = Lv;
    ldsl = n;
    Tr = Rv;
    ldtr = n;
  } else {
    // W := G (tall) or G^T (wide), p x q, ld p
    for (int e = tid; e < k * l; e += NT) {
      const int a = e % k, b = e / k;
      const double g = ent.get(I[a], J[b]);
      if (tall) s.W[a + b * (p | 1)] = g;
      else s.W[b + a * (p | 1)] = g;
    }
    __syncthreads();
    SLRA_PROF(9);
    // Only sigma_i > 1e-10 sigma_1 enter the nucleus (pinv cut, linalg.cpp:111-121;
    // rank checks cur.cpp:156-157): columns below 1e-10/sqrt(q) of the largest
    // column norm jointly carry less than that, so pairs of two such columns
    // are not rotated (the noise directions of rank-deficient generators, as in
    // configs 3 and 5, otherwise keep the sweeps going to the cap).
    cta_jacobi<NT, CMAX>(s.W, p | 1, p, q, s.V, q | 1, s.flag, 1e-10 / sqrt((double)q));
    SLRA_PROF(10);
    // finish into S (p x q, ld p) and Gt (q x q, ld q): for tall G the left
    // vectors are in S; for wide G (SVD of G^T) they are the rows of V.
    cta_svd_finish<NT>(s.W, p | 1, p, q, s.V, q | 1, s.sigma, s.order, s.S, p, s.Gt, q, s.sgn);
    if (!tall) {
      // G^T = S' Sigma V'^T -> G = V' Sigma S'^T: left vectors of G = V'
      // (columns of Gt), right = S'. Re-apply the sign rule on the left ones.
      for (int t = threadIdx.x >> 5; t < q; t += NT / 32) {
        const int lane = threadIdx.x & 31;
        ArgMax a{-1.0, INT64_MAX};
        for (int i = lane; i < q; i += 32) a = argmax_merge(a, ArgMax{fabs(s.Gt[i + t * q]), i});
        a = warp_argmax(a);
        const double f = (s.Gt[a.i + t * q] < 0.0) ? -1.0 : 1.0;
        __syncwarp();
        for (int i = lane; i < q; i += 32) s.Gt[i + t * q] *= f;
        for (int i = lane; i < p; i += 32) s.S[i + t * p] *= f;
      }
      __syncthreads();
    }
    Sl = tall ? s.S : s.Gt;
    ldsl = tall ? p : q;
    Tr = tall ? s.Gt : s.S;
    ldtr = tall ? q : p;
  }
  const double s0 = s.sigma[0];
  int r = r_req;
  if (r <= 0) {
    r = 0;
    for (int i = 0; i < q; ++i) r += (s.sigma[i] > 1e-10 * s0) ? 1 : 0;
    if (r == 0) return SLRA_ERR_GENERATOR_RANK_FAILURE;
  } else {
    if (r > q) return SLRA_ERR_INVALID_ARGUMENT;
    if (s0 <= 0.0 || s.sigma[r - 1] <= 1e-10 * s0) return SLRA_ERR_GENERATOR_RANK_FAILURE;
  }
  *r_out = r;
  for (int e = tid; e < l * r; e += NT) {
    const int a = e % l, j = e / l;
    s.Tm[a + j * l] = Tr[a + j * ldtr] / s.sigma[j];
  }
  for (int e = tid; e < k * r; e += NT) {
    const int a = e % k, j = e / k;
    s.Sm[a + j * k] = Sl[a + j * ldsl];
  }
  __syncthreads();
  return SLRA_OK;
}

// ||B - P Q||_F^2 and ||B||_F^2 of one block inside the C-A kernel (the
// residual of cur_evaluate, cur.cpp:76-82, with the nucleus factored:
// C U R = (C T_r Sigma_r^-1)(S_r^T R) = P Q, inner dimension r). P (m x r) is
// computed a row per thread and moved into DMMA A-fragments by shuffles
// (warp w owns rows 32w..32w+31, exactly the rows its threads computed);
// Q (r x n) a column per thread, stored in shared memory in the B-fragment
// order ((n-tile, k-step) -> 32 consecutive doubles, one per lane: conflict
// free). The block is then streamed once from global memory in C-fragment
// order (8 rows x 4 column pairs per load: full sectors) and E = B - P Q is
// formed by DMMA 8x8x4 with -P as the A operand. KS = k-steps (r <= 4 KS),
// MTP = m-tiles per pass (a warp's 4 m-tiles in 4 / MTP passes).
template <int NT, int KS, int MTP, class E>
__device__ void fused_block_residual(const E& ent, int m, int n, const int* I, int k, const int* J, int l,
                                     const double* Tm, const double* Sm, int r, double* QS, double* red,
                                     double* out_pair) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int RP = 4 * KS;
  const int ksn = (r + 3) >> 2;  // k-steps in use (QS holds n x 4 ksn doubles)
  constexpr int NB = KS <= 4 ? 16 : 8;  // global loads in flight per thread (register budget)
  // Q first, into shared memory, then P in registers: q and p never live together
  // Q(:, col) = Sm^T A(I, col), col = tid, into the B-fragment layout
  if (tid < n) {
    double q[RP];
#pragma unroll
    for (int j = 0; j < RP; ++j) q[j] = 0.0;
    for (int t0 = 0; t0 < k; t0 += NB) {
      double a[NB];
#pragma unroll
      for (int u = 0; u < NB; ++u) a[u] = ent.get(I[t0 + u < k ? t0 + u : k - 1], tid);  // Q = Sm^T A(I, :)
#pragma unroll
      for (int u = 0; u < NB; ++u)
        if (t0 + u < k) {
#pragma unroll
          for (int j = 0; j < RP; ++j)
            if (j < r) q[j] = fma(Sm[t0 + u + j * k], a[u], q[j]);
        }
    }
    const int nt = tid >> 3, g = tid & 7;
#pragma unroll
    for (int j = 0; j < RP; ++j)
      if ((j >> 2) < ksn) QS[((nt * ksn) + (j >> 2)) * 32 + g * 4 + (j & 3)] = q[j];
  }
#ifdef SLRA_PHASE_PROF
  __syncthreads();
  SLRA_PROF(14);
#endif
  // P(i, :) = A(i, J) Tm, row i = tid (zero for j >= r)
  double p[RP];
#pragma unroll
  for (int j = 0; j < RP; ++j) p[j] = 0.0;
  if (tid < m) {
    for (int t0 = 0; t0 < l; t0 += NB) {
      double c[NB];
#pragma unroll
      for (int u = 0; u < NB; ++u) c[u] = ent.get(tid, J[t0 + u < l ? t0 + u : l - 1]);
#pragma unroll
      for (int u = 0; u < NB; ++u)
        if (t0 + u < l) {
#pragma unroll
          for (int j = 0; j < RP; ++j)
            if (j < r) p[j] = fma(c[u], Tm[t0 + u + j * l], p[j]);
        }
    }
  }
  __syncthreads();
  SLRA_PROF(12);
  const int g = lane >> 2, q4 = lane & 3;
  double rs = 0.0, ns = 0.0;
#pragma unroll
  for (int pass = 0; pass < 4 / MTP; ++pass) {
    // A-fragments of -P for this pass' m-tiles: lane (g, q4) of m-tile mt
    // needs P(32 warp + 8 mt + g, 4 ks + q4), held by lane 8 mt + g as p[4 ks + q4]
    double af[MTP][KS];
#pragma unroll
    for (int u = 0; u < MTP; ++u) {
      const int src = 8 * (pass * MTP + u) + g;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        double v = 0.0;
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          const double t = __shfl_sync(0xffffffffu, p[4 * ks + qq], src);
          if (qq == q4) v = t;
        }
        af[u][ks] = -v;
      }
    }
    const int row0 = 32 * warp + 8 * pass * MTP;
    if (row0 < m) {
      // NTU n-tiles per iteration, all their loads issued before any use
      // (the block may come from DRAM: one round trip per NTU tiles)
      constexpr int NTU = 2;
      const int ntiles = n >> 3;
      for (int nt0 = 0; nt0 < ntiles; nt0 += NTU) {
        double c[NTU][MTP][2];
#pragma unroll
        for (int q = 0; q < NTU; ++q) {
          const int col = 8 * (nt0 + q) + 2 * q4;
#pragma unroll
          for (int u = 0; u < MTP; ++u) {
            const int row = row0 + 8 * u + g;
            const bool ok = row < m && nt0 + q < ntiles;
            if constexpr (E::kDense) {
              c[q][u][0] = load_sel(ent.A, row + (int64_t)col * ent.lda, ok);
              c[q][u][1] = load_sel(ent.A, row + (int64_t)(col + 1) * ent.lda, ok);
            } else {  // evaluated at a clamped index, then the select
              const double e0 = ent.get(ok ? row : 0, ok ? col : 0), e1 = ent.get(ok ? row : 0, ok ? col + 1 : 0);
              c[q][u][0] = ok ? e0 : 0.0;
              c[q][u][1] = ok ? e1 : 0.0;
            }
          }
        }
#pragma unroll
        for (int q = 0; q < NTU; ++q) {
          if (nt0 + q < ntiles) {
#pragma unroll
            for (int u = 0; u < MTP; ++u) {
              ns = fma(c[q][u][0], c[q][u][0], ns);
              ns = fma(c[q][u][1], c[q][u][1], ns);
            }
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
              if (ks < ksn) {
                const double bf = QS[((nt0 + q) * ksn + ks) * 32 + lane];
#pragma unroll
                for (int u = 0; u < MTP; ++u) dmma_8x8x4(c[q][u][0], c[q][u][1], af[u][ks], bf);
              }
            }
#pragma unroll
            for (int u = 0; u < MTP; ++u) {
              rs = fma(c[q][u][0], c[q][u][0], rs);
              rs = fma(c[q][u][1], c[q][u][1], rs);
            }
          }
        }
      }
    }
  }
  rs = warp_sum(rs);
  ns = warp_sum(ns);
  if (lane == 0) {
    red[2 * warp] = rs;
    red[2 * warp + 1] = ns;
  }
  __syncthreads();
  if (tid == 0) {
    double a = 0.0, b2 = 0.0;
    for (int w = 0; w < NT / 32; ++w) {
      a += red[2 * w];
      b2 += red[2 * w + 1];
    }
    out_pair[0] = a;
    out_pair[1] = b2;
  }
  SLRA_PROF(13);
}

// two resident CTAs per SM (<= 128 registers): the block is latency bound
// CMAX = 32 (k, l <= 32): register variants sized for 32 columns so that
// two CTAs fit an SM; CMAX = 64: one CTA per SM
template <int CMAX, class E>
__global__ void __launch_bounds__(kCT, CMAX <= 32 ? 2 : 1) ca_block_kernel(CaParams P) {
  extern __shared__ __align__(16) char smem_raw[];
  const int b = blockIdx.x;
  const int tid = threadIdx.x;
  CaSmem s = ca_carve(smem_raw, P.m, P.n, P.k, P.l);
  SLRA_PROF(-1);
  const double* A = E::kDense ? P.A + (int64_t)b * P.stride : nullptr;
  E ent;
  if constexpr (E::kDense) ent = E{A, P.lda};
  else ent = E{P.px + (int64_t)b * P.m, P.py + (int64_t)b * P.m, P.qx + (int64_t)b * P.n, P.qy + (int64_t)b * P.n};
  int status = SLRA_OK;
  if (P.mode == 0) {
#ifndef SLRA_C5_L2
#define SLRA_C5_L2 2
#endif
    if (tid == 0) {
      mbar_init(s.mbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const bool bulk = E::kDense && (P.m & 1) == 0 && (P.lda & 1) == 0 && ((uintptr_t)A & 15) == 0;
    if (E::kDense && P.pairs && SLRA_C5_L2 > 0) {
      // the block is read by every half-sweep's strip gather and by the fused
      // residual: pull it into L2 once before the first gather — one TMA bulk
      // prefetch per column (evict-last), else full-line prefetches
      if (bulk) {
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        for (int c = tid; c < P.n; c += kCT) {
          if (SLRA_C5_L2 == 2)
            asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(A + (int64_t)c * P.lda),
                         "r"(P.m * 8), "l"(pol)
                         : "memory");
          else
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A + (int64_t)c * P.lda), "r"(P.m * 8)
                         : "memory");
        }
      } else {
        for (int j = tid; j < P.n * ((P.m + 15) / 16); j += kCT) {
          const int c = j / ((P.m + 15) / 16), i = 16 * (j % ((P.m + 15) / 16));
          if (SLRA_C5_L2 == 2) asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(A + i + (int64_t)c * P.lda));
          else asm volatile("prefetch.global.L2 [%0];" ::"l"(A + i + (int64_t)c * P.lda));
        }
      }
    }
    for (int t = tid; t < P.k; t += kCT) s.Icur[t] = (int)P.init_rows[(int64_t)b * P.k + t];
    __syncthreads();
    unsigned phase = 0;  // parity of the column-strip mbarrier
    SLRA_PROF(0);
    for (int loop = 0; loop < P.loops && status == SLRA_OK; ++loop) {
      double* vol = (b == 0 && P.trace_vol) ? P.trace_vol + 2 * loop : nullptr;
      status = select_strip<kCT, CMAX>(s, ent, true, s.Icur, P.k, P.n, P.l, P.h, s.Jcur, vol);
      if (status != SLRA_OK) break;
      if (b == 0 && P.trace_rows) {
        for (int t = tid; t < P.k; t += kCT) P.trace_rows[(int64_t)(2 * loop) * P.k + t] = s.Icur[t];
        for (int t = tid; t < P.l; t += kCT) P.trace_cols[(int64_t)(2 * loop) * P.l + t] = s.Jcur[t];
      }
      vol = (b == 0 && P.trace_vol) ? P.trace_vol + 2 * loop + 1 : nullptr;
      status = select_strip<kCT, CMAX>(s, ent, false, s.Jcur, P.l, P.m, P.k, P.h, s.Icur, vol,
                                       bulk ? &phase : nullptr);
      if (status != SLRA_OK) break;
      if (b == 0 && P.trace_rows) {
        for (int t = tid; t < P.k; t += kCT) P.trace_rows[(int64_t)(2 * loop + 1) * P.k + t] = s.Icur[t];
        for (int t = tid; t < P.l; t += kCT) P.trace_cols[(int64_t)(2 * loop + 1) * P.l + t] = s.Jcur[t];
      }
      __syncthreads();
    }
  } else {
    for (int t = tid; t < P.k; t += kCT) s.Icur[t] = (int)P.I_out[(int64_t)b * P.k + t];
    for (int t = tid; t < P.l; t += kCT) s.Jcur[t] = (int)P.J_out[(int64_t)b * P.l + t];
    __syncthreads();
  }
  int r = 0;
  if (status == SLRA_OK) status = cta_nucleus<kCT, CMAX>(s, ent, s.Icur, P.k, s.Jcur, P.l, P.r, &r);
  if (tid == 0) {
    P.status[b] = status;
    P.r_out[b] = status == SLRA_OK ? r : 0;
  }
  if (P.mode == 0) {
    for (int t = tid; t < P.k; t += kCT) P.I_out[(int64_t)b * P.k + t] = s.Icur[t];
    for (int t = tid; t < P.l; t += kCT) P.J_out[(int64_t)b * P.l + t] = s.Jcur[t];
  }
  if (status != SLRA_OK) {
    if (P.pairs) {  // a failed block's residual is ||B|| (r = 0)
      __syncthreads();
      fused_block_residual<kCT, 4, 4>(ent, P.m, P.n, s.Icur, P.k, s.Jcur, P.l, s.Tm, s.Sm, 0, s.S, s.rv,
                                      P.pairs + 2 * (int64_t)b);
      return;
    }
    // zero the residual factors so a batched residual of a failed block is ||B||
    if (P.P) {
      for (int64_t e = tid; e < (int64_t)P.m * P.rq; e += kCT) P.P[(int64_t)b * P.m * P.rq + e] = 0.0;
      for (int64_t e = tid; e < (int64_t)P.rq * P.n; e += kCT) P.Q[(int64_t)b * P.rq * P.n + e] = 0.0;
    }
    return;
  }
  if (b == 0 && P.Tsig_out) {
    for (int e = tid; e < P.l * r; e += kCT) P.Tsig_out[e] = s.Tm[e];
    for (int e = tid; e < P.k * r; e += kCT) P.Sr_out[e] = s.Sm[e];
  }
  // nucleus U = Tm Sm^T (l x k)
  double* U = P.nucleus + (int64_t)b * P.l * P.k;
  for (int e = tid; e < P.l * P.k; e += kCT) {
    const int a = e % P.l, c = e / P.l;
    double acc = 0.0;
    for (int j = 0; j < r; ++j) acc += s.Tm[a + j * P.l] * s.Sm[c + j * P.k];
    U[a + (int64_t)c * P.l] = acc;
  }
  if (P.pairs) {
    __syncthreads();
    SLRA_PROF(11);
    if (E::kDense && SLRA_C5_L2 == 2) {
      // the block's last pass follows: its lines go back to normal priority
      // as they are consumed (the next blocks' prefetches may evict them)
      for (int j = tid; j < P.n * ((P.m + 15) / 16); j += kCT) {
        const int c = j / ((P.m + 15) / 16), i = 16 * (j % ((P.m + 15) / 16));
        asm volatile("applypriority.global.L2::evict_normal [%0], 128;" ::"l"(A + i + (int64_t)c * P.lda));
      }
    }
    if (r <= 16) fused_block_residual<kCT, 4, 4>(ent, P.m, P.n, s.Icur, P.k, s.Jcur, P.l, s.Tm, s.Sm, r, s.S,
                                                 s.rv, P.pairs + 2 * (int64_t)b);
    else fused_block_residual<kCT, 8, 2>(ent, P.m, P.n, s.Icur, P.k, s.Jcur, P.l, s.Tm, s.Sm, r, s.S, s.rv,
                                         P.pairs + 2 * (int64_t)b);
    return;
  }
  if (P.P) {
    // P = A(:,J) Tm (m x rq, zero beyond r), Q = Sm^T A(I,:) (rq x n). The
    // strips are staged in shared memory one after the other (S is free
    // after the nucleus): C = A(:,J) (m x l, coalesced columns), then
    // R^T = A(I,:)^T (n x k); a thread per row of P / column of Q, with r
    // independent FMA chains each.
    double* Pb = P.P + (int64_t)b * P.m * P.rq;
    double* Qb = P.Q + (int64_t)b * P.rq * P.n;
    __syncthreads();
    stage_strip<kCT>(s.S, ent, false, s.Jcur, P.l, P.m);
    __syncthreads();
    // accumulators in chunks of kCH outputs (registers stay within the
    // two-CTAs-per-SM budget); each chunk re-reads its strip from smem
    constexpr int kCH = 16;
    for (int i = tid; i < P.m; i += kCT) {
      for (int j0 = 0; j0 < P.rq; j0 += kCH) {
        double acc[kCH];
#pragma unroll
        for (int j = 0; j < kCH; ++j) acc[j] = 0.0;
        for (int t = 0; t < P.l; ++t) {
          const double cv = s.S[i + t * P.m];
#pragma unroll
          for (int j = 0; j < kCH; ++j)
            if (j0 + j < r) acc[j] = fma(cv, s.Tm[t + (j0 + j) * P.l], acc[j]);
        }
#pragma unroll
        for (int j = 0; j < kCH; ++j)
          if (j0 + j < P.rq) Pb[i + (int64_t)(j0 + j) * P.m] = acc[j];  // zero beyond r
      }
    }
    __syncthreads();  // every row of P is done with C: stage R^T over it
    stage_strip<kCT>(s.S, ent, true, s.Icur, P.k, P.n);
    __syncthreads();
    for (int c = tid; c < P.n; c += kCT) {
      for (int j0 = 0; j0 < P.rq; j0 += kCH) {
        double acc[kCH];
#pragma unroll
        for (int j = 0; j < kCH; ++j) acc[j] = 0.0;
        for (int t = 0; t < P.k; ++t) {
          const double rv = s.S[c + t * P.n];
#pragma unroll
          for (int j = 0; j < kCH; ++j)
            if (j0 + j < r) acc[j] = fma(s.Sm[t + (j0 + j) * P.k], rv, acc[j]);
        }
#pragma unroll
        for (int j = 0; j < kCH; ++j)
          if (j0 + j < P.rq) Qb[j0 + j + (int64_t)c * P.rq] = acc[j];
      }
    }
  }
}

static bool ca_fits(int m, int n, int k, int l) {
  // the CTA-resident strip QR forms Q in registers for at most 256 rows
  // (cta_form_q); taller strips take the TSQR + grid-wide maxvol path
  return k >= 1 && l >= 1 && k <= 64 && l <= 64 && k <= m && l <= n && m <= 256 && n <= 256 &&
         ca_smem_bytes(m, n, k, l) <= 227 * 1024;
}

int launch_ca_block(Context* c, const CaParams& p, int nprob) {
#ifdef SLRA_ONE_CTA_PER_SM  // profiling experiment: occupancy one block per SM
  const size_t smem = 160 * 1024;
#else
  const size_t smem = ca_smem_bytes(p.m, p.n, p.k, p.l);
#endif
  if (!p.px || p.k > 32 || p.l > 32) return SLRA_ERR_UNSUPPORTED;
  SLRA_CUDA(cudaFuncSetAttribute(ca_block_kernel<32, LogEntries>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
  SLRA_TIMED(c, "cross_approx", (ca_block_kernel<32, LogEntries><<<nprob, kCT, smem, c->stream>>>(p));)
  SLRA_CHECK_LAUNCH(c);
  return SLRA_OK;
}


// Host-streamed batched C-A: per-chunk inputs cross the bus on a copy
// stream while the previous chunk is factorised and the one before it
// returns its results (two buffer sets). `in_doubles` = input doubles per
// block; upload(d_in, b0, nb, stream) copies chunk [b0, b0 + nb)'s inputs
// into d_in; run(d_in, nb, d_init, outputs...) launches its factorisation.
template <class Upload, class Run>
static int ca_batched_host_stream(slra_ctx ctx, int64_t nblocks, int64_t in_doubles, int64_t k, int64_t l,
                                  const int64_t* h_init, int64_t* h_I, int64_t* h_J, double* h_nucleus, int64_t* h_r,
                                  int32_t* h_status, double* h_resid_sq, double* h_norm_sq, Upload upload, Run run,
                                  int64_t max_chunk = INT64_MAX) {
  Context* cx = C(ctx);
  if (!cx->h2d) {
    SLRA_CUDA(cudaStreamCreateWithFlags(&cx->h2d, cudaStreamNonBlocking));
    SLRA_CUDA(cudaStreamCreateWithFlags(&cx->d2h, cudaStreamNonBlocking));
    for (auto& e : cx->ev) SLRA_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  // two chunk buffers of ~1 GiB of inputs each
  const int64_t blk = in_doubles * 8;
  const int64_t chunk =
      std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(nblocks, max_chunk), (int64_t(1) << 30) / blk));
  const int64_t outd = l * k + 2;  // nucleus + (resid_sq, norm_sq) per block
  const int64_t outi = k + l + 1;  // I, J, r per block
  const size_t per = (size_t)chunk * (in_doubles + outd + outi) + (size_t)chunk * k + (size_t)chunk;  // + init, status
  char* base = static_cast<char*>(arena(cx, 12, 2 * per * 8 + 1024));
  if (!base) return SLRA_ERR_CUDA;
  struct Buf {
    double *A, *U, *rs, *ns;
    int64_t *I, *J, *rr, *init;
    int32_t* st;
  } bf[2];
  for (int i = 0; i < 2; ++i) {
    double* d = reinterpret_cast<double*>(base + i * per * 8);
    bf[i].A = d; d += chunk * in_doubles;
    bf[i].U = d; d += chunk * l * k;
    bf[i].rs = d; d += chunk;
    bf[i].ns = d; d += chunk;
    int64_t* q = reinterpret_cast<int64_t*>(d);
    bf[i].I = q; q += chunk * k;
    bf[i].J = q; q += chunk * l;
    bf[i].rr = q; q += chunk;
    bf[i].init = q; q += chunk * k;
    bf[i].st = reinterpret_cast<int32_t*>(q);
  }
  cudaEvent_t* ev_h2d = cx->ev;      // chunk copied in
  cudaEvent_t* ev_comp = cx->ev + 2;  // chunk factorised (its input buffer is free)
  cudaEvent_t* ev_out = cx->ev + 4;   // chunk results copied out (its output buffers are free)
  const int64_t nch = (nblocks + chunk - 1) / chunk;
  for (int64_t c = 0; c < nch; ++c) {
    const int i = (int)(c & 1);
    const int64_t b0 = c * chunk, nb = std::min(chunk, nblocks - b0);
    if (c >= 2) SLRA_CUDA(cudaStreamWaitEvent(cx->h2d, ev_comp[i], 0));
    SLRA_TRY(upload(bf[i].A, b0, nb, chunk, cx->h2d));
    SLRA_CUDA(cudaMemcpyAsync(bf[i].init, h_init + b0 * k, (size_t)nb * k * 8, cudaMemcpyHostToDevice, cx->h2d));
    SLRA_CUDA(cudaEventRecord(ev_h2d[i], cx->h2d));
    SLRA_CUDA(cudaStreamWaitEvent(cx->stream, ev_h2d[i], 0));
    if (c >= 2) SLRA_CUDA(cudaStreamWaitEvent(cx->stream, ev_out[i], 0));
    SLRA_TRY(run(bf[i].A, nb, chunk, bf[i].init, bf[i].I, bf[i].J, bf[i].U, bf[i].rr, bf[i].st, bf[i].rs, bf[i].ns));
    SLRA_CUDA(cudaEventRecord(ev_comp[i], cx->stream));
    SLRA_CUDA(cudaStreamWaitEvent(cx->d2h, ev_comp[i], 0));
    if (h_I) SLRA_CUDA(cudaMemcpyAsync(h_I + b0 * k, bf[i].I, (size_t)nb * k * 8, cudaMemcpyDeviceToHost, cx->d2h));
    if (h_J) SLRA_CUDA(cudaMemcpyAsync(h_J + b0 * l, bf[i].J, (size_t)nb * l * 8, cudaMemcpyDeviceToHost, cx->d2h));
    if (h_nucleus)
      SLRA_CUDA(cudaMemcpyAsync(h_nucleus + b0 * l * k, bf[i].U, (size_t)nb * l * k * 8, cudaMemcpyDeviceToHost,
                                cx->d2h));
    if (h_r) SLRA_CUDA(cudaMemcpyAsync(h_r + b0, bf[i].rr, (size_t)nb * 8, cudaMemcpyDeviceToHost, cx->d2h));
    if (h_status) SLRA_CUDA(cudaMemcpyAsync(h_status + b0, bf[i].st, (size_t)nb * 4, cudaMemcpyDeviceToHost, cx->d2h));
    if (h_resid_sq)
      SLRA_CUDA(cudaMemcpyAsync(h_resid_sq + b0, bf[i].rs, (size_t)nb * 8, cudaMemcpyDeviceToHost, cx->d2h));
    if (h_norm_sq)
      SLRA_CUDA(cudaMemcpyAsync(h_norm_sq + b0, bf[i].ns, (size_t)nb * 8, cudaMemcpyDeviceToHost, cx->d2h));
    SLRA_CUDA(cudaEventRecord(ev_out[i], cx->d2h));
  }
  SLRA_CUDA(cudaStreamSynchronize(cx->d2h));
  return SLRA_OK;
}
}  // namespace logk
}  // namespace slra_dev

using namespace slra_dev::logk;
using slra_dev::Context;
using slra_dev::C;

extern "C" {

int slra_cross_approx_batched_logkernel(slra_ctx ctx, const double* px, const double* py, const double* qx,
                                        const double* qy, int64_t nblocks, int64_t m, int64_t n, int64_t r, int64_t k,
                                        int64_t l, const int64_t* init_rows, int loops, double h, int64_t* I_out,
                                        int64_t* J_out, double* nucleus, int64_t* r_out, int32_t* status,
                                        double* resid_sq, double* norm_sq) {
  if (!ctx || !px || !py || !qx || !qy || loops < 1 || k < 1 || l < 1 || nblocks < 0 || (r > 0 && (k < r || l < r)))
    return SLRA_ERR_INVALID_ARGUMENT;
  if (!ca_fits((int)m, (int)n, (int)k, (int)l)) return SLRA_ERR_UNSUPPORTED;
  // the residual is always fused here (the blocks are never materialised)
  if (k > 32 || l > 32 || m % 8 || n % 8) return SLRA_ERR_UNSUPPORTED;
  if (nblocks == 0) return SLRA_OK;
  Context* cx = C(ctx);
  double* pairs = static_cast<double*>(workspace(cx, sizeof(double) * 2 * (size_t)nblocks));
  if (!pairs) return SLRA_ERR_CUDA;
  const int rq = (int)(k < l ? k : l);
  CaParams p{nullptr, m, m * n, (int)m, (int)n, (int)r, (int)k, (int)l, loops, h, init_rows, I_out, J_out, nucleus,
             r_out, status, nullptr, nullptr, nullptr, nullptr, nullptr, rq, 0};
  p.pairs = pairs;
  p.px = px;
  p.py = py;
  p.qx = qx;
  p.qy = qy;
  SLRA_TRY(launch_ca_block(cx, p, (int)nblocks));
  if (resid_sq) SLRA_CUDA(cudaMemcpy2DAsync(resid_sq, 8, pairs, 16, 8, nblocks, cudaMemcpyDeviceToDevice, cx->stream));
  if (norm_sq) SLRA_CUDA(cudaMemcpy2DAsync(norm_sq, 8, pairs + 1, 16, 8, nblocks, cudaMemcpyDeviceToDevice, cx->stream));
  return SLRA_OK;
}

int slra_cross_approx_batched_logkernel_host(slra_ctx ctx, const double* h_px, const double* h_py,
                                             const double* h_qx, const double* h_qy, int64_t nblocks, int64_t m,
                                             int64_t n, int64_t r, int64_t k, int64_t l, const int64_t* h_init,
                                             int loops, double h, int64_t* h_I, int64_t* h_J, double* h_nucleus,
                                             int64_t* h_r, int32_t* h_status, double* h_resid_sq,
                                             double* h_norm_sq) {
  if (!ctx || !h_px || !h_py || !h_qx || !h_qy || !h_init || loops < 1 || k < 1 || l < 1 || nblocks < 0 ||
      (r > 0 && (k < r || l < r)))
    return SLRA_ERR_INVALID_ARGUMENT;
  if (!ca_fits((int)m, (int)n, (int)k, (int)l) || k > 32 || l > 32 || m % 8 || n % 8) return SLRA_ERR_UNSUPPORTED;
  if (nblocks == 0) return SLRA_OK;
  // per block: m + m + n + n doubles of points (a chunk's px | py | qx | qy)
  auto upload = [&](double* d, int64_t b0, int64_t nb, int64_t chunk, cudaStream_t st) -> int {
    SLRA_CUDA(cudaMemcpyAsync(d, h_px + b0 * m, (size_t)nb * m * 8, cudaMemcpyHostToDevice, st));
    SLRA_CUDA(cudaMemcpyAsync(d + chunk * m, h_py + b0 * m, (size_t)nb * m * 8, cudaMemcpyHostToDevice, st));
    SLRA_CUDA(cudaMemcpyAsync(d + 2 * chunk * m, h_qx + b0 * n, (size_t)nb * n * 8, cudaMemcpyHostToDevice, st));
    SLRA_CUDA(cudaMemcpyAsync(d + 2 * chunk * m + chunk * n, h_qy + b0 * n, (size_t)nb * n * 8,
                              cudaMemcpyHostToDevice, st));
    return SLRA_OK;
  };
  auto run = [&](double* d, int64_t nb, int64_t chunk, const int64_t* init, int64_t* I, int64_t* J, double* U,
                 int64_t* rr, int32_t* st, double* rs, double* ns) -> int {
    return slra_cross_approx_batched_logkernel(ctx, d, d + chunk * m, d + 2 * chunk * m, d + 2 * chunk * m + chunk * n,
                                               nb, m, n, r, k, l, init, loops, h, I, J, U, rr, st, rs, ns);
  };
  // eight chunks: the points of chunk c + 1 cross the bus during chunk c
  return ca_batched_host_stream(ctx, nblocks, 2 * m + 2 * n, k, l, h_init, h_I, h_J, h_nucleus, h_r, h_status,
                                h_resid_sq, h_norm_sq, upload, run, (nblocks + 7) / 8);
}

}  // extern "C"
