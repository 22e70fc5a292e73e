// Probe: per-phase cycles of one round of the 8-lane-group one-sided Jacobi
// (cta_jacobi_g8, csrc/dense_cta.cuh) on a 48 x 48 graded matrix.
#include <cstdio>
#include <cmath>
#include <vector>

constexpr int NT = 256;
constexpr double kEps = 2.220446049250313e-16;

__global__ void __launch_bounds__(NT) probe(const double* A, int n, long long* clk, int* sweeps_out) {
  __shared__ double W[48 * 48], V[48 * 48];
  __shared__ unsigned short pair_tab[64 * 32];
  __shared__ int flag[2];
  const int p = n, ldw = n, ldv = n;
  constexpr int RPG = 8;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = lane >> 3, sub = lane & 7;
  constexpr int NW = NT / 32;
  for (int e = tid; e < n * n; e += NT) {
    W[e] = A[e];
    V[e] = (e % n == e / n) ? 1.0 : 0.0;
  }
  const int ne = n + (n & 1);
  for (int e = tid; e < (ne - 1) * (ne / 2); e += NT) {
    const int rd = e / (ne / 2), pi = e % (ne / 2);
    int a, b;
    if (pi == 0) { a = rd; b = ne - 1; } else { a = (rd + pi) % (ne - 1); b = (rd - pi + ne - 1) % (ne - 1); }
    if (a > b) { const int t = a; a = b; b = t; }
    pair_tab[e] = (unsigned short)((a << 8) | b);
  }
  const double tol = 16.0 * (double)p * kEps;
  if (tid == 0) flag[0] = flag[1] = 0;
  __syncthreads();
  const int npairs = ne / 2;
  long long ph[6] = {0, 0, 0, 0, 0, 0};
  long long rounds = 0;
  int sw = 0;
  for (int sweep = 0; sweep < 40; ++sweep) {
    const int fl = sweep & 1;
    for (int rd = 0; rd < ne - 1; ++rd) {
      long long t0 = clock64();
      const int pi = warp * 4 + grp;
      const int ab = pair_tab[rd * npairs + (pi < npairs ? pi : 0)];
      const bool valid = pi < npairs && (ab & 255) < n;
      const int a = ab >> 8, b = valid ? (ab & 255) : a;
      double* wp = W + a * ldw;
      double* wq = W + b * ldw;
      double* vp = V + a * ldv;
      double* vq = V + b * ldv;
      double x[RPG], y[RPG], u[RPG], v[RPG];
      double aa = 0.0, bb = 0.0, gg = 0.0;
#pragma unroll
      for (int r = 0; r < RPG; ++r) {
        const int i = sub + 8 * r;
        x[r] = i < p ? wp[i] : 0.0;
        y[r] = i < p ? wq[i] : 0.0;
        u[r] = i < n ? vp[i] : 0.0;
        v[r] = i < n ? vq[i] : 0.0;
      }
#pragma unroll
      for (int r = 0; r < RPG; ++r) {
        aa = fma(x[r], x[r], aa);
        bb = fma(y[r], y[r], bb);
        gg = fma(x[r], y[r], gg);
      }
      long long t1 = clock64();
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        aa += __shfl_xor_sync(0xffffffffu, aa, o);
        bb += __shfl_xor_sync(0xffffffffu, bb, o);
        gg += __shfl_xor_sync(0xffffffffu, gg, o);
      }
      long long t2 = clock64(), t3 = t2, t4 = t2, t5 = t2;
      const bool rot = valid && gg != 0.0 && gg * gg > tol * tol * (aa * bb);
      if (rot) {
        const double d = bb - aa, g2 = 2.0 * gg;
        const double rr = sqrt(fma(d, d, g2 * g2));
        const double t = copysign(1.0, d) * g2 / (fabs(d) + rr);
        const double cs = rsqrt(fma(t, t, 1.0));
        const double sn = cs * t;
        t3 = clock64();
#pragma unroll
        for (int r = 0; r < RPG; ++r) {
          const int i = sub + 8 * r;
          if (i < p) { wp[i] = cs * x[r] - sn * y[r]; wq[i] = sn * x[r] + cs * y[r]; }
          if (i < n) { vp[i] = cs * u[r] - sn * v[r]; vq[i] = sn * u[r] + cs * v[r]; }
        }
        t4 = clock64();
        t5 = t4;
        if (sub == 0) flag[fl] = 1;
      }
      __syncthreads();
      long long t6 = clock64();
      if (tid == 0) {
        ph[0] += t1 - t0; ph[1] += t2 - t1; ph[2] += t3 - t2; ph[3] += t4 - t3; ph[4] += t5 - t4; ph[5] += t6 - t5;
        ++rounds;
      }
    }
    const int rotated = flag[fl];
    if (tid == 0) flag[fl ^ 1] = 0;
    __syncthreads();
    sw = sweep + 1;
    if (!rotated) break;
  }
  if (tid == 0) {
    for (int k = 0; k < 6; ++k) clk[k] = ph[k];
    clk[6] = rounds;
    *sweeps_out = sw;
  }
}

int main() {
  const int n = 48;
  std::vector<double> h(n * n);
  srand(1);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) h[i + j * n] = ((double)rand() / RAND_MAX - 0.5) * pow(0.5, j < 32 ? j : 40);
  double* dA;
  long long* dclk;
  int* dsw;
  cudaMalloc(&dA, 8 * n * n);
  cudaMalloc(&dclk, 64);
  cudaMalloc(&dsw, 4);
  cudaMemcpy(dA, h.data(), 8 * n * n, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<<<1, NT>>>(dA, n, dclk, dsw);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c[7];
    int sw;
    cudaMemcpy(c, dclk, 56, cudaMemcpyDeviceToHost);
    cudaMemcpy(&sw, dsw, 4, cudaMemcpyDeviceToHost);
    const double r = (double)c[6];
    printf("jacobi 48: %.1f us, %d sweeps, %lld rounds; per round: load+dot %.0f shfl %.0f rot %.0f W %.0f V %.0f "
           "bar %.0f\n", ms * 1e3, sw, c[6], c[0] / r, c[1] / r, c[2] / r, c[3] / r, c[4] / r, c[5] / r);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
