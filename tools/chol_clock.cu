// Probe: per-phase cycles of one Cholesky column step (48 x 48, 256 threads),
// the step structure of chol_small_kernel (csrc/cholqr.cu).
#include <cstdio>
#include <cmath>
#include <vector>

constexpr int NT = 256, NMAX = 64;

__global__ void __launch_bounds__(NT) probe(const double* G, int n, long long* clk, double* out) {
  __shared__ double L[NMAX * (NMAX + 1)];
  const int tid = threadIdx.x, ld = n + 1;
  long long ts0 = clock64();
  // the partial-sum phase of chol_small_kernel: 32 partial Grams (here all = G / 32)
  const int64_t nn = (int64_t)n * n;
  for (int e = tid; e < n * n; e += NT) {
    const int i = e % n, c = e / n;
    if (i > c) continue;
    double s = 0.0;
#pragma unroll 8
    for (int k = 0; k < 32; ++k) s += G[k * nn + e];
    L[c + i * ld] = s;
    L[i + c * ld] = s;
  }
  __syncthreads();
  long long ts1 = clock64();
  if (tid == 0) clk[4] = ts1 - ts0;
  constexpr int kQ = NMAX / 4;
  const int ti = tid & 63, tc = tid >> 6;
  long long tA = 0, tB = 0, tC = 0, tD = 0;
  for (int j = 0; j < n; ++j) {
    long long t0 = clock64();
    const double piv = L[j + j * ld];
    const double ljj = sqrt(piv);
    const double inv = 1.0 / ljj;
    long long t1 = clock64();
    const bool row = ti > j && ti < n;
    const double lij = row ? L[ti + j * ld] * inv : 0.0;
    double lcj[kQ], cur[kQ];
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      const int c = tc + 4 * q;
      const bool act = row && c > j && c <= ti;
      lcj[q] = act ? L[c + j * ld] * inv : 0.0;
      cur[q] = act ? L[ti + c * ld] : 0.0;
    }
    long long t2 = clock64();
    __syncthreads();
    long long t3 = clock64();
    if (tc == 0 && ti >= j && ti < n) L[ti + j * ld] = (ti == j) ? ljj : lij;
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      const int c = tc + 4 * q;
      if (row && c > j && c <= ti) L[ti + c * ld] = cur[q] - lij * lcj[q];
    }
    __syncthreads();
    long long t4 = clock64();
    tA += t1 - t0; tB += t2 - t1; tC += t3 - t2; tD += t4 - t3;
  }
  if (tid == 0) { clk[0] = tA; clk[1] = tB; clk[2] = tC; clk[3] = tD; out[0] = L[(n - 1) + (n - 1) * ld]; }
}

// microbench of the special functions in a dependent chain
__global__ void ops(double x, long long* clk, double* out) {
  double a = x;
  long long t0 = clock64();
  for (int i = 0; i < 64; ++i) a = sqrt(a + 1.0);
  long long t1 = clock64();
  for (int i = 0; i < 64; ++i) a = 1.0 / (a + 1.0);
  long long t2 = clock64();
  for (int i = 0; i < 64; ++i) a = fma(a, 0.999, 0.5);
  long long t3 = clock64();
  clk[0] = (t1 - t0) / 64; clk[1] = (t2 - t1) / 64; clk[2] = (t3 - t2) / 64;
  out[0] = a;
}

int main() {
  const int n = 48;
  std::vector<double> h(32 * n * n, 0.0);
  for (int k = 0; k < 32; ++k)
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) h[k * n * n + i + j * n] = ((i == j ? n : 0.0) + 1.0 / (1 + i + j)) / 32;
  double *dG, *dout;
  long long* dclk;
  cudaMalloc(&dG, 8 * 32 * n * n);
  cudaMalloc(&dout, 64);
  cudaMalloc(&dclk, 64);
  cudaMemcpy(dG, h.data(), 8 * 32 * n * n, cudaMemcpyHostToDevice);
  long long c[5];
  for (int rep = 0; rep < 3; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<<<1, NT>>>(dG, n, dclk, dout);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(c, dclk, 40, cudaMemcpyDeviceToHost);
    printf("chol n=%d: %.1f us; partial sums %lld cycles; per step cycles: sqrt+rcp %.0f, stage %.0f, bar1 %.0f, "
           "write+bar2 %.0f\n", n, ms * 1e3, c[4], c[0] / (double)n, c[1] / (double)n, c[2] / (double)n,
           c[3] / (double)n);
  }
  ops<<<1, 1>>>(2.0, dclk, dout);
  cudaMemcpy(c, dclk, 24, cudaMemcpyDeviceToHost);
  printf("dependent-chain cycles: sqrt %lld, 1/x %lld, fma %lld  (%s)\n", c[0], c[1], c[2],
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
