// Probe: Jacobi sweeps actually used (flag-based) for random n x n on the device.
#include <cstdio>
#include <vector>
#include "../paper_1611_01391_b200/csrc/dense_cta.cuh"
using namespace slra_dev;
__global__ void __launch_bounds__(256) probe(const double* A, int n, long long* clk, double* out) {
  __shared__ double W[48 * 48], V[48 * 48];
  __shared__ int flag[4];
  for (int e = threadIdx.x; e < n * n; e += 256) W[e] = A[e];
  __syncthreads();
  long long t0 = clock64();
  cta_jacobi<256>(W, n, n, n, V, n, flag, 0.0);
  long long t1 = clock64();
  __syncthreads();
  // off-diagonality after
  if (threadIdx.x == 0) {
    double off = 0;
    for (int a = 0; a < n; ++a) for (int b = a + 1; b < n; ++b) {
      double aa = 0, bb = 0, gg = 0;
      for (int i = 0; i < n; ++i) { aa += W[i + a * n] * W[i + a * n]; bb += W[i + b * n] * W[i + b * n]; gg += W[i + a * n] * W[i + b * n]; }
      off = fmax(off, fabs(gg) / sqrt(aa * bb));
    }
    clk[0] = t1 - t0; out[0] = off; clk[1] = flag[2];
  }
}
int main() {
  for (int n : {8, 16, 32, 48}) {
    std::vector<double> h(n * n);
    for (auto& x : h) x = (double)rand() / RAND_MAX - 0.5;
    double *dA, *dout; long long* dclk;
    cudaMalloc(&dA, 8 * n * n); cudaMalloc(&dout, 64); cudaMalloc(&dclk, 64);
    cudaMemcpy(dA, h.data(), 8 * n * n, cudaMemcpyHostToDevice);
    probe<<<1, 256>>>(dA, n, dclk, dout);
    long long c, cc[2]; double off;
    cudaMemcpy(cc, dclk, 16, cudaMemcpyDeviceToHost); c = cc[0]; cudaMemcpy(&off, dout, 8, cudaMemcpyDeviceToHost);
    printf("n=%d jacobi %lld cycles (%.0f per round at %d rounds/sweep) offdiag %.3e sweeps %lld %s\n", n, c, c / (double)(n - 1), n - 1, off, cc[1], cudaGetErrorString(cudaGetLastError()));
  }
}
