// Probe: dependent-chain latency (cycles/op) of FP64 primitives on one warp.
#include <cstdio>
__device__ double warp_sum(double v) { for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o); return v; }
__global__ void k(double x0, long long* clk, double* out) {
  double x = x0 + threadIdx.x * 1e-9; long long t0, t1; const int N = 64;
  __shared__ double sm[1024];
  t0 = clock64(); for (int i = 0; i < N; ++i) x = sqrt(x + 1.0); t1 = clock64(); if (threadIdx.x == 0) clk[0] = (t1 - t0) / N;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = 1.0 / (x + 1.0); t1 = clock64(); if (threadIdx.x == 0) clk[1] = (t1 - t0) / N;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = __drcp_rn(x + 1.0); t1 = clock64(); if (threadIdx.x == 0) clk[2] = (t1 - t0) / N;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = rsqrt(x + 1.0); t1 = clock64(); if (threadIdx.x == 0) clk[3] = (t1 - t0) / N;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = fma(x, 1.0000001, 1e-9); t1 = clock64(); if (threadIdx.x == 0) clk[4] = (t1 - t0) / N;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = warp_sum(x) * 1e-3; t1 = clock64(); if (threadIdx.x == 0) clk[5] = (t1 - t0) / N;
  t0 = clock64(); for (int i = 0; i < N; ++i) { sm[threadIdx.x] = x; __syncthreads(); x = sm[(threadIdx.x + 1) & 31] * 0.5; __syncthreads(); } t1 = clock64(); if (threadIdx.x == 0) clk[6] = (t1 - t0) / N;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = (x + 1.0) / (x + 2.0); t1 = clock64(); if (threadIdx.x == 0) clk[7] = (t1 - t0) / N;
  out[threadIdx.x] = x;
}
int main() {
  long long* d; double* o; cudaMalloc(&d, 128); cudaMalloc(&o, 8 * 1024);
  const char* names[] = {"sqrt", "1/x", "__drcp_rn", "rsqrt", "fma", "warp_sum(5 shfl)", "sts+bar+lds+bar", "a/b"};
  for (int nt : {32, 512}) {
    k<<<1, nt>>>(2.0, d, o); long long h[8]; cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    printf("threads=%d: ", nt); for (int i = 0; i < 8; ++i) printf("%s=%lld  ", names[i], h[i]); printf("\n");
  }
}
