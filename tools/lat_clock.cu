// Probe: dependent-chain latencies (cycles) of the FP64 operations the small
// dense kernels are built from, measured on one warp.
#include <cstdio>

__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)::"memory");
  return c;
}

template <int K>
__global__ void lat(const double* in, double* out, long long* cyc) {
  __shared__ double sm[1024];
  double a = in[threadIdx.x], b = in[32 + threadIdx.x];
  for (int i = threadIdx.x; i < 1024; i += 32) sm[i] = in[i % 64] + i;
  __syncwarp();
  constexpr int N = 256;
  long long t0 = clk();
#pragma unroll 1
  for (int i = 0; i < N; ++i) {
    if (K == 0) a = fma(a, b, 0.5);
    if (K == 1) a = sqrt(a + 2.0);
    if (K == 2) a = 1.0 / (a + 2.0);
    if (K == 3) a = b / (a + 2.0);
    if (K == 4) a = rsqrt(a + 2.0);
    if (K == 5) a = __shfl_xor_sync(0xffffffffu, a, 1) + 1.0;
    if (K == 6) a = sm[((int)a) & 1023] + 1.0;
    if (K == 7) { __syncthreads(); a = a + 1.0; }
    if (K == 8) a = __drcp_rn(a + 2.0);
    if (K == 9) a = a * b + 1.0;
  }
  long long t1 = clk();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[K] = (t1 - t0) / N;
}

int main() {
  double *in, *out;
  long long* cyc;
  cudaMalloc(&in, 8 * 1024);
  cudaMalloc(&out, 8 * 1024);
  cudaMalloc(&cyc, 8 * 16);
  double h[1024];
  for (int i = 0; i < 1024; ++i) h[i] = 1.0 + i * 1e-3;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  lat<0><<<1, 32>>>(in, out, cyc);
  lat<1><<<1, 32>>>(in, out, cyc);
  lat<2><<<1, 32>>>(in, out, cyc);
  lat<3><<<1, 32>>>(in, out, cyc);
  lat<4><<<1, 32>>>(in, out, cyc);
  lat<5><<<1, 32>>>(in, out, cyc);
  lat<6><<<1, 32>>>(in, out, cyc);
  lat<7><<<1, 256>>>(in, out, cyc);
  lat<8><<<1, 32>>>(in, out, cyc);
  lat<9><<<1, 32>>>(in, out, cyc);
  long long c[16];
  cudaMemcpy(c, cyc, 8 * 16, cudaMemcpyDeviceToHost);
  const char* nm[] = {"dfma", "sqrt", "1/x", "a/b", "rsqrt", "shfl+add", "lds+add", "bar(256)+add", "drcp_rn", "dmul+add"};
  for (int k = 0; k < 10; ++k) printf("%-14s %lld cycles\n", nm[k], c[k]);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
