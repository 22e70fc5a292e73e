// FP64 peak microbenchmarks for the roofline denominator (DMMA and DFMA pipes).
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
}

template <int NACC>
__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-9;
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1234.5) out[0] = s;
}

template <int NACC>
__global__ void dfma(double* out, int iters) {
  double c[NACC];
  double a = 1.0 + threadIdx.x * 1e-12, b = 0.999999;
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 1234.5) out[0] = s;
}

template <typename F>
double run(F kern, int blocks, int threads, int iters, double flop_per_iter_per_warp) {
  double* d; cudaMalloc(&d, 8);
  kern<<<blocks, threads>>>(d, 10);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  cudaFree(d);
  double warps = (double)blocks * threads / 32;
  return warps * iters * flop_per_iter_per_warp / (best * 1e-3) / 1e12;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int it = 20000;
  for (int bpsm : {1, 2, 4}) {
    for (int th : {128, 256, 512}) {
      printf("{\"kind\":\"dmma_m8n8k4\",\"blocks_per_sm\":%d,\"threads\":%d,\"tflops\":%.2f}\n", bpsm, th,
             run(dmma_m8n8k4<8>, sms * bpsm, th, it, 8 * 512.0));
      printf("{\"kind\":\"dmma_m16n8k16\",\"blocks_per_sm\":%d,\"threads\":%d,\"tflops\":%.2f}\n", bpsm, th,
             run(dmma_m16n8k16<4>, sms * bpsm, th, it / 4, 4 * 4096.0));
      printf("{\"kind\":\"dfma\",\"blocks_per_sm\":%d,\"threads\":%d,\"tflops\":%.2f}\n", bpsm, th,
             run(dfma<8>, sms * bpsm, th, it, 8 * 64.0));
    }
  }
  return 0;
}
