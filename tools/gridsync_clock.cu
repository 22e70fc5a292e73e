// Probe: cost of one cooperative-groups grid barrier vs a hand-rolled
// flag barrier (one atomic per CTA + spin on a generation counter).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void cg_sync(int iters, long long* out) {
  cg::grid_group g = cg::this_grid();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (clock64() - t0) / iters;
}

__global__ void flag_sync(int iters, unsigned* count, volatile unsigned* gen, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned my = *gen;
      __threadfence();
      if (atomicAdd(count, 1u) == gridDim.x - 1) {
        *count = 0;
        __threadfence();
        *gen = my + 1;
      } else {
        while (*gen == my) {
        }
      }
      __threadfence();
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[1] = (clock64() - t0) / iters;
}

int main() {
  long long* out;
  unsigned* cnt;
  unsigned* gen;
  cudaMalloc(&out, 16);
  cudaMalloc(&cnt, 4);
  cudaMalloc(&gen, 4);
  for (int G : {16, 64, 148}) {
    cudaMemset(cnt, 0, 4);
    cudaMemset(gen, 0, 4);
    int iters = 1000;
    void* args[] = {&iters, &out};
    cudaLaunchCooperativeKernel((void*)cg_sync, G, 256, args, 0, 0);
    void* args2[] = {&iters, &cnt, &gen, &out};
    cudaLaunchCooperativeKernel((void*)flag_sync, G, 256, args2, 0, 0);
    long long h[2];
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("G=%d: cg grid.sync %lld cycles, flag barrier %lld cycles  (%s)\n", G, h[0], h[1],
           cudaGetErrorString(cudaGetLastError()));
  }
}
