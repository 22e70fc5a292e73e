// Probe: device time of the LSR solve kernels (Cholesky d x d, two-sided
// triangular solve) in isolation, d = 256.
#include <cmath>
#include <cstdio>
#include <vector>

#include "../paper_1611_01391_b200/csrc/lsr.cu"

using namespace slra_dev;
namespace slra_dev {
#include "lsr_probe_chol.cuh"
}

int main() {
  const int d = 256;
  std::vector<double> G((size_t)d * d, 0.0);
  srand(7);
  std::vector<double> X((size_t)d * 2 * d);
  for (auto& x : X) x = (double)rand() / RAND_MAX - 0.5;
  for (int i = 0; i < d; ++i)  // G = X X^T (2d columns): SPD, cond ~ 10
    for (int j = 0; j < d; ++j) {
      double s = 0;
      for (int t = 0; t < 2 * d; ++t) s += X[i + (size_t)t * d] * X[j + (size_t)t * d];
      G[i + (size_t)j * d] = s;
    }
  double *dG, *dL, *rhs, *x;
  int32_t* st;
  cudaMalloc(&dG, 8 * G.size());
  cudaMalloc(&dL, 8 * G.size());
  cudaMalloc(&rhs, 8 * d);
  cudaMalloc(&x, 8 * d);
  cudaMalloc(&st, 4);
  cudaMemcpy(dG, G.data(), 8 * G.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(rhs, G.data(), 8 * d, cudaMemcpyHostToDevice);
  cudaMemset(st, 0, 4);
  const size_t smem = sizeof(double) * ((size_t)(d + 1) * kPW + d + kPW);
  cudaFuncSetAttribute(cholesky_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e[3];
  for (auto& v : e) cudaEventCreate(&v);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(dL, dG, 8 * G.size(), cudaMemcpyDeviceToDevice);
    cudaEventRecord(e[0]);
    cholesky_kernel<<<1, kLT, smem>>>(dL, d, 1e-30, st);
    if (rep == 2) {
      long long* dclk; cudaMalloc(&dclk, 64);
      cudaMemcpy(dL, dG, 8 * G.size(), cudaMemcpyDeviceToDevice);
      cudaFuncSetAttribute(chol_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      chol_probe<<<1, kLT, smem>>>(dL, d, 1e-30, st, dclk);
      long long c[5]; cudaMemcpy(c, dclk, 40, cudaMemcpyDeviceToHost);
      printf("chol phases (cycles, all panels): load %lld diag %lld L21 %lld writeback %lld trailing %lld\n", c[0], c[1], c[2], c[3], c[4]);
      cudaMemcpy(dL, dG, 8 * G.size(), cudaMemcpyDeviceToDevice);
      cholesky_kernel<<<1, kLT, smem>>>(dL, d, 1e-30, st);
    }
    cudaEventRecord(e[1]);
    chol_solve_kernel<<<1, kST, 8 * d>>>(dL, d, rhs, x, st, 0);
    cudaEventRecord(e[2]);
    cudaEventSynchronize(e[2]);
    float a, b;
    cudaEventElapsedTime(&a, e[0], e[1]);
    cudaEventElapsedTime(&b, e[1], e[2]);
    int hs;
    cudaMemcpy(&hs, st, 4, cudaMemcpyDeviceToHost);
    std::vector<double> hx(d);
    cudaMemcpy(hx.data(), x, 8 * d, cudaMemcpyDeviceToHost);
    // x should be G^-1 G(:,0) = e_0
    double err = std::fabs(hx[0] - 1.0);
    for (int i = 1; i < d; ++i) err = std::fmax(err, std::fabs(hx[i]));
    printf("cholesky %.1f us  solve %.1f us  status %d  |x - e0| %.2e  %s\n", a * 1e3, b * 1e3, hs, err,
           cudaGetErrorString(cudaGetLastError()));
  }
}
