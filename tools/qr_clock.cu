// Probe: cycles per phase of the CTA-resident Householder QR / Q formation / Jacobi.
#include <cstdio>
#include <vector>
#include "../paper_1611_01391_b200/csrc/dense_cta.cuh"
using namespace slra_dev;
template <int NT>
__global__ void probe(const double* A, int m, int c, long long* clk, double* out) {
  extern __shared__ double sm[];
  double* S = sm; double* Q = S + m * c; double* tau = Q + m * c; double* red = tau + 64;
  for (int e = threadIdx.x; e < m * c; e += NT) S[e] = A[e];
  __syncthreads();
  long long t0 = clock64();
  cta_house_qr<NT>(S, m, m, c, tau, red);
  long long t1 = clock64();
  cta_form_q<NT>(S, m, m, c, tau, Q, m);
  __syncthreads();
  long long t2 = clock64();
  // jacobi on the c x c top block (as W), V after
  double* W = Q; double* V = Q + m * c - c * c; int* flag = (int*)(red + 80);
  cta_jacobi<NT>(S, m, c, c, V, c, flag);
  long long t3 = clock64();
  if (threadIdx.x == 0) { clk[0] = t1 - t0; clk[1] = t2 - t1; clk[2] = t3 - t2; out[0] = S[0] + Q[1]; }
}
int main() {
  for (int c : {8, 16, 32, 48}) {
    int m = 256;
    std::vector<double> h(m * c);
    for (auto& x : h) x = (double)rand() / RAND_MAX - 0.5;
    double *dA, *dout; long long* dclk;
    cudaMalloc(&dA, 8 * m * c); cudaMalloc(&dout, 64); cudaMalloc(&dclk, 64);
    cudaMemcpy(dA, h.data(), 8 * m * c, cudaMemcpyHostToDevice);
    size_t smem = 8 * (2 * m * c + 64 + 200);
    cudaFuncSetAttribute(probe<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(probe<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    long long clk[3];
    probe<512><<<1, 512, smem>>>(dA, m, c, dclk, dout);
    cudaMemcpy(clk, dclk, 24, cudaMemcpyDeviceToHost);
    printf("NT=512 m=%d c=%d  qr %lld cyc (%.0f/col)  formQ %lld  jacobi(cxc) %lld  err=%s\n", m, c, clk[0], clk[0] / (double)c, clk[1], clk[2], cudaGetErrorString(cudaGetLastError()));
    probe<256><<<1, 256, smem>>>(dA, m, c, dclk, dout);
    cudaMemcpy(clk, dclk, 24, cudaMemcpyDeviceToHost);
    printf("NT=256 m=%d c=%d  qr %lld cyc (%.0f/col)  formQ %lld  jacobi(cxc) %lld\n", m, c, clk[0], clk[0] / (double)c, clk[1], clk[2]);
  }
}
