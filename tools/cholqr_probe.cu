// Probe: device time of the CholeskyQR3 kernels in isolation (events), to
// separate kernel cost from launch gaps in the bench's family timings.
#include <cstdio>
#include <vector>

#include "../paper_1611_01391_b200/csrc/cholqr.cu"

using namespace slra_dev;

int main() {
  const int m = 4096, n = 48, nb = 2;
  const int64_t per = (int64_t)cholqr3_workspace_doubles(m, n);
  std::vector<double> hY((size_t)nb * m * n);
  srand(3);
  for (auto& x : hY) x = (double)rand() / RAND_MAX - 0.5;
  double *Y, *ws;
  int32_t* st;
  cudaMalloc(&Y, 8 * hY.size());
  cudaMalloc(&ws, 8 * per * nb);
  cudaMalloc(&st, 4 * nb);
  cudaMemcpy(Y, hY.data(), 8 * hY.size(), cudaMemcpyHostToDevice);
  cudaMemset(st, 0, 4 * nb);
  const int64_t nn = (int64_t)n * n, nch = (m + 127) / 128;
  double* P = ws + (int64_t)m * n;
  double* R1 = P + nch * 64 * 64;
  double* rinv = R1 + 3 * nn;
  const size_t gsm = sizeof(double) * (128 + 1) * n;
  cudaFuncSetAttribute(gram_partial_kernel<48>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsm);
  cudaEvent_t e[4];
  for (auto& x : e) cudaEventCreate(&x);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e[0]);
    gram_partial_kernel<48><<<dim3(nch, nb), 256, gsm>>>(Y, m, (int64_t)m * n, m, n, P, per, st);
    cudaEventRecord(e[1]);
    chol_small_kernel<48><<<nb, 256>>>(P, per, (int)nch, n, 1e-12, R1, per, rinv, per, st);
    cudaEventRecord(e[2]);
    trsm_rows_kernel<48><<<dim3((m + 127) / 128, nb), 128>>>(Y, m, (int64_t)m * n, m, n, R1, per, rinv, per, ws,
                                                             m, per, st);
    cudaEventRecord(e[3]);
    cudaEventSynchronize(e[3]);
    float a, b, c;
    cudaEventElapsedTime(&a, e[0], e[1]);
    cudaEventElapsedTime(&b, e[1], e[2]);
    cudaEventElapsedTime(&c, e[2], e[3]);
    int32_t hs[2];
    cudaMemcpy(hs, st, 8, cudaMemcpyDeviceToHost);
    printf("gram %.1f us  chol %.1f us  trsm %.1f us  status %d %d  %s\n", a * 1e3, b * 1e3, c * 1e3, hs[0], hs[1],
           cudaGetErrorString(cudaGetLastError()));
  }
}
