// Timing + accuracy of k_inverse_cholesky (csrc/nys_inverse.cuh) in isolation:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I paper_1901_06112_b200/csrc tools/microbench/inv_phases.cu
// Reads L from device memory, and from mapped pinned memory with the image copy.
#include <cstdio>
#include <cmath>
#include <vector>
#define NYS_INV_STAMPS
#include "nys_inverse.cuh"
using namespace nys;
int main() {
  for (int n : {64, 48, 13}) {
    std::vector<double> A((size_t)n * n), L((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) A[i * n + j] = std::exp(-0.02 * (i - j) * (i - j)) + (i == j ? 0.5 : 0.0);
    for (int j = 0; j < n; ++j) {
      double s = A[j * n + j];
      for (int k = 0; k < j; ++k) s -= L[j * n + k] * L[j * n + k];
      L[j * n + j] = std::sqrt(s);
      for (int i = j + 1; i < n; ++i) {
        double t = A[i * n + j];
        for (int k = 0; k < j; ++k) t -= L[i * n + k] * L[j * n + k];
        L[i * n + j] = t / L[j * n + j];
      }
    }
    double *dL, *hL;
    float *dM, *img_h, *img_d;
    const int m0q = 72, nf4 = 1500;
    cudaMalloc(&dL, n * n * 8);
    cudaMalloc(&dM, 64 * m0q * 4);
    cudaHostAlloc(&hL, n * n * 8, 0);
    cudaHostAlloc(&img_h, nf4 * 16, 0);
    cudaMalloc(&img_d, nf4 * 16);
    memcpy(hL, L.data(), n * n * 8);
    cudaMemcpy(dL, L.data(), n * n * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_inverse_cholesky, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kInvSmemBytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode = 0; mode < 2; ++mode) {
      const double* src = mode ? hL : dL;
      const float4* is = mode ? (const float4*)img_h : nullptr;
      for (int it = 0; it < 3; ++it) k_inverse_cholesky<<<1, 1024, kInvSmemBytes>>>(src, n, dM, m0q, nullptr, is, (float4*)img_d, nf4, nullptr);
      cudaEventRecord(a);
      for (int it = 0; it < 20; ++it) k_inverse_cholesky<<<1, 1024, kInvSmemBytes>>>(src, n, dM, m0q, nullptr, is, (float4*)img_d, nf4, nullptr);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      std::vector<float> M((size_t)64 * m0q);
      cudaMemcpy(M.data(), dM, M.size() * 4, cudaMemcpyDeviceToHost);
      double err = 0.0;  // || A M - I ||_max
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          double t = 0.0;
          for (int k = 0; k < n; ++k) t += A[i * n + k] * (double)M[(size_t)j * m0q + k];
          err = std::fmax(err, std::fabs(t - (i == j ? 1.0 : 0.0)));
        }
      long long st[8];
      cudaMemcpyFromSymbol(st, g_inv_stamps, sizeof(st));
      printf("n=%d %s  %.2f us/launch  |AM-I|max %.2e  cycles: load %lld diag %lld doubling %lld product %lld  %s\n", n,
             mode ? "pinned+image" : "device     ", ms * 1000 / 20, err, st[1] - st[0], st[2] - st[1], st[3] - st[2],
             st[4] - st[3], cudaGetErrorString(cudaGetLastError()));
    }
  }
}
