// Phase timing of the blocked Cholesky-inverse kernel (k_inverse_cholesky in
// nys_filter.cu), standalone: nvcc -O3 -gencode arch=compute_100a,code=sm_100a inv_phases.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
__global__ void __launch_bounds__(1024) kinv(const double* __restrict__ Lg, int n, float* __restrict__ MT, int m0q,
                                             long long* stamps) {
  extern __shared__ double cs[];
  long long t0 = clock64();
  const int np = (n + 7) & ~7, nb = np / 8;
  double* Ls = cs;
  double* X = Ls + np * np;
  double* Di = X + np * np;
  double* R = Di + np * 8;
  for (int e = threadIdx.x; e < np * np; e += blockDim.x) {
    const int i = e / np, j = e - i * np;
    Ls[e] = (i < n && j < n) ? Lg[i * n + j] : (i == j ? 1.0 : 0.0);
    X[e] = 0.0;
  }
  __syncthreads();
  long long t1 = clock64();
  if ((int)threadIdx.x < np) {
    const int I = threadIdx.x >> 3, c = threadIdx.x & 7, o = 8 * I;
    double col[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      double t = (a == c) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < a; ++k) t = fma(-Ls[(o + a) * np + o + k], col[k], t);
      col[a] = (a < c) ? 0.0 : t / Ls[(o + a) * np + o + a];
    }
#pragma unroll
    for (int a = 0; a < 8; ++a) Di[(o + a) * 8 + c] = col[a];
  }
  __syncthreads();
  long long t2 = clock64();
  for (int I = 0; I < nb; ++I) {
    const int o = 8 * I, w = o + 8;
    for (int e = threadIdx.x; e < 8 * w; e += blockDim.x) {
      const int a = e / w, j = e - a * w;
      const double* lr = Ls + (o + a) * np;
      double q0 = (o + a == j) ? 1.0 : 0.0, q1 = 0.0, q2 = 0.0, q3 = 0.0;
      int k = j;
      for (; k + 3 < o; k += 4) {
        q0 = fma(-lr[k], X[k * np + j], q0);
        q1 = fma(-lr[k + 1], X[(k + 1) * np + j], q1);
        q2 = fma(-lr[k + 2], X[(k + 2) * np + j], q2);
        q3 = fma(-lr[k + 3], X[(k + 3) * np + j], q3);
      }
      for (; k < o; ++k) q0 = fma(-lr[k], X[k * np + j], q0);
      R[a * np + j] = (q0 + q1) + (q2 + q3);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 8 * w; e += blockDim.x) {
      const int a = e / w, j = e - a * w;
      double t = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) t = fma(Di[(o + a) * 8 + q], R[q * np + j], t);
      X[(o + a) * np + j] = t;
    }
    __syncthreads();
  }
  long long t3 = clock64();
  const int nq = (n + 3) / 4;
  for (int e = threadIdx.x; e < n * nq; e += blockDim.x) {
    const int i = e / nq, j0 = 4 * (e - i * nq);
    double t[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = max(i, j0); k < n; ++k) {
      const double xi = X[k * np + i];
#pragma unroll
      for (int q = 0; q < 4; ++q) t[q] = fma(xi, X[k * np + j0 + q], t[q]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (j0 + q < n) MT[(size_t)(j0 + q) * m0q + i] = (float)t[q];
  }
  __syncthreads();
  long long t4 = clock64();
  if (threadIdx.x == 0) { stamps[0] = t1 - t0; stamps[1] = t2 - t1; stamps[2] = t3 - t2; stamps[3] = t4 - t3; }
}
int main() {
  for (int n : {64, 90}) {
    std::vector<double> L(n * n, 0.0);
    for (int i = 0; i < n; ++i) for (int j = 0; j <= i; ++j) L[i * n + j] = i == j ? 2.0 : 0.01 * ((i * 7 + j * 3) % 11);
    double* dL; float* dM; long long* ds;
    cudaMalloc(&dL, n * n * 8); cudaMalloc(&dM, n * 96 * 4); cudaMalloc(&ds, 64);
    cudaMemcpy(dL, L.data(), n * n * 8, cudaMemcpyHostToDevice);
    const int np = (n + 7) & ~7;
    const size_t smem = (2 * (size_t)np * np + 16 * (size_t)np) * 8;
    cudaFuncSetAttribute(kinv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int it = 0; it < 3; ++it) kinv<<<1, 1024, smem>>>(dL, n, dM, 96, ds);
    cudaEventRecord(a);
    for (int it = 0; it < 20; ++it) kinv<<<1, 1024, smem>>>(dL, n, dM, 96, ds);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    long long st[4]; cudaMemcpy(st, ds, 32, cudaMemcpyDeviceToHost);
    printf("n=%d  %.2f us/launch  cycles: load %lld  diag %lld  blockrows %lld  product %lld  err=%s\n", n, ms * 1000 / 20,
           st[0], st[1], st[2], st[3], cudaGetErrorString(cudaGetLastError()));
  }
}
