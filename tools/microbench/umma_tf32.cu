// Standalone check of the tcgen05 kind::tf32 3xTF32 product used by K2:
// D[128 x N] = A[128 x K] * B[N x K]^T, operands K-major/no-swizzle in SMEM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1901_06112_b200/csrc umma_tf32.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "nys_umma.cuh"
using namespace nys::umma;

template <int K, int N>
__global__ void k_test(const float* A, const float* B, float* D, int split, int swap) {
  extern __shared__ __align__(1024) float sm[];
  float* Ah = sm;               // 128 x K
  float* Al = Ah + 128 * K;
  float* Bh = Al + 128 * K;     // N x K
  float* Bl = Bh + N * K;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < 128 * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    const float v = A[e], h = to_tf32(v);
    Ah[kmajor_offset(r, k, 128)] = h;
    Al[kmajor_offset(r, k, 128)] = to_tf32(v - h);
  }
  for (int e = tid; e < N * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    const float v = B[e], h = to_tf32(v);
    Bh[kmajor_offset(r, k, N)] = h;
    Bl[kmajor_offset(r, k, N)] = to_tf32(v - h);
  }
  if (warp == 0) tmem_alloc(&tbase, 128);
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tm = tbase;
  if (tid == 0) {
    constexpr uint32_t id = idesc_tf32(128, N);
    const uint32_t lboA = swap ? 128 : 128 * 16, sboA = swap ? 128 * 16 : 128;
    const uint32_t lboB = swap ? 128 : N * 16, sboB = swap ? N * 16 : 128;
    int first = 1;
    for (int pass = 0; pass < (split ? 3 : 1); ++pass) {
      const float* a = pass == 2 ? Al : Ah;
      const float* b = pass == 1 ? Bl : Bh;
      for (int kk = 0; kk < K / 8; ++kk) {
        const uint64_t da = desc_kmajor(a + kk * 2 * 128 * 4, lboA, sboA);
        const uint64_t db = desc_kmajor(b + kk * 2 * N * 4, lboB, sboB);
        mma_tf32_ss(tm, da, db, id, first ? 0u : 1u);
        first = 0;
      }
    }
    commit(&bar);
  }
  mbar_wait(&bar, 0);
  fence_after();
  // 4 warps: warp w reads lanes 32w..32w+31
  for (int c = 0; c < N; c += 8) {
    float v[8];
    ld_32x32b_x8(tm + ((uint32_t)(32 * warp) << 16) + c, v);
    ld_wait();
    for (int q = 0; q < 8; ++q) D[(32 * warp + lane) * N + c + q] = v[q];
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 128);
}

// A from TMEM (tcgen05.st), B from SMEM
template <int K, int N>
__global__ void k_test_ts(const float* A, const float* B, float* D) {
  extern __shared__ __align__(1024) float sm[];
  float* Bh = sm;
  float* Bl = Bh + N * K;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < N * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    const float v = B[e], h = to_tf32(v);
    Bh[kmajor_offset(r, k, N)] = h;
    Bl[kmajor_offset(r, k, N)] = to_tf32(v - h);
  }
  if (warp == 0) tmem_alloc(&tbase, 256);
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tm = tbase, ta = tm + 128;  // D cols [0,N), A_hi [128,128+K), A_lo [128+K, 128+2K)
  {
    const int r = 32 * warp + lane;
    const uint32_t lanebase = (uint32_t)(32 * warp) << 16;
    for (int j0 = 0; j0 < K; j0 += 4) {
      float h[4], l[4];
      for (int e = 0; e < 4; ++e) { const float v = A[r * K + j0 + e]; h[e] = to_tf32(v); l[e] = to_tf32(v - h[e]); }
      st_32x32b_x4(ta + lanebase + j0, h[0], h[1], h[2], h[3]);
      st_32x32b_x4(ta + lanebase + K + j0, l[0], l[1], l[2], l[3]);
    }
    st_wait();
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (tid == 0) {
    constexpr uint32_t id = idesc_tf32(128, N);
    int first = 1;
    for (int pass = 0; pass < 3; ++pass) {
      const uint32_t a = ta + (pass == 2 ? K : 0);
      const float* b = pass == 1 ? Bl : Bh;
      for (int kk = 0; kk < K / 8; ++kk) {
        const uint64_t db = desc_kmajor(b + kk * 2 * N * 4, N * 16, 128);
        mma_tf32_ts(tm, a + kk * 8, db, id, first ? 0u : 1u);
        first = 0;
      }
    }
    commit(&bar);
  }
  mbar_wait(&bar, 0);
  fence_after();
  for (int c = 0; c < N; c += 8) {
    float v[8];
    ld_32x32b_x8(tm + ((uint32_t)(32 * warp) << 16) + c, v);
    ld_wait();
    for (int q = 0; q < 8; ++q) D[(32 * warp + lane) * N + c + q] = v[q];
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 256);
}

int main() {
  constexpr int K = 64, N = 80;
  std::vector<float> A(128 * K), B(N * K), D(128 * N);
  srand(1);
  for (auto& x : A) x = (float)rand() / RAND_MAX;
  for (auto& x : B) x = ((float)rand() / RAND_MAX - 0.5f) * 1000.f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = (2 * 128 * K + 2 * N * K) * 4;
  cudaFuncSetAttribute(k_test<K, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int rc = 0;
  for (int swap = 0; swap < 1; ++swap)
    for (int split = 0; split < 2; ++split) {
      cudaMemset(dD, 0, D.size() * 4);
      k_test<K, N><<<1, 128, smem>>>(dA, dB, dD, split, swap);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("swap=%d split=%d: %s\n", swap, split, cudaGetErrorString(e)); return 1; }
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      double maxerr = 0, maxref = 0;
      for (int r = 0; r < 128; ++r)
        for (int c = 0; c < N; ++c) {
          double ref = 0;
          for (int k = 0; k < K; ++k) ref += (double)A[r * K + k] * B[c * K + k];
          maxerr = fmax(maxerr, fabs(ref - D[r * N + c]));
          maxref = fmax(maxref, fabs(ref));
        }
      printf("swap=%d split=%d maxerr=%.3e rel=%.3e\n", swap, split, maxerr, maxerr / maxref);
    }
  {
    cudaMemset(dD, 0, D.size() * 4);
    const int smem2 = 2 * N * K * 4;
    cudaFuncSetAttribute(k_test_ts<K, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
    k_test_ts<K, N><<<1, 128, smem2>>>(dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("ts: %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int r = 0; r < 128; ++r)
      for (int c = 0; c < N; ++c) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)A[r * K + k] * B[c * K + k];
        maxerr = fmax(maxerr, fabs(ref - D[r * N + c]));
        maxref = fmax(maxref, fabs(ref));
      }
    printf("ts 3xtf32 maxerr=%.3e rel=%.3e\n", maxerr, maxerr / maxref);
  }
  return rc;
}
