// Microbenchmark: FP32 FMA issue rate on sm_100a for the operand forms the FIR
// kernels can use (3-register, constant-bank weight, packed f32x2).
#include <cstdio>
#include <cuda_runtime.h>

__constant__ float cw[64];

template <int NACC>
__global__ void k_reg3(float* out, float a0, float b0, int iters) {
  float acc[NACC], x[NACC];
#pragma unroll
  for (int k = 0; k < NACC; ++k) { acc[k] = threadIdx.x * 1e-3f + k; x[k] = a0 + k * 1e-4f; }
  float b = b0 + threadIdx.x * 1e-7f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = fmaf(x[k], b, acc[k]);
    b = b * 0.9999f;
  }
  float s = 0; for (int k = 0; k < NACC; ++k) s += acc[k];
  if (s == 12345.f) out[threadIdx.x] = s;
}

// weight from constant bank with compile-time offset (FFMA R, R, c[..], R)
template <int NACC>
__global__ void k_const(float* out, float a0, int iters) {
  float acc[NACC], x[NACC];
#pragma unroll
  for (int k = 0; k < NACC; ++k) { acc[k] = threadIdx.x * 1e-3f + k; x[k] = a0 + k * 1e-4f + threadIdx.x; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 16; ++t) {
#pragma unroll
      for (int k = 0; k < NACC; ++k) acc[k] = fmaf(x[(k + t) % NACC], cw[t], acc[k]);
    }
  }
  float s = 0; for (int k = 0; k < NACC; ++k) s += acc[k];
  if (s == 12345.f) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void k_f32x2(float* out, float a0, float b0, int iters) {
  static_assert(NACC % 2 == 0, "");
  unsigned long long acc[NACC / 2], x[NACC / 2];
#pragma unroll
  for (int k = 0; k < NACC / 2; ++k) {
    float2 t = make_float2(threadIdx.x * 1e-3f + k, k + 0.5f);
    acc[k] = *reinterpret_cast<unsigned long long*>(&t);
    float2 u = make_float2(a0 + k * 1e-4f, a0 - k * 1e-4f);
    x[k] = *reinterpret_cast<unsigned long long*>(&u);
  }
  float bb = b0 + threadIdx.x * 1e-7f;
  for (int it = 0; it < iters; ++it) {
    float2 bt = make_float2(bb, bb);
    unsigned long long b = *reinterpret_cast<unsigned long long*>(&bt);
#pragma unroll
    for (int k = 0; k < NACC / 2; ++k)
      asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[k]) : "l"(x[k]), "l"(b));
    bb = bb * 0.9999f;
  }
  float s = 0;
  for (int k = 0; k < NACC / 2; ++k) { float2 t = *reinterpret_cast<float2*>(&acc[k]); s += t.x + t.y; }
  if (s == 12345.f) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void k_dfma(double* out, double a0, double b0, int iters) {
  double acc[NACC], x[NACC];
#pragma unroll
  for (int k = 0; k < NACC; ++k) { acc[k] = threadIdx.x * 1e-3 + k; x[k] = a0 + k * 1e-4; }
  double b = b0 + threadIdx.x * 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = fma(x[k], b, acc[k]);
    b = b * 0.9999;
  }
  double s = 0; for (int k = 0; k < NACC; ++k) s += acc[k];
  if (s == 12345.0) out[threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("%s SMs=%d clk=%d kHz\n", p.name, p.multiProcessorCount, clk);
  float* out; cudaMalloc(&out, 4096 * 4);
  float w[64]; for (int i = 0; i < 64; ++i) w[i] = 0.5f + i * 1e-3f;
  cudaMemcpyToSymbol(cw, w, sizeof(w));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = p.multiProcessorCount * 4, threads = 256, iters = 4096;
  auto run = [&](const char* name, auto launch, double fma_per_thread) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    double fmas = fma_per_thread * blocks * threads;
    double per_clk_sm = fmas / (ms * 1e-3) / p.multiProcessorCount / (clk * 1e3);
    printf("%-10s %.3f ms  %.2f TFMA/s  %.1f FMA/clk/SM(@max clk)\n", name, ms, fmas / ms / 1e9, per_clk_sm);
  };
  run("reg3", [&] { k_reg3<16><<<blocks, threads>>>(out, 1.f, 0.5f, iters); }, 16.0 * iters);
  run("const", [&] { k_const<16><<<blocks, threads>>>(out, 1.f, iters / 16); }, 16.0 * 16 * (iters / 16));
  run("f32x2", [&] { k_f32x2<16><<<blocks, threads>>>(out, 1.f, 0.5f, iters); }, 16.0 * iters);
  double* dout; cudaMalloc(&dout, 4096 * 8);
  run("dfma", [&] { k_dfma<16><<<blocks, threads>>>(dout, 1.0, 0.5, iters); }, 16.0 * iters);
  cudaError_t err = cudaGetLastError(); printf("err=%s\n", cudaGetErrorString(err));
  return 0;
}
