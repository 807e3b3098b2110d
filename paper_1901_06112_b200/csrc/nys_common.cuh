// Shared helpers for the sm_100a kernels of the Nystrom filter hot path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/nysfilter_b200.h"

#define NYS_MAX_TAPS (2 * NYS_MAX_RADIUS + 1)

#define NYS_CUDA_TRY(expr)                                   \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) return NYS_ECUDA + (int)_e;       \
  } while (0)

#define NYS_LAUNCH_CHECK() NYS_CUDA_TRY(cudaGetLastError())

namespace nys {

// number of kernels this library has launched (host-side, relaxed atomic);
// exported as nys_kernel_launches() so benchmarks can report their launches
unsigned long long* launch_counter();
inline void count_launch() { __atomic_add_fetch(launch_counter(), 1ull, __ATOMIC_RELAXED); }

__host__ __device__ __forceinline__ int clampi(int v, int lo, int hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// exp(-d2/(2 theta^2)) evaluated as exp2(d2 * k2) with k2 = -log2(e)/(2 theta^2):
// one FMUL + MUFU.EX2 (ex2.approx.ftz has ~2 ulp error, well inside the 1e-4 budget)
__device__ __forceinline__ float range_kernel(float d2, float k2) { return exp2f(d2 * k2); }
// one MUFU.EX2: exp2f adds a range fix-up (FSETP + two predicated FMULs) for results below
// 2^-126, which flush to zero here -- features that small are zero to the filter
__device__ __forceinline__ float range_kernel_fast(float d2, float k2) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(d2 * k2));
  return y;
}

// deterministic warp sums
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace nys
