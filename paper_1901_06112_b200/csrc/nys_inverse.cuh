// M = A^{-1} = X^T X with X = L^{-1}, A = L L^T (the host's Cholesky factor, FP64),
// for m0 <= 64, in one CTA of 1024 threads (included by nys_filter.cu and by
// tools/microbench/inv_phases.cu).
//
// The factor is padded to 64 x 64 with an identity tail (which leaves the
// leading n x n block of X unchanged and adds only zero terms to X^T X):
//   1. the 8 diagonal 8 x 8 blocks are inverted by forward substitution with
//      reciprocal pivots (one thread per block column);
//   2. three doubling levels b = 8, 16, 32 assemble X from 2 x 2 block
//      inverses, X21 = -X22 (L21 X11): two b x b products per block pair, all
//      pairs of a level at once (two barriers per level);
//   3. M[i][j] = sum_k X[k][i] X[k][j] in 4 x 4 register tiles whose k range
//      starts at the warp's (uniform) first nonzero row.
// Every loop is warp-uniform (lanes never diverge on the triangle: the zero
// upper triangle supplies exact zero terms), chains are <= 8 FMAs deep with four
// accumulators, and shared-memory rows are padded to 66 doubles.
// Optionally the kernel first copies the workspace-constant image from mapped
// pinned memory (the in-stream plan's staging buffer) into the workspace and
// reads the factor from there, replacing a host->device copy.
#pragma once

namespace nys {

#ifdef NYS_INV_STAMPS  // phase timing in tools/microbench/inv_phases.cu
__device__ long long g_inv_stamps[8];
#define NYS_INV_STAMP(k) \
  if (threadIdx.x == 0) g_inv_stamps[k] = clock64()
#else
#define NYS_INV_STAMP(k)
#endif

constexpr int kInvN = 64;
constexpr int kInvLd = 66;  // padded row stride (doubles)
constexpr size_t kInvSmemBytes = 3 * (size_t)kInvN * kInvLd * sizeof(double) + kInvN * sizeof(double);

// one doubling level: for every block pair (o = 2 B p) T = L21 X11, then X21 = -X22 T.
// All loops run over the whole block, warp-uniformly: X11 / X22 are lower
// triangular and X starts zeroed, so the extra terms are exact zeros.
template <int B>
__device__ __forceinline__ void inv_level(const double* __restrict__ Ls, double* __restrict__ X, double* __restrict__ T) {
  constexpr int kPer = B * B, kTotal = (kInvN / (2 * B)) * kPer;  // 32 B outputs
  for (int e = threadIdx.x; e < kTotal; e += blockDim.x) {
    const int p = e / kPer, rc = e % kPer, r = rc / B, c = rc % B, o = 2 * B * p;
    const double* l21 = Ls + (o + B + r) * kInvLd + o;  // row r of L21
    const double* x11 = X + o * kInvLd + o + c;         // column c of X11
    double t[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < B; ++k) t[k & 3] = fma(l21[k], x11[k * kInvLd], t[k & 3]);
    T[(o + B + r) * kInvLd + o + c] = (t[0] + t[1]) + (t[2] + t[3]);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < kTotal; e += blockDim.x) {
    const int p = e / kPer, rc = e % kPer, r = rc / B, c = rc % B, o = 2 * B * p;
    const double* x22 = X + (o + B + r) * kInvLd + o + B;  // row r of X22
    const double* tc = T + (o + B) * kInvLd + o + c;       // column c of T
    double t[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < B; ++k) t[k & 3] = fma(x22[k], tc[k * kInvLd], t[k & 3]);
    X[(o + B + r) * kInvLd + o + c] = -((t[0] + t[1]) + (t[2] + t[3]));
  }
  __syncthreads();
}

// Active gate (the in-stream plan): thread 0 polls a mapped host word until it reaches `seq`
// (acquire, system scope), bounded by 60 s of %globaltimer; everything after the barrier sees
// the host's writes that preceded the word.  A stream-level cuStreamWaitValue32 on the same
// word occasionally noticed a late write only milliseconds (once 130 ms) later.
// Returns (in every thread) whether the word arrived; on a timeout the caller marks the step
// failed (FilterStats::gate_timeout -> nys_filter_finish publishes a sentinel) instead of
// silently computing on a stale staging image.
__device__ __forceinline__ bool wait_host_word(const unsigned* gate, unsigned seq) {
  __shared__ int s_timed_out;
  if (threadIdx.x == 0) {
    s_timed_out = 0;
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      unsigned v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(gate) : "memory");
      if ((int)(v - seq) >= 0) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 60ull * 1000000000ull) {
        s_timed_out = 1;
        break;
      }
      __nanosleep(256);
    }
  }
  __syncthreads();
  return s_timed_out == 0;
}

// FilterStats as 32-bit words (nys_filter_common.cuh): reset for a new filter, and the
// gate-timeout mark
__device__ __forceinline__ void reset_filter_stats(unsigned* w, bool timed_out) {
  w[0] = 0x7f800000u;  // min|eta| = +inf
#pragma unroll
  for (int k = 1; k < 8; ++k) w[k] = 0u;
  w[6] = timed_out ? 1u : 0u;  // gate_timeout
}

// gate + statistics reset for the plans whose image carries M (m0 > 64)
__global__ void k_wait_gate(const unsigned* gate, unsigned seq, unsigned* stats) {
  const bool ok = wait_host_word(gate, seq);
  if (threadIdx.x == 0) reset_filter_stats(stats, !ok);
}

// The staging image (img_src) and the factor (Lg) may live in mapped pinned memory that the
// host writes while this kernel is already resident (before `done`): they are read with
// ordinary (not read-only-cache) loads after the gate's acquire.
__global__ void __launch_bounds__(1024) k_inverse_cholesky(const double* Lg, int n, float* __restrict__ MT,
                                                          int m0q, double* __restrict__ M64, const float4* img_src,
                                                          float4* __restrict__ img_dst, int img_f4,
                                                          unsigned* __restrict__ stats_reset,
                                                          const unsigned* gate = nullptr, unsigned seq = 0) {
  extern __shared__ double cs[];
  double* Ls = cs;                     // 64 x kInvLd
  double* X = Ls + kInvN * kInvLd;     // 64 x kInvLd, X = L^{-1}
  double* T = X + kInvN * kInvLd;      // 64 x kInvLd scratch (L21 X11 per block pair)
  double* rd = T + kInvN * kInvLd;     // 64 reciprocal pivots
  const int tid = threadIdx.x;  // blockDim.x == 1024
  const bool gate_ok = gate ? wait_host_word(gate, seq) : true;
  NYS_INV_STAMP(0);
  if (stats_reset && tid == 0) reset_filter_stats(stats_reset, !gate_ok);
  {
    // every load of a thread is issued before its first store: over PCIe (mapped pinned
    // memory) the round trips overlap instead of queueing
    float4 vi[3];
    double vl[4];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int k = q * 1024 + tid;
      if (img_src && k < img_f4) vi[q] = img_src[k];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = q * 1024 + tid, i = e >> 6, j = e & 63;
      vl[q] = (i < n && j < n) ? Lg[i * n + j] : (i == j ? 1.0 : 0.0);
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int k = q * 1024 + tid;
      if (img_src && k < img_f4) img_dst[k] = vi[q];
    }
    if (img_src)
      for (int k = 3 * 1024 + tid; k < img_f4; k += 1024) img_dst[k] = img_src[k];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = q * 1024 + tid, i = e >> 6, j = e & 63;
      Ls[i * kInvLd + j] = vl[q];
      X[i * kInvLd + j] = 0.0;
      if (i == j) rd[i] = 1.0 / vl[q];
    }
  }
  __syncthreads();
  NYS_INV_STAMP(1);
  // 1. diagonal 8 x 8 blocks: column c of block I
  if (tid < kInvN) {
    const int o = tid & ~7, c = tid & 7;
    double col[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      double t = (a == c) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < a; ++k) t = fma(-Ls[(o + a) * kInvLd + o + k], col[k], t);
      col[a] = (a < c) ? 0.0 : t * rd[o + a];
    }
#pragma unroll
    for (int a = 0; a < 8; ++a) X[(o + a) * kInvLd + o + c] = col[a];
  }
  __syncthreads();
  NYS_INV_STAMP(2);
  // 2. doubling levels
  inv_level<8>(Ls, X, T);
  inv_level<16>(Ls, X, T);
  inv_level<32>(Ls, X, T);
  NYS_INV_STAMP(3);
  // 3. M = X^T X in 4 x 4 tiles: warp w covers row tiles 2w, 2w+1 (uniform k start), lanes the
  //    16 column tiles; X[k][i] = 0 for k < i
  if (tid < 256) {
    const int ti = tid >> 4, tj = tid & 15, i = 4 * ti, j = 4 * tj;
    double m[4][4] = {};
    for (int k = 4 * (tid >> 5) * 2; k < kInvN; ++k) {
      const double2 a0 = *reinterpret_cast<const double2*>(X + k * kInvLd + i);
      const double2 a1 = *reinterpret_cast<const double2*>(X + k * kInvLd + i + 2);
      const double2 b0 = *reinterpret_cast<const double2*>(X + k * kInvLd + j);
      const double2 b1 = *reinterpret_cast<const double2*>(X + k * kInvLd + j + 2);
      const double av[4] = {a0.x, a0.y, a1.x, a1.y}, bv[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) m[u][v] = fma(av[u], bv[v], m[u][v]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (i + u < n && j + v < n) {
          MT[(size_t)(j + v) * m0q + i + u] = (float)m[u][v];
          if (M64) M64[(size_t)(i + u) * n + j + v] = m[u][v];  // FP64 copy for nys_filter_finish
        }
  }
#ifdef NYS_INV_STAMPS
  __syncthreads();
#endif
  NYS_INV_STAMP(4);
}

}  // namespace nys
