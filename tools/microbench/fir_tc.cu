// Microbenchmark + check of the tensor-core FIR building block (DESIGN.md §3,
// "FIR on tcgen05"): D[128 planes x 16 outputs] = Z[128 x K] * T[16 x K]^T with
// the data Z in TMEM (lane = plane, column = source sample) and the banded
// Toeplitz tap matrix T[o][k] = w[k - o] (K = 16 + 2R rounded up to 8) in SMEM,
// 3xTF32 (Z = Zhi + Zlo with Zhi = the raw FP32 bits, which the MMA truncates,
// and Zlo = Z - trunc(Z); T likewise).  Times STTM, MMA and LDTM per CTA.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1901_06112_b200/csrc fir_tc.cu -o fir_tc
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "nys_umma.cuh"
using namespace nys::umma;

constexpr int R = 15, T = 2 * R + 1, NOUT = 64, NSRC = NOUT + 2 * R, KW = 48;  // 16 + 30 -> 48
constexpr int NT = NOUT / 16;                                                   // N-tiles

__device__ __forceinline__ float trunc_tf32(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// one CTA = 128 threads (lane = plane); `reps` repetitions of (fill Z, MMA, drain D)
__global__ void k_fir(const float* Z, const float* w, float* out, int reps, int mode, long long* cyc) {
  __shared__ __align__(128) float Th[KW * 16], Tl[KW * 16];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < KW * 16; e += blockDim.x) {
    const int o = e / KW, k = e % KW, t = k - o;
    const float v = (t >= 0 && t < T) ? w[t] : 0.f;
    const float h = __uint_as_float(__float_as_uint(v) & 0xffffe000u);
    Th[kmajor_offset(o, k, 16)] = h;
    Tl[kmajor_offset(o, k, 16)] = v - h;
  }
  if (warp == 0) tmem_alloc(&tbase, 256);
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t zh = tbase, zl = tbase + 96, dcol = tbase + 192;  // Z hi: 96 cols, Z lo: 96, D: 64
  const uint32_t lb = (uint32_t)(32 * warp) << 16;
  const int p = 32 * warp + lane;
  long long t_st = 0, t_mma = 0, t_ld = 0;
  uint32_t phase = 0;
  float acc = 0.f;
  for (int it = 0; it < reps; ++it) {
    long long c0 = clock64();
    for (int s0 = 0; s0 < 96; s0 += 16) {
      float h[16], l[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int s = s0 + q;
        const float v = s < NSRC ? Z[(size_t)p * NSRC + s] * (1.f + 1e-7f * it) : 0.f;
        h[q] = v;                      // raw bits: the MMA reads them as TF32 (truncation)
        l[q] = v - trunc_tf32(v);
      }
      st_32x32b_x16(zh + lb + s0, h);
      st_32x32b_x16(zl + lb + s0, l);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    fence_before();
    __syncthreads();
    fence_after();
    long long c1 = clock64();
    if (tid == 0) {
      constexpr uint32_t id = idesc_tf32(128, 16);
      for (int j = 0; j < NT; ++j) {
        uint32_t acc1 = 0;
        for (int pass = 0; pass < 3; ++pass) {
          const uint32_t A = (pass == 1 ? zl : zh) + 16 * j;
          const float* B = pass == 2 ? Tl : Th;
          for (int kk = 0; kk < KW / 8; ++kk) {
            mma_tf32_ts(dcol + 16 * j, A + 8 * kk, desc_kmajor(B + kk * 8 * 16, 16 * 16, 128), id, acc1);
            acc1 = 1;
          }
        }
      }
      commit(&bar);
    }
    mbar_wait(&bar, phase);
    phase ^= 1u;
    fence_after();
    long long c2 = clock64();
    for (int j = 0; j < NT; ++j) {
      float v[16];
      ld_32x32b_x16(dcol + lb + 16 * j, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (it == 0 && mode == 0 && blockIdx.x == 0)
        for (int q = 0; q < 16; ++q) out[(size_t)p * NOUT + 16 * j + q] = v[q];
      acc += v[0];
    }
    fence_before();
    __syncthreads();
    fence_after();
    long long c3 = clock64();
    t_st += c1 - c0;
    t_mma += c2 - c1;
    t_ld += c3 - c2;
  }
  if (tid == 0 && blockIdx.x == 0) {
    cyc[0] = t_st / reps;
    cyc[1] = t_mma / reps;
    cyc[2] = t_ld / reps;
  }
  if (acc == 12345.f) out[0] = acc;
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 256);
}


// MMA issue-rate probe: `nmma` back-to-back tf32 MMAs, M = 128, N = NN, A in TMEM (ss = 0) or
// SMEM (ss = 1), rotating over `nd` independent accumulators
template <int NN>
__global__ void k_rate(int nmma, long long* cyc, int nd, int ss) {
  __shared__ __align__(128) float Bs[NN * 8 * 4];
  __shared__ __align__(128) float As[128 * 8 * 4];
  for (int e = threadIdx.x; e < 128 * 8 * 4; e += blockDim.x) As[e] = 0.002f * (e % 5);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < NN * 8 * 4; e += blockDim.x) Bs[e] = 0.001f * (e % 7);
  if (warp == 0) tmem_alloc(&tbase, 256);
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  if (tid == 0) {
    const uint32_t id = idesc_tf32(128, NN);
    const uint64_t db = desc_kmajor(Bs, NN * 16, 128);
    const uint32_t a = tbase + 128, d = tbase;
    const uint64_t da = desc_kmajor(As, 128 * 16, 128);
    long long c0 = clock64();
    if (ss)
      for (int i = 0; i < nmma; ++i) mma_tf32_ss(d + (uint32_t)((i % nd) * NN), da, db, id, i >= nd);
    else
      for (int i = 0; i < nmma; ++i) mma_tf32_ts(d + (uint32_t)((i % nd) * NN), a + 8 * (i & 7), db, id, i >= nd);
    commit(&bar);
    mbar_wait(&bar, 0);
    long long c1 = clock64();
    cyc[0] = (c1 - c0);
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 256);
}

// unrolled issue: 64 MMAs in straight-line code per issuing warp; `nw` warps issue concurrently,
// each to its own accumulator (D columns 64 w .. ) with A in TMEM
template <int NN>
__global__ void k_rate2(long long* cyc, int nw) {
  __shared__ __align__(128) float Bs[NN * 8 * 4];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < NN * 8 * 4; e += blockDim.x) Bs[e] = 0.001f * (e % 7);
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (tid < 4) mbar_init(&bar[tid], 1);
  asm volatile("fence.mbarrier_init.release.cluster;");
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  long long c0 = clock64();
  if ((warp < nw || (nw < 0 && warp == 0)) && lane == 0) {
    const uint32_t id = idesc_tf32(128, NN);
    const uint64_t db = desc_kmajor(Bs, NN * 16, 128);
    const uint32_t a = tbase + 384, d = tbase + (uint32_t)(warp * 64);
    if (nw < 0) {  // one warp rotating over 4 accumulators (N <= 16: columns 16 k ..)
#pragma unroll
      for (int i = 0; i < 64; ++i) mma_tf32_ts(tbase + (uint32_t)(16 * (i & 3)), a + 8 * ((i >> 2) & 7), db, id, i >= 4 ? 1u : 0u);
    } else {
      mma_tf32_ts(d, a, db, id, 0u);
#pragma unroll
      for (int i = 1; i < 64; ++i) mma_tf32_ts(d, a + 8 * (i & 7), db, id, 1u);
    }
    commit(&bar[warp]);
    mbar_wait(&bar[warp], 0);
  }
  __syncthreads();
  long long c1 = clock64();
  if (tid == 0) cyc[0] = c1 - c0;
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

int main() {
  std::vector<float> Z(128 * NSRC), w(T), out(128 * NOUT);
  srand(1);
  for (auto& v : Z) v = (float)(rand() / (double)RAND_MAX * 2 - 1) * (float)(rand() % 7 + 1);
  for (int t = 0; t < T; ++t) w[t] = (float)std::exp(-(double)(t - R) * (t - R) / 50.0);
  float *dZ, *dw, *dout;
  long long* dc;
  cudaMalloc(&dZ, Z.size() * 4);
  cudaMalloc(&dw, w.size() * 4);
  cudaMalloc(&dout, out.size() * 4);
  cudaMalloc(&dc, 64);
  cudaMemcpy(dZ, Z.data(), Z.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dw, w.data(), w.size() * 4, cudaMemcpyHostToDevice);
  k_fir<<<1, 128>>>(dZ, dw, dout, 1, 0, dc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
  double maxrel = 0, maxabs = 0;
  for (int p = 0; p < 128; ++p)
    for (int o = 0; o < NOUT; ++o) {
      double ref = 0, mag = 0;
      for (int t = 0; t < T; ++t) {
        ref += (double)w[t] * Z[p * NSRC + o + t];
        mag += std::fabs((double)w[t] * Z[p * NSRC + o + t]);
      }
      const double d = std::fabs(out[p * NOUT + o] - ref);
      maxabs = std::max(maxabs, d);
      maxrel = std::max(maxrel, d / mag);
    }
  printf("check: max |err| %.3e, max |err| / sum|terms| %.3e (FP32 eps 6e-8)\n", maxabs, maxrel);

  {
    long long* dc2;
    cudaMalloc(&dc2, 16);
    long long h;
    const int nm = 720;
#define RATE(NN, ND, SS)                                                             \
  k_rate<NN><<<1, 128>>>(nm, dc2, ND, SS);                                           \
  cudaDeviceSynchronize();                                                           \
  cudaMemcpy(&h, dc2, 8, cudaMemcpyDeviceToHost);                                    \
  printf("N=%3d acc=%d %s: %.1f cycles per MMA (floor %d)\n", NN, ND, SS ? "SS" : "TS", (double)h / nm, 128 * NN / 256);
#define RATE2(NN, NW)                                                                \
  k_rate2<NN><<<1, 128>>>(dc2, NW);                                                  \
  cudaDeviceSynchronize();                                                           \
  cudaMemcpy(&h, dc2, 8, cudaMemcpyDeviceToHost);                                    \
  printf("unrolled N=%3d warps=%d: %.1f cycles per MMA per warp (%d MMAs/warp)\n", NN, NW, (double)h / 64, 64);
    RATE2(16, -1) RATE2(16, 1) RATE2(16, 2) RATE2(16, 4) RATE2(32, 1) RATE2(64, 1) RATE2(64, 2) RATE2(64, 4) RATE2(128, 1) RATE2(128, 2)
    RATE(16, 1, 0) RATE(16, 2, 0) RATE(16, 4, 0) RATE(16, 8, 0) RATE(32, 4, 0) RATE(64, 1, 0) RATE(64, 2, 0)
    RATE(128, 1, 0) RATE(16, 1, 1) RATE(16, 4, 1) RATE(64, 1, 1) RATE(64, 2, 1)
  }
  long long c[3];
  for (int grid : {1, 148, 296}) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int reps = 200;
    cudaEventRecord(a);
    k_fir<<<grid, 128>>>(dZ, dw, dout, reps, 1, dc);
    cudaEventRecord(b);
    cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaMemcpy(c, dc, 24, cudaMemcpyDeviceToHost);
    const double outs = (double)grid * reps * 128 * NOUT;
    printf("grid %d: %.3f ms, %.1f G plane-outputs/s; per rep cycles: fill %lld, mma %lld (floor %d), drain %lld\n",
           grid, ms, outs / ms / 1e6, c[0], c[1], NT * 3 * (KW / 8) * 8, c[2]);
  }
  return 0;
}
