// Lloyd assignment for high-dimensional guides on the 5th-generation tensor
// cores (BASELINE north_star (1): "tcgen05 3xTF32-split distance GEMM only for
// d >= 16 if ncu shows it wins").
//
// Reference region replaced: landmarks.py:37-57 (_assign, the loop form), with
// the labels of the FP32 differenced search the rest of the B200 k-means uses
// (first index on ties).  Per tile of 128 points:
//   1. every thread stores its point's coordinates, split x = x_hi + x_lo into
//      TF32 pairs, into the A operand in TMEM (lane = point);
//   2. one thread issues 3 x K/8 tcgen05.mma kind::tf32 (A from TMEM, centroids
//      as B from shared memory): dot = x_hi c_hi + x_lo c_hi + x_hi c_lo, FP32
//      accumulation in TMEM;
//   3. epilogue: approx_j = |x|^2 + |c_j|^2 - 2 dot_j; every centroid within
//      2 delta of the smallest approx is re-checked with the exact FP32
//      difference form, in ascending j with strict '<'.  delta bounds
//      |approx_j - d2_fp32(x, c_j)| (3xTF32 products, TF32 accumulation, FP32
//      norms) with a 10x margin, so no other centroid can reach the minimum:
//      the labels equal the full FP32 search's.
// Sums, counts, objective and changed count per block exactly as k_assign
// (deterministic warp butterflies), so the step-wise Lloyd loop
// (k_reduce / k_finalize / k_repair) consumes them unchanged.
//
// Opt-in (NYS_KM_TC=1): measured on cfg 3 (rho 27, m0 64) at 1.0 ms per
// iteration against 0.34 ms for the bounded cooperative kernel -- the full
// per-iteration FP64 warp-butterfly sums of every point (45 % of the stall
// samples, profiles/r1_cfg3_assign_tc_ncu.md) and one 128-point tile in flight
// per CTA dominate; the distance GEMM itself is cheap.  The cooperative kernel
// keeps its exact changed-point deltas and Hamerly bounds.
#include "nys_kmeans_dev.cuh"
#include "nys_umma.cuh"

namespace nys {

constexpr int KTC_THREADS = 128;  // = UMMA M = TMEM lanes: one point per thread
constexpr int KTC_TMEM_COLS = 256;

template <int GR>
__global__ void __launch_bounds__(KTC_THREADS, 1) k_assign_tc(const float* __restrict__ pts, long long ps, long long m,
                                                              int rho, const float* __restrict__ Cf, int m0,
                                                              int* __restrict__ labels, int first,
                                                              double* __restrict__ part, int S, const KState* st,
                                                              int KU, int NU) {
  extern __shared__ __align__(128) double dsm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  __shared__ float ccmax_sh;
  if (st && st->converged) return;  // uniform: the step-wise loop keeps launching after convergence
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int slots = m0 * (rho + 1);
  double* wacc = dsm;                                                         // 4 x slots
  float* Bh = reinterpret_cast<float*>(dsm + ((4 * (size_t)slots + 15) & ~(size_t)15));  // NU x KU (128 B aligned)
  float* Bl = Bh + (size_t)NU * KU;
  float* Cs = Bl + (size_t)NU * KU;                                           // m0 x rho (exact re-check)
  float* cc = Cs + (size_t)m0 * rho;                                          // m0: |c_j|^2
  for (int k = tid; k < 4 * slots; k += KTC_THREADS) wacc[k] = 0.0;
  for (int k = tid; k < NU * KU; k += KTC_THREADS) {
    const int j = k / KU, d = k - j * KU;
    const float v = (j < m0 && d < rho) ? Cf[(size_t)j * rho + d] : 0.f;
    const float h = umma::to_tf32(v);
    const int o = umma::kmajor_offset(j, d, NU);
    Bh[o] = h;
    Bl[o] = umma::to_tf32(v - h);
  }
  for (int k = tid; k < m0 * rho; k += KTC_THREADS) Cs[k] = Cf[k];
  for (int j = tid; j < m0; j += KTC_THREADS) {
    float s = 0.f;
    for (int d = 0; d < rho; ++d) s = fmaf(Cf[(size_t)j * rho + d], Cf[(size_t)j * rho + d], s);
    cc[j] = s;
  }
  if (w == 0) umma::tmem_alloc(&tmem_base, KTC_TMEM_COLS);
  if (tid == 0) {
    umma::mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  umma::fence_proxy_async();  // B operand: generic-proxy writes -> tensor core
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  if (tid == 0) {
    float mx = 0.f;
    for (int j = 0; j < m0; ++j) mx = fmaxf(mx, cc[j]);
    ccmax_sh = mx;
  }
  const uint32_t dcol = tmem_base, a_hi = tmem_base + (uint32_t)((NU + 31) & ~31), a_lo = a_hi + (uint32_t)((KU + 31) & ~31);
  const uint32_t lane_base = (uint32_t)(32 * w) << 16;
  const uint32_t idesc = umma::idesc_tf32(KTC_THREADS, NU);
  const uint32_t lbo_b = (uint32_t)NU * 16;
  double* my = wacc + (size_t)w * slots;
  double near_sum = 0.0;
  long long changed = 0;
  const long long chunk = ceil_div(m, (long long)gridDim.x);
  const long long lo = blockIdx.x * chunk, hi = min(m, lo + chunk);
  uint32_t phase = 0;
  __syncthreads();
  const float ccmax = ccmax_sh;
  for (long long base = lo; base < hi; base += KTC_THREADS) {
    const long long i = base + tid;
    const bool valid = i < hi;
    float x[GR];
#pragma unroll
    for (int d = 0; d < GR; ++d) x[d] = (valid && d < rho) ? __ldg(pts + d * ps + i) : 0.f;
    float xx = 0.f;
#pragma unroll
    for (int d = 0; d < GR; ++d)
      if (d < rho) xx = fmaf(x[d], x[d], xx);
    // 1. A operand (this thread's TMEM lane): x_hi, x_lo in K chunks of 4 columns
#pragma unroll
    for (int c4 = 0; c4 < (GR + 3) / 4; ++c4) {
      if (4 * c4 < KU) {
        float h[4], l[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int d = 4 * c4 + e;
          const float v = d < GR ? x[d < GR ? d : 0] : 0.f;
          h[e] = umma::to_tf32(v);
          l[e] = umma::to_tf32(v - h[e]);
        }
        umma::st_32x32b_x4(a_hi + lane_base + (uint32_t)(4 * c4), h[0], h[1], h[2], h[3]);
        umma::st_32x32b_x4(a_lo + lane_base + (uint32_t)(4 * c4), l[0], l[1], l[2], l[3]);
      }
    }
    umma::st_wait();
    umma::fence_before();
    __syncthreads();
    // 2. dot products on the tensor core: 3xTF32 split
    if (tid == 0) {
      umma::fence_after();
      uint32_t acc = 0;
#pragma unroll 1
      for (int pass = 0; pass < 3; ++pass) {
        const uint32_t A = pass == 1 ? a_lo : a_hi;
        const float* B = pass == 2 ? Bl : Bh;
#pragma unroll 1
        for (int kk = 0; kk < KU / 8; ++kk) {
          umma::mma_tf32_ts(dcol, A + (uint32_t)(8 * kk), umma::desc_kmajor(B + kk * 8 * NU, lbo_b, 128), idesc, acc);
          acc = 1;
        }
      }
      umma::commit(&bar);
    }
    umma::mbar_wait(&bar, phase);
    phase ^= 1u;
    umma::fence_after();
    // 3. smallest approximate distance, then exact re-check of the near candidates
    float mn = INFINITY;
    for (int c8 = 0; c8 < NU / 8; ++c8) {
      float v[8];
      umma::ld_32x32b_x8(dcol + lane_base + (uint32_t)(8 * c8), v);
      umma::ld_wait();
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int j = 8 * c8 + e;
        if (j < m0) mn = fminf(mn, xx + cc[j] - 2.f * v[e]);
      }
    }
    const float lim = mn + 2.f * (1e-4f * (xx + ccmax) + 1e-30f);
    float best = INFINITY;
    int arg = 0;
    for (int c8 = 0; c8 < NU / 8; ++c8) {
      float v[8];
      umma::ld_32x32b_x8(dcol + lane_base + (uint32_t)(8 * c8), v);
      umma::ld_wait();
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int j = 8 * c8 + e;
        if (j < m0 && xx + cc[j] - 2.f * v[e] <= lim) {
          float d2 = 0.f;
#pragma unroll
          for (int d = 0; d < GR; ++d)
            if (d < rho) {
              const float t = x[d] - Cs[j * rho + d];
              d2 = fmaf(t, t, d2);
            }
          if (d2 < best) {  // strict, ascending j: first index wins ties (np.argmin)
            best = d2;
            arg = j;
          }
        }
      }
    }
    if (valid) {
      near_sum += (double)best;
      const int old = labels[i];
      if (first || old != arg) ++changed;
      labels[i] = arg;
    }
    unsigned rem = __ballot_sync(0xffffffffu, valid);
    while (rem) {
      const int leader = __ffs(rem) - 1;
      const int Lb = __shfl_sync(0xffffffffu, arg, leader);
      const unsigned grp = __ballot_sync(0xffffffffu, valid && arg == Lb);
      const bool in = (grp >> lane) & 1u;
#pragma unroll
      for (int d = 0; d < GR; ++d)
        if (d < rho) {
          const double s = warp_sum(in ? (double)x[d] : 0.0);
          if (lane == 0) my[Lb * (rho + 1) + d] += s;
        }
      if (lane == 0) my[Lb * (rho + 1) + rho] += (double)__popc(grp);
      rem &= ~grp;
    }
    umma::fence_before();
    __syncthreads();  // every lane's TMEM reads are done before the next tile's MMAs
  }
  near_sum = warp_sum(near_sum);
  const double ch = warp_sum((double)changed);
  __shared__ double extra[2][4];
  if (lane == 0) {
    extra[0][w] = near_sum;
    extra[1][w] = ch;
  }
  umma::fence_before();
  __syncthreads();
  if (w == 0) umma::tmem_dealloc(tmem_base, KTC_TMEM_COLS);
  double* out = part + (size_t)blockIdx.x * S;
  for (int k = tid; k < slots; k += KTC_THREADS) {
    double s = 0.0;
    for (int q = 0; q < 4; ++q) s += wacc[(size_t)q * slots + k];
    out[k] = s;
  }
  if (tid == 0) {
    double a = 0.0, b = 0.0;
    for (int q = 0; q < 4; ++q) {
      a += extra[0][q];
      b += extra[1][q];
    }
    out[slots] = a;
    out[slots + 1] = b;
  }
}

int launch_assign_tc(const float* pts, long long ps, long long m, int rho, const float* Cf, int m0, int* labels,
                     int first, double* part, int nb, int S, const KState* st, cudaStream_t s) {
  const int KU = (int)ceil_div(rho, 8) * 8, NU = (int)ceil_div(m0, 16) * 16;
  if (KU > 64 || NU > 128 || ((NU + 31) & ~31) + 2 * ((KU + 31) & ~31) > KTC_TMEM_COLS) return NYS_EUNSUPPORTED;
  const int slots = m0 * (rho + 1);
  const size_t smem = (((size_t)4 * slots + 15) & ~(size_t)15) * 8 + ((size_t)2 * NU * KU + (size_t)m0 * rho + m0) * 4;
  if (smem > 200 * 1024) return NYS_EUNSUPPORTED;
#define NYS_TC_CASE(G)                                                                                            \
  NYS_CUDA_TRY(cudaFuncSetAttribute(k_assign_tc<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));      \
  count_launch();                                                                                                 \
  k_assign_tc<G><<<nb, KTC_THREADS, smem, s>>>(pts, ps, m, rho, Cf, m0, labels, first, part, S, st, KU, NU);
  if (rho <= 16) {
    NYS_TC_CASE(16)
  } else if (rho <= 32) {
    NYS_TC_CASE(32)
  } else {
    NYS_TC_CASE(64)
  }
#undef NYS_TC_CASE
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

}  // namespace nys
