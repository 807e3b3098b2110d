// K2 on the 5th-generation tensor cores: features b, y = M b on tcgen05,
// horizontal pass.
//
// Same contract and output as k_feat_hpass (nys_hpass.cu; reference regions
// nystrom.py:43-79, 112-114, filters.py:228-230, spatial.py:194-209), with
// the [px x m0] x [m0 x (m0+1)] product moved from CUDA-core FMAs to
// tcgen05.mma kind::tf32.  TF32 alone loses the y-form's precision (y = M b
// cancels: DESIGN.md §3), so the product is the 3xTF32 split
//   y = M_hi b_hi + M_lo b_hi + M_hi b_lo,   x_hi = tf32(x), x_lo = tf32(x - x_hi)
// accumulated in FP32 in tensor memory, which matches FP32 FMA accuracy
// (tools/precision_tf32.py; tools/microbench/umma_tf32.cu).
//
// One tile = one virtual row x TW output columns, i.e. TW + 2R <= 128 source
// pixels = the 128 rows (TMEM lanes) of one UMMA M=128 tile:
//   1. all 256 threads: pixel s = tid % 128 evaluates b_j for half of the
//      landmarks and writes b_hi / b_lo into the K-major A operand (SMEM);
//   2. one thread issues 3 x K/8 tcgen05.mma into TMEM and commits to an
//      mbarrier; meanwhile the threads stage the tile's f rows;
//   3. tcgen05.ld drains the accumulator (lane = pixel, column = i) into the
//      y rows in SMEM (aliasing the dead A operand);
//   4. FIR items (4 planes x 16 columns) write the blocked plane buffer.
// The B operand (M and u0, split hi/lo) is built once per persistent CTA.
#include <cstdlib>

#include "nys_hpass.cuh"
#include "nys_umma.cuh"

namespace nys {

constexpr int K2T_THREADS = 256;
constexpr int K2T_PX = 128;  // UMMA M: source pixels per tile

__host__ __device__ inline int align32f(int v) { return (v + 31) & ~31; }

template <int RT, int GR>
__global__ void __launch_bounds__(K2T_THREADS, 2) k_feat_hpass_tc(const HArgs a) {
  extern __shared__ __align__(128) float sm[];
  __shared__ uint64_t mma_bar;
  __shared__ uint32_t tmem_base;
  const int R = RT > 0 ? RT : a.R;
  const int m0 = a.m0, m0q = a.m0q, n = a.n, rho = a.rho, rhop = a.rhop, W = a.W, H = a.H;
  const int NC = n + 1, L = m0 + 1, pitch = a.pitch, TW = a.TW;
  const int KU = a.ku, NU = a.nu;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  float* Cs = sm;                                  // m0 x rhop
  float* Bh = Cs + align32f(m0 * rhop);            // NU x KU, K-major core matrices
  float* Bl = Bh + NU * KU;
  float* Fs = Bl + NU * KU;                        // n x pitch
  float* U = Fs + align32f(n * pitch);             // A hi/lo (2 x 128 x KU) | y rows (m0q x pitch)
  float* Ah = U;
  float* Al = U + K2T_PX * KU;
  float* Ys = U;

  for (int k = tid; k < m0 * rhop; k += K2T_THREADS) Cs[k] = a.cst[k];
  {
    const float* MTg = a.cst + (size_t)m0 * rhop;  // MT[j][i] = M[i][j], MT[j][m0] = u0[j]
    for (int k = tid; k < NU * KU; k += K2T_THREADS) {
      const int i = k / KU, j = k - (k / KU) * KU;
      const float v = (i < m0q && j < m0) ? MTg[(size_t)j * m0q + i] : 0.f;
      const float h = umma::to_tf32(v);
      const int o = umma::kmajor_offset(i, j, NU);
      Bh[o] = h;
      Bl[o] = umma::to_tf32(v - h);
    }
  }
  if (warp == 0) umma::tmem_alloc(&tmem_base, (uint32_t)a.tcols);
  if (tid == 0) {
    umma::mbar_init(&mma_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = umma::idesc_tf32(K2T_PX, NU);

  const int ncols = TW + 2 * R;  // <= 128
  const int ncol4 = (ncols + 3) & ~3;
  const int nchunks = (NC + K2_CC - 1) / K2_CC;
  const int XG = TW / K2_XR;
  const int fir_items = L * nchunks * XG;
  const int ntiles = a.tiles_x * a.vrows;
  const int khalf = KU / 2;  // landmarks per feature thread (multiple of 4)

  uint32_t phase = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, phase ^= 1u) {
    const int vr = a.v0 + tile / a.tiles_x;  // virtual row
    const int x0 = (tile % a.tiles_x) * TW;
    const int row = clampi(clampi(vr, 0, H - 1), a.rlo, a.rhi - 1);
    __syncthreads();  // the previous tile's FIR is done with Ys (= A) and Fs
    // 1. features -> A operand (b_hi, b_lo), raw b planes for K3 when requested
    {
      const int s = tid & (K2T_PX - 1), h = tid >> 7;
      if (s < ncols && !(a.dbg & 1)) {
        const int xs = x0 - R + s;
        const int x = clampi(xs, 0, W - 1);
        float gv[GR];
#pragma unroll
        for (int dd = 0; dd < GR; ++dd)
          gv[dd] = dd < rho ? guide_at(a.g, a.gps, a.f, a.fps, a.gkind, dd, row, x, H, W) : 0.f;
        float* bdst = nullptr;
        if (a.bplanes && s >= R && s < R + TW && xs < ((W + 31) & ~31))
          bdst = a.hp + (long long)(vr - a.v0) * a.rs + (long long)(xs >> 5) * (a.npl * 32) +
                 (long long)(L * NC) * 32 + (xs & 31);
        for (int j0 = h * khalf; j0 < (h + 1) * khalf; j0 += 4) {
          float bv[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int j = j0 + e;
            float v = 0.f;
            if (j < m0) {
              const float4* cj = reinterpret_cast<const float4*>(Cs + (size_t)j * rhop);
              float d2 = 0.f;
#pragma unroll
              for (int d4 = 0; d4 < GR / 4; ++d4) {
                if (4 * d4 < rho) {
                  const float4 c4 = cj[d4];
                  const float t0 = gv[4 * d4] - c4.x, t1 = gv[4 * d4 + 1] - c4.y;
                  const float t2 = gv[4 * d4 + 2] - c4.z, t3 = gv[4 * d4 + 3] - c4.w;
                  d2 = fmaf(t0, t0, d2);
                  d2 = fmaf(t1, t1, d2);
                  d2 = fmaf(t2, t2, d2);
                  d2 = fmaf(t3, t3, d2);
                }
              }
              v = range_kernel(d2, a.k2);
              if (bdst) bdst[(size_t)j * 32] = v;
            }
            bv[e] = v;
          }
          float4 hi, lo;
          hi.x = umma::to_tf32(bv[0]);
          hi.y = umma::to_tf32(bv[1]);
          hi.z = umma::to_tf32(bv[2]);
          hi.w = umma::to_tf32(bv[3]);
          lo.x = umma::to_tf32(bv[0] - hi.x);
          lo.y = umma::to_tf32(bv[1] - hi.y);
          lo.z = umma::to_tf32(bv[2] - hi.z);
          lo.w = umma::to_tf32(bv[3] - hi.w);
          const int o = umma::kmajor_offset(s, j0, K2T_PX);
          *reinterpret_cast<float4*>(Ah + o) = hi;
          *reinterpret_cast<float4*>(Al + o) = lo;
        }
      }
    }
    umma::fence_proxy_async();  // generic-proxy SMEM writes -> visible to the tensor core
    __syncthreads();
    // 2. y = M b: 3 x K/8 MMAs (M=128, N=NU, K=8 each), one issuing thread
    if (tid == 0 && !(a.dbg & 2)) {
      umma::fence_after();
      const uint32_t lbo_a = K2T_PX * 16, lbo_b = (uint32_t)NU * 16;
      uint32_t acc = 0;
#pragma unroll 1
      for (int pass = 0; pass < 3; ++pass) {
        const float* A = pass == 2 ? Al : Ah;
        const float* B = pass == 1 ? Bl : Bh;
#pragma unroll 1
        for (int kk = 0; kk < KU / 8; ++kk) {
          const uint64_t da = umma::desc_kmajor(A + kk * 8 * K2T_PX, lbo_a, 128);
          const uint64_t db = umma::desc_kmajor(B + kk * 8 * NU, lbo_b, 128);
          umma::mma_tf32_ss(tmem, da, db, idesc, acc);
          acc = 1;
        }
      }
      umma::commit(&mma_bar);
    }
    // stage the tile's f rows while the tensor core runs
    for (int k = tid; k < n * ncol4; k += K2T_THREADS) {
      const int c = k / ncol4, s = k - c * ncol4;
      const int x = clampi(x0 - R + s, 0, W - 1);
      Fs[(size_t)c * pitch + s] = __ldg(a.f + (long long)c * a.fps + (long long)row * W + x);
    }
    if (!(a.dbg & 2)) {
      umma::mbar_wait(&mma_bar, phase);
      umma::fence_after();
      // 3. accumulator -> y rows: warp w drains TMEM lanes 32(w%4).. (its
      // sub-partition), warps w and w+4 take half of the columns each
      const int q = warp & 3, hh = warp >> 2;
      const int s = 32 * q + lane;
      const int nch = NU / 8, c0 = hh * (nch / 2), c1 = c0 + nch / 2;
      for (int c = c0; c < c1; ++c) {
        float v[8];
        umma::ld_32x32b_x8(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(8 * c), v);
        umma::ld_wait();
        if (s < ncols) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int i = 8 * c + e;
            if (i < L) Ys[(size_t)i * pitch + s] = v[e];
          }
        }
      }
    }
    umma::fence_before();
    __syncthreads();
    // 4. horizontal FIR of the (m0+1)(n+1) planes, blocked-layout stores
    for (int it = tid; it < fir_items; it += K2T_THREADS) {
      const int i = it % L;
      const int rest = it / L;
      const int ch = rest % nchunks;
      const int xg = rest / nchunks;
      const int xo = x0 + xg * K2_XR;
      if (xo >= W) continue;
      float acc[K2_CC][K2_XR];
      if (a.dbg & 4) {
#pragma unroll
        for (int cc = 0; cc < K2_CC; ++cc)
#pragma unroll
          for (int o = 0; o < K2_XR; ++o) acc[cc][o] = Ys[(size_t)i * pitch + o + cc];
      } else {
        hfir<RT>(a, Ys + (size_t)i * pitch + xg * K2_XR, Fs, pitch, xg * K2_XR, ch * K2_CC, acc);
      }
      if (a.dbg & 8) {
        if (acc[0][0] == 1234.5f) a.hp[0] = acc[1][1];
        continue;
      }
      float* dst0 = a.hp + (long long)(vr - a.v0) * a.rs + (long long)(xo >> 5) * (a.npl * 32) + (xo & 31);
#pragma unroll
      for (int cc = 0; cc < K2_CC; ++cc) {
        const int c = ch * K2_CC + cc;
        if (c < NC) {
          float* dst = dst0 + (i * NC + c) * 32;
#pragma unroll
          for (int q4 = 0; q4 < K2_XR / 4; ++q4)
            reinterpret_cast<float4*>(dst)[q4] =
                make_float4(acc[cc][4 * q4], acc[cc][4 * q4 + 1], acc[cc][4 * q4 + 2], acc[cc][4 * q4 + 3]);
        }
      }
    }
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, (uint32_t)a.tcols);
}

int launch_hpass_tc(HArgs& a, const nys_filter_desc* d, cudaStream_t s) {
  const int R = d->radius;
  int TW = ((K2T_PX - 2 * R) / K2_XR) * K2_XR;
  if (TW < K2_XR) return NYS_EUNSUPPORTED;
  TW = (int)std::min<int64_t>(TW, ceil_div(d->W, K2_XR) * K2_XR);
  const int KU = (int)ceil_div(d->m0, 8) * 8;
  const int NU = (int)ceil_div(d->m0 + 1, 16) * 16;
  if (NU > 256) return NYS_EUNSUPPORTED;
  int tcols = 32;
  while (tcols < NU) tcols *= 2;
  int pitch = (int)ceil_div(TW + 2 * R + 4, 4) * 4;
  pitch += ((4 - pitch % 32) + 32) % 32;  // = 4 (mod 32): the FIR's LDS.128 across rows is conflict-free
  const size_t floats = (size_t)align32f(d->m0 * a.rhop) + 2 * (size_t)NU * KU + align32f(d->n * pitch) +
                        std::max<size_t>(2 * (size_t)K2T_PX * KU, (size_t)a.m0q * pitch);
  const size_t smem = floats * 4;
  if (smem > 220 * 1024) return NYS_EUNSUPPORTED;
  a.TW = TW;
  a.rpt = 1;
  a.pitch = pitch;
  a.tiles_x = (int)ceil_div(d->W, TW);
  a.ku = KU;
  a.nu = NU;
  a.tcols = tcols;
  const long long ntiles = (long long)a.tiles_x * a.vrows;
  const int GR = d->rho <= 4 ? 4 : (d->rho <= 16 ? 16 : (d->rho <= 32 ? 32 : 64));
  auto go = [&](auto kern) -> int {
    NYS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // all of the unified L1 as shared memory: two ~110 KB CTAs per SM
    NYS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    // CTAs per SM: shared memory (228 KB per SM, 1 KB reserved per CTA) and
    // TMEM (512 columns) -- the occupancy API under-reports the former here
    const int occ = std::max(1, std::min<int>((int)((228 * 1024) / (smem + 2048)), std::min(2, 512 / tcols)));
    const int grid = (int)std::min<long long>(ntiles, (long long)num_sms() * occ);
    count_launch();
    kern<<<grid, K2T_THREADS, smem, s>>>(a);
    NYS_LAUNCH_CHECK();
    return NYS_OK;
  };
#define NYS_HT_GR(RV)                                      \
  switch (GR) {                                            \
    case 4: return go(k_feat_hpass_tc<RV, 4>);             \
    case 16: return go(k_feat_hpass_tc<RV, 16>);           \
    case 32: return go(k_feat_hpass_tc<RV, 32>);           \
    default: return go(k_feat_hpass_tc<RV, 64>);           \
  }
  const int rsel = a.box ? 0 : R;
  switch (rsel) {
    case 9: NYS_HT_GR(9)
    case 12: NYS_HT_GR(12)
    case 15: NYS_HT_GR(15)
    case 18: NYS_HT_GR(18)
    default: NYS_HT_GR(0)
  }
#undef NYS_HT_GR
}

}  // namespace nys
