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
//   1. features: pixel p (TMEM lane p) evaluates b_j for half of the
//      landmarks and stores b_hi / b_lo into the A operand in TMEM (tcgen05.st);
//   2. one thread issues 3 x K/8 tcgen05.mma (A from TMEM, B = M from SMEM)
//      into the TMEM accumulator and commits to an mbarrier;
//   3. epilogue: tcgen05.ld drains the accumulator (lane = pixel, column = i)
//      into the y rows in SMEM, and the tile's f rows are staged;
//   4. FIR items (4 planes x 16 columns) write the blocked plane buffer.
// Steps 1-2 of tile t+1 run before step 4 of tile t, so the tensor core works
// while the CUDA cores filter.  A persistent CTA (one per SM) runs two such
// pipelines (groups of 256 threads, own TMEM columns, y/f buffers and group
// barrier) that share one copy of the B operand (M and u0, split hi/lo,
// K-major core matrices); with double-buffered y/f rows a group needs one
// barrier per tile, and the other group fills the SM while it waits.
#include <cstdio>
#include <cstdlib>

#include "nys_hpass.cuh"
#include "nys_umma.cuh"

namespace nys {

constexpr int K2T_GROUP = 256;               // threads per pipeline group
constexpr int K2T_THREADS = 2 * K2T_GROUP;     // two groups per CTA share the B operand
constexpr int K2T_PX = 128;                    // UMMA M: source pixels per tile

__host__ __device__ inline int align32f(int v) { return (v + 31) & ~31; }

__device__ __forceinline__ void group_sync(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(K2T_GROUP) : "memory");
}

// shared-memory accesses by 32-bit shared address: the generic-pointer forms re-derived the
// shared window base (S2UR SR_CgaCtaId, UMOV, ULEA) per landmark in the feature loop
__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
// exp2 of a non-positive argument as one MUFU (exp2f adds a range fix-up for results below
// 2^-126, which flush to zero here: features that small are zero to the filter)
__device__ __forceinline__ float ex2_fast(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 3xTF32 split of a finite value: hi = x rounded to TF32 (integer round-half-up on the 13
// dropped bits; cvt.rna.tf32 expands to 4 instructions with its inf/nan path), lo = x - hi,
// exact in FP32 -- the tensor core reads TF32 by truncation, so lo needs no rounding of its own
// (its dropped bits are below 2^-22 |x|)
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
  lo = x - hi;
}

// packed FP32 pairs (one issue slot per two lanes of arithmetic): d = a * b + c on both halves
__device__ __forceinline__ unsigned long long ffma2_pk(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
  unsigned long long v;
  asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "f"(lo), "f"(hi));
  return v;
}
__device__ __forceinline__ void lds128_pk(uint32_t addr, unsigned long long& a, unsigned long long& b) {
  asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "r"(addr));
}

// GR: guide dimensions held in registers per pixel, a multiple of 4 -- or 3 for rho == 3
// exactly (colour guides: the padded fourth dimension costs a subtract and an FMA per landmark)
template <int RT, int GR>
__global__ void __launch_bounds__(K2T_THREADS, 1) k_feat_hpass_tc(const HArgs a) {
  extern __shared__ __align__(128) float sm[];
  __shared__ uint64_t mma_bar[2];
  __shared__ uint32_t tmem_base;
  const int R = RT > 0 ? RT : a.R;
  const int m0 = a.m0, m0q = a.m0q, n = a.n, rho = a.rho, rhop = a.rhop, W = a.W, H = a.H;
  const int NC = n + 1, L = m0 + 1, pitch = a.pitch, TW = a.TW;
  const int KU = a.ku, NU = a.nu, nbuf = a.nbuf;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = tid / K2T_GROUP, gtid = tid % K2T_GROUP;
  const int nchunks = (NC + K2_CC - 1) / K2_CC;
  const int nfr = nchunks * K2_CC;  // f rows per buffer: f_c, 1 (y plane), 0 padding

  float* Cs = sm;                                  // KU x rhop, rows >= m0 zero (none when the features come from b planes)
  float* Bh = Cs + (a.bfrom ? 0 : align32f(KU * rhop));  // NU x KU, K-major core matrices
  float* Bl = Bh + NU * KU;
  float* gbase = Bl + NU * KU;                     // per group, per buffer: Fs (nfr x pitch), Ys (m0q x pitch)
  const int buf_floats = align32f(nfr * pitch) + m0q * pitch;
  auto Fs_of = [&](int b) { return gbase + (size_t)(g * nbuf + b) * buf_floats; };
  auto Ys_of = [&](int b) { return Fs_of(b) + align32f(nfr * pitch); };

  if (!a.bfrom)  // landmarks padded to KU rows: the feature loop runs over all KU without a bound check
    for (int k = tid; k < KU * rhop; k += K2T_THREADS) {
      int src = k;  // row-major [landmark][rhop]
      if constexpr (GR <= 4) {
        // colour guides: landmark pairs interleaved per dimension, [pair][d][2] (rhop == 4), so one
        // LDS.128 yields the (x, y) pairs and the next the (z, w) pairs of two landmarks as packed
        // f32x2 operands
        const int pr = k >> 3, d = (k >> 1) & 3, h = k & 1;
        src = (2 * pr + h) * 4 + d;
      }
      Cs[k] = src < m0 * rhop ? a.cst[src] : 0.f;
    }
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
  if (warp == 0) umma::tmem_alloc(&tmem_base, (uint32_t)(2 * a.tcols));
  if (tid < 2) {
    umma::mbar_init(&mma_bar[tid], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  umma::fence_proxy_async();  // B operand: generic-proxy writes -> tensor core
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  // this group's TMEM columns: D = [0, NU), A_hi = [a_hi, +KU), A_lo = [a_lo, +KU)
  const uint32_t tmem = tmem_base + (uint32_t)(g * a.tcols);
  const uint32_t a_hi = tmem + (uint32_t)align32f(NU), a_lo = a_hi + (uint32_t)align32f(KU);
  const uint32_t idesc = umma::idesc_tf32(K2T_PX, NU);
  const int q = warp & 3, hh = (warp >> 2) & 1;  // TMEM sub-partition (lanes 32q..) and column half
  const uint32_t lane_base = (uint32_t)(32 * q) << 16;
  const int px = 32 * q + lane;                  // this thread's source pixel (TMEM lane) in a tile
  uint64_t* bar = &mma_bar[g];

  const int ncols = TW + 2 * R;  // <= 128
  const int ncol4 = (ncols + 3) & ~3;
  const int XG = TW / K2_XR;
  const int fir_items = L * nchunks * XG;
  const int ntiles = a.tiles_x * a.vrows;
  const int khalf = KU / 2;  // landmarks per feature thread (multiple of 4)
  const uint32_t cs_half = umma::smem_addr(Cs) + (uint32_t)(hh * khalf * rhop) * 4u;  // this thread's first landmark
  const uint32_t rhob = (uint32_t)rhop * 4u;
  const float k2 = a.k2;

  // 1. features of the tile at virtual row vr, columns x0..: pixel px evaluates b_j for its
  // half of the landmarks and stores b_hi / b_lo into the A operand in TMEM (raw b planes for K3 too)
  auto features = [&](int vr, int x0) {
    const int row = clampi(clampi(vr, 0, H - 1), a.rlo, a.rhi - 1);
    const int xs = x0 - R + px;
    const int x = clampi(xs, 0, W - 1);
    if (a.bfrom) {  // wide guide: b_j(x) from the planes k_bplanes_wide wrote for this virtual row
      const float* bsrc = a.hp + (long long)(vr - a.v0) * a.rs + (long long)(x >> 5) * (a.npl * 32) +
                          (long long)(L * NC) * 32 + (x & 31);
      for (int j0 = hh * khalf; j0 < (hh + 1) * khalf; j0 += 4) {
        float hi[4], lo[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) split_tf32(j0 + e < m0 ? bsrc[(size_t)(j0 + e) * 32] : 0.f, hi[e], lo[e]);
        umma::st_32x32b_x4(a_hi + lane_base + (uint32_t)j0, hi[0], hi[1], hi[2], hi[3]);
        umma::st_32x32b_x4(a_lo + lane_base + (uint32_t)j0, lo[0], lo[1], lo[2], lo[3]);
      }
      umma::st_wait();
      return;
    }
    float gv[GR];
#pragma unroll
    for (int dd = 0; dd < GR; ++dd)
      gv[dd] = dd < rho ? guide_at(a.g, a.gps, a.f, a.fps, a.gkind, dd, row, x, H, W) : 0.f;
    float* bdst = nullptr;
    if (a.bplanes && !a.phi && px >= R && px < R + TW && xs < ((W + 31) & ~31))
      bdst = a.hp + (long long)(vr - a.v0) * a.rs + (long long)(xs >> 5) * (a.npl * 32) + (long long)(L * NC) * 32 +
             (xs & 31) + (long long)(hh * khalf) * 32;
    const int jlim = m0 - hh * khalf;  // stores of raw b planes stop at landmark m0
    uint32_t ca = cs_half;
    const uint32_t t_hi = a_hi + lane_base + (uint32_t)(hh * khalf), t_lo = a_lo + lane_base + (uint32_t)(hh * khalf);
    if constexpr (GR <= 4) {
      // Two landmarks per packed f32x2 operation (fma.rn.f32x2: one issue slot for both).  With
      // the pair-interleaved centroids: t = (g, g) - (c_j, c_j+1) per dimension as an FMA with -1,
      // d2 = t0 t0, + t1 t1, + t2 t2 in the scalar order, one packed scale by k2 -- every half
      // rounds exactly as the scalar form did -- then two MUFUs and the TF32 splits.  The next four
      // landmarks' centroids are loaded before this four's arithmetic (ordered asm loads; the
      // last prefetch reads past the landmarks into the B operand, still this CTA's shared memory).
      const unsigned long long neg1 = pack2(-1.f, -1.f), k2p = pack2(k2, k2);
      unsigned long long g2[GR];
#pragma unroll
      for (int d = 0; d < GR; ++d) g2[d] = pack2(gv[d], gv[d]);
      unsigned long long nx[2], ny[2], nz[2], nw[2];
      auto load_pairs = [&](uint32_t addr) {
#pragma unroll
        for (int pr = 0; pr < 2; ++pr) {
          lds128_pk(addr + 32u * pr, nx[pr], ny[pr]);
          if constexpr (GR == 4) {
            lds128_pk(addr + 32u * pr + 16u, nz[pr], nw[pr]);
          } else {
            asm volatile("ld.shared.b64 %0, [%1];" : "=l"(nz[pr]) : "r"(addr + 32u * pr + 16u));
            nw[pr] = 0ull;
          }
        }
      };
      load_pairs(ca);
      for (int jj = 0; jj < khalf; jj += 4) {
        unsigned long long cx[2], cy[2], cz[2], cw[2];
#pragma unroll
        for (int pr = 0; pr < 2; ++pr) {
          cx[pr] = nx[pr];
          cy[pr] = ny[pr];
          cz[pr] = nz[pr];
          cw[pr] = nw[pr];
        }
        ca += 64u;
        load_pairs(ca);
        float hi[4], lo[4];
#pragma unroll
        for (int pr = 0; pr < 2; ++pr) {
          const unsigned long long t0 = ffma2_pk(cx[pr], neg1, g2[0]), t1 = ffma2_pk(cy[pr], neg1, g2[1]),
                                   t2 = ffma2_pk(cz[pr], neg1, g2[2]);
          unsigned long long d2 = ffma2_pk(t0, t0, 0ull);
          d2 = ffma2_pk(t1, t1, d2);
          d2 = ffma2_pk(t2, t2, d2);
          if constexpr (GR == 4) {
            const unsigned long long t3 = ffma2_pk(cw[pr], neg1, g2[3]);
            d2 = ffma2_pk(t3, t3, d2);
          }
          float e0, e1;
          unpack2(ffma2_pk(d2, k2p, 0ull), e0, e1);
          // (no raw b planes here: K3 reads them only for rho > 8 / patch guides, use_bplanes(); the
          // phi-form stores phi from the drain instead)
          split_tf32(ex2_fast(e0), hi[2 * pr], lo[2 * pr]);
          split_tf32(ex2_fast(e1), hi[2 * pr + 1], lo[2 * pr + 1]);
        }
        umma::st_32x32b_x4(t_hi + (uint32_t)jj, hi[0], hi[1], hi[2], hi[3]);
        umma::st_32x32b_x4(t_lo + (uint32_t)jj, lo[0], lo[1], lo[2], lo[3]);
      }
    } else {
      // wide guides: two dimensions per packed f32x2 operation.  The centroid rows are read as
      // (c_d, c_d+1) pairs straight from the LDS.128, t = g - c as an FMA with -1, and the squares
      // accumulate in an (even dimensions, odd dimensions) pair added at the end -- a different
      // summation order from the scalar form (b differs in the last bits; K3 reads these very
      // values from the b planes, so the two kernels stay consistent).
      const unsigned long long neg1 = pack2(-1.f, -1.f);
      unsigned long long g2[GR / 2];
#pragma unroll
      for (int d = 0; d < GR / 2; ++d) g2[d] = pack2(gv[2 * d], gv[2 * d + 1]);
      for (int jj = 0; jj < khalf; jj += 4) {
        float hi[4], lo[4];
#pragma unroll
        for (int e = 0; e < 4; ++e, ca += rhob) {
          unsigned long long acc2 = 0ull;
#pragma unroll
          for (int d4 = 0; d4 < GR / 4; ++d4) {
            if (4 * d4 < rho) {
              unsigned long long c01, c23;
              lds128_pk(ca + 16u * d4, c01, c23);
              const unsigned long long t01 = ffma2_pk(c01, neg1, g2[2 * d4]), t23 = ffma2_pk(c23, neg1, g2[2 * d4 + 1]);
              acc2 = ffma2_pk(t01, t01, acc2);
              acc2 = ffma2_pk(t23, t23, acc2);
            }
          }
          float de, dod;
          unpack2(acc2, de, dod);
          const float v = ex2_fast((de + dod) * k2);
          if (bdst && jj + e < jlim) bdst[(size_t)(jj + e) * 32] = v;
          split_tf32(v, hi[e], lo[e]);
        }
        umma::st_32x32b_x4(t_hi + (uint32_t)jj, hi[0], hi[1], hi[2], hi[3]);
        umma::st_32x32b_x4(t_lo + (uint32_t)jj, lo[0], lo[1], lo[2], lo[3]);
      }
    }
    umma::st_wait();
  };
  // 2. y = M b: 3 x K/8 MMAs (M=128, N=NU, K=8).  Issued by the group's last warp, converged,
  // one elected lane per MMA (mma_tf32_ts_elect): a divergent `if (gtid == 0)` made every MMA an
  // ELECT / R2UR.BROADCAST waterfall loop (~125 cycles each) in the warp that also carries the most
  // FIR items, and the group's next barrier waited for it; the last warp's threads have one FIR
  // item fewer per tile (items are dealt from thread 0 up) and the slack to issue
  const uint64_t desc_bh = umma::desc_kmajor(Bh, (uint32_t)NU * 16, 128), desc_bl = umma::desc_kmajor(Bl, (uint32_t)NU * 16, 128);
  const uint64_t desc_step = (uint64_t)((8 * NU * 4) >> 4);  // one K step (8 columns) in the address field
  const int gwarp_u = __shfl_sync(0xffffffffu, gtid >> 5, 0);  // warp index within the group, warp-uniform to the compiler
  const bool issuer = gwarp_u == K2T_GROUP / 32 - 1;
  auto issue_mma = [&]() {
    uint32_t acc = 0;
#pragma unroll 1
    for (int pass = 0; pass < 3; ++pass) {
      const uint32_t A = pass == 2 ? a_lo : a_hi;
      uint64_t B = pass == 1 ? desc_bl : desc_bh;
#pragma unroll 1
      for (int kk = 0; kk < KU / 8; ++kk, B += desc_step) {
        umma::mma_tf32_ts_elect(tmem, A + (uint32_t)(8 * kk), B, idesc, acc);
        acc = 1;
      }
    }
    umma::commit_elect(bar);
  };
  // 3. accumulator -> y rows in SMEM (warps w, w+4 of the group drain half of
  // the column chunks of TMEM lanes 32(w%4)..), and the tile's f rows
  const int nch = (L + 7) / 8;                       // 8-column chunks holding y_0 .. y_m0 (the lead column last)
  const int ch0 = hh ? (nch + 1) / 2 : 0, ch1 = hh ? nch : (nch + 1) / 2;
  auto epilogue = [&](int vr, int x0, int b) {
    const uint32_t ys = umma::smem_addr(Ys_of(b)) + (uint32_t)px * 4u;
    const uint32_t pitchb = (uint32_t)pitch * 4u;
    float* Fs = Fs_of(b);
    const bool phi_out = a.phi && a.bplanes && px >= R && px < R + TW && (x0 - R + px) < ((W + 31) & ~31);
    float* pdst = nullptr;
    if (phi_out) {  // phi-form: phi_i = y_i is K3's contraction weight
      const int xs = x0 - R + px;
      pdst = a.hp + (long long)(vr - a.v0) * a.rs + (long long)(xs >> 5) * (a.npl * 32) + (long long)(L * NC) * 32 +
             (xs & 31);
    }
    for (int c = ch0; c < ch1; ++c) {
      float v[8];
      umma::ld_32x32b_x8(tmem + lane_base + (uint32_t)(8 * c), v);
      umma::ld_wait();
      if (px < ncols) {
        const uint32_t yc = ys + (uint32_t)(8 * c) * pitchb;
        if (8 * c + 8 <= L) {
#pragma unroll
          for (int e = 0; e < 8; ++e) sts32(yc + (uint32_t)e * pitchb, v[e]);
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (8 * c + e < L) sts32(yc + (uint32_t)e * pitchb, v[e]);
        }
      }
      if (pdst) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int i = 8 * c + e;
          if (i < m0) pdst[(size_t)i * 32] = v[e];
        }
      }
    }
    // f rows: thread (s, c0) stages column s of rows c0, c0 + 2, ... (ncol4 <= 128 = K2T_GROUP / 2)
    const int row = clampi(clampi(vr, 0, H - 1), a.rlo, a.rhi - 1);
    const int s = gtid & (K2T_PX - 1);
    if (s < ncol4) {
      const int x = clampi(x0 - R + s, 0, W - 1);
      const float* fsrc = a.f + (long long)row * W + x;
      for (int c = gtid / K2T_PX; c < nfr; c += K2T_GROUP / K2T_PX)
        Fs[(size_t)c * pitch + s] = c < n ? __ldg(fsrc + (long long)c * a.fps) : (c == n ? 1.f : 0.f);
    }
  };
  // 4. horizontal FIR of the (m0+1)(n+1) planes, blocked-layout stores
  const int strideL = K2T_GROUP % L, strideR = K2T_GROUP / L;  // item stride in (i, rest) digits
  auto fir = [&](int vr, int x0, int b) {
    const float* Ys = Ys_of(b);
    const float* Fs = Fs_of(b);
    // (i, ch, xg) of item it = ((xg * nchunks + ch) * L + i), advanced incrementally by the
    // group stride (no divisions per item)
    // Items are dealt from FIR thread 0 up, so the first fir_items - 256 threads carry one item more.
    // Group 1 rotates its thread numbering by two warps: the warps with the extra item then sit on
    // different SM sub-partitions in the two groups (CTA warp w issues on sub-partition w % 4; without
    // the rotation sub-partition 0 carried 8 warp-items per tile pair against 6 on the others).
    const int ftid = (gtid + 64 * g) & (K2T_GROUP - 1);
    int i = ftid % L, ch = (ftid / L) % nchunks, xg = (ftid / L) / nchunks;
    auto advance = [&]() {
      i += strideL;
      ch += strideR;
      if (i >= L) {
        i -= L;
        ++ch;
      }
      if (nchunks == 1) {  // the common case (n <= 3): rest == xg
        xg += ch;
        ch = 0;
      } else if (ch >= nchunks) {
        const int q = ch / nchunks;
        xg += q;
        ch -= q * nchunks;
      }
    };
    for (int it = ftid; it < fir_items; it += K2T_GROUP, advance()) {
      const int xo = x0 + xg * K2_XR;
      if (xo >= W) continue;
      const float* yrow = Ys + (size_t)i * pitch + xg * K2_XR;
      float* dst0 = a.hp + (long long)(vr - a.v0) * a.rs + (long long)(xo >> 5) * (a.npl * 32) + (xo & 31);
      const int cend = min(K2_CC, NC - ch * K2_CC);
      if (RT == 0 && a.box) {  // running sums: all planes of the item share the y loads
        float acc[K2_CC][K2_XR];
        hfir<0, true>(a, yrow, Fs, pitch, xg * K2_XR, ch * K2_CC, acc);
#pragma unroll
        for (int cc = 0; cc < K2_CC; ++cc) {
          if (cc < cend) {
            float* dst = dst0 + (i * NC + ch * K2_CC + cc) * 32;
#pragma unroll
            for (int q4 = 0; q4 < K2_XR / 4; ++q4)
              reinterpret_cast<float4*>(dst)[q4] =
                  make_float4(acc[cc][4 * q4], acc[cc][4 * q4 + 1], acc[cc][4 * q4 + 2], acc[cc][4 * q4 + 3]);
          }
        }
        continue;
      }
#pragma unroll 1
      for (int cc = 0; cc < cend; ++cc) {
        const int c = ch * K2_CC + cc;
        float acc[K2_XR];
        hfir_plane<RT>(a, yrow, Fs + (size_t)c * pitch + xg * K2_XR, acc);
        float* dst = dst0 + (i * NC + c) * 32;
#pragma unroll
        for (int q4 = 0; q4 < K2_XR / 4; ++q4)
          reinterpret_cast<float4*>(dst)[q4] = make_float4(acc[4 * q4], acc[4 * q4 + 1], acc[4 * q4 + 2], acc[4 * q4 + 3]);
      }
    }
  };

  // Software pipeline per group: the MMAs of tile t+1 run on the tensor core
  // while the CUDA cores filter tile t.  With two y/f buffers one group
  // barrier per tile suffices: it orders epilogue(t) before FIR(t) and MMA(t+1),
  // features(t+1) before MMA(t+1), and FIR(t-1) before epilogue(t+1).
  const int stride = 2 * gridDim.x;
  int tile = 2 * blockIdx.x + g;
  // (virtual row, first column) of a tile, stepped by the grid stride without a division per tile
  const int dvr = stride / a.tiles_x, dtx = stride - dvr * a.tiles_x;
  int tr = tile / a.tiles_x, tx = tile - tr * a.tiles_x;
  uint32_t phase = 0;
  int b = 0;
  if (tile < ntiles) {
    features(a.v0 + tr, tx * TW);
    umma::fence_before();
    group_sync(g);
    if (issuer) {
      umma::fence_after();
      issue_mma();
    }
    umma::mbar_wait(bar, phase);
    phase ^= 1u;
    umma::fence_after();
    epilogue(a.v0 + tr, tx * TW, b);
  }
  for (; tile < ntiles; tile += stride) {
    const int next = tile + stride;
    const bool more = next < ntiles;
    int nr = tr + dvr, nx = tx + dtx;
    if (nx >= a.tiles_x) {
      nx -= a.tiles_x;
      ++nr;
    }
    if (more) features(a.v0 + nr, nx * TW);
    umma::fence_before();
    group_sync(g);
    umma::fence_after();
    if (more && issuer) issue_mma();
    fir(a.v0 + tr, tx * TW, b);
    if (more) {
      umma::mbar_wait(bar, phase);
      phase ^= 1u;
      umma::fence_after();
      if (nbuf == 1) group_sync(g);  // single buffer: FIR(tile) must be done with Ys / Fs
      b = (b + 1 == nbuf) ? 0 : b + 1;
      epilogue(a.v0 + nr, nx * TW, b);
    }
    tr = nr;
    tx = nx;
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem_base, (uint32_t)(2 * a.tcols));
}

// Features of a wide guide (rho > NYS_MAX_RHO) for every virtual row of the band, written as
// the raw b planes K3 reads anyway (plane index (m0+1)(n+1) + j): one CTA per 32-column block
// of a virtual row; the 32 guide vectors are staged in shared memory ([rho][32], lane = pixel),
// warp w evaluates landmarks w, w + 8, ... (difference form, FP32, exp2 as in the fast kernels).
__global__ void __launch_bounds__(256) k_bplanes_wide(const HArgs a) {
  extern __shared__ __align__(16) float gsm[];  // rho x 32 guide values, then m0 x rhop centroids
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int rho = a.rho, rhop = a.rhop, m0 = a.m0, W = a.W, H = a.H;
  const int nxb = (W + 31) >> 5;
  const int vr = a.v0 + blockIdx.x / nxb, xb = blockIdx.x % nxb;
  const int row = clampi(clampi(vr, 0, H - 1), a.rlo, a.rhi - 1);
  float* Cs = gsm + (size_t)rho * 32;
  for (int k = threadIdx.x; k < m0 * rhop; k += blockDim.x) Cs[k] = a.cst[k];
  for (int k = threadIdx.x; k < rho * 32; k += blockDim.x) {
    const int dd = k >> 5, x = min(xb * 32 + (k & 31), W - 1);
    gsm[k] = guide_at(a.g, a.gps, a.f, a.fps, a.gkind, dd, row, x, H, W);
  }
  __syncthreads();
  const int L = m0 + 1, NC = a.n + 1;
  float* dst = a.hp + (long long)(vr - a.v0) * a.rs + (long long)xb * (a.npl * 32) + (long long)(L * NC) * 32 + lane;
  for (int j = w; j < m0; j += 8) {
    const float* c = Cs + (size_t)j * rhop;
    float d2 = 0.f;
    for (int dd = 0; dd < rho; ++dd) {
      const float t = gsm[dd * 32 + lane] - c[dd];
      d2 = fmaf(t, t, d2);
    }
    dst[(size_t)j * 32] = range_kernel(d2, a.k2);
  }
}

int launch_hpass_tc(HArgs& a, const nys_filter_desc* d, cudaStream_t s) {
  if (d->rho > NYS_MAX_RHO) {
    if (a.phi) return NYS_EUNSUPPORTED;  // the phi-form stores phi, not b, in the feature planes
    const size_t wsm = ((size_t)d->rho * 32 + (size_t)d->m0 * a.rhop) * sizeof(float);
    if (wsm > 220 * 1024) return NYS_EUNSUPPORTED;
    NYS_CUDA_TRY(cudaFuncSetAttribute(k_bplanes_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm));
    const long long nblk = (long long)a.vrows * ((d->W + 31) / 32);
    count_launch();
    k_bplanes_wide<<<(unsigned)nblk, 256, wsm, s>>>(a);
    NYS_LAUNCH_CHECK();
    a.bfrom = 1;
  }
  const int R = d->radius;
  int TW = ((K2T_PX - 2 * R) / K2_XR) * K2_XR;
  if (TW < K2_XR) return NYS_EUNSUPPORTED;
  TW = (int)std::min<int64_t>(TW, ceil_div(d->W, K2_XR) * K2_XR);
  const int KU = (int)ceil_div(d->m0, 8) * 8;
  const int NU = (int)ceil_div(d->m0 + 1, 16) * 16;
  // TMEM per group: accumulator (NU columns) + A_hi + A_lo (KU columns each),
  // 32-column aligned; the two groups of a CTA share one allocation
  const int need = align32f(NU) + 2 * align32f(KU);
  if (NU > 256 || need > 256) return NYS_EUNSUPPORTED;
  int tcols = 32;
  while (tcols < need) tcols *= 2;
  int pitch = (int)ceil_div(TW + 2 * R + 4, 4) * 4;
  pitch += ((4 - pitch % 32) + 32) % 32;  // = 4 (mod 32): the FIR's LDS.128 across rows is conflict-free
  const int nfr = (int)ceil_div(d->n + 1, K2_CC) * K2_CC;
  const size_t fixed = (a.bfrom ? 0 : (size_t)align32f(KU * a.rhop)) + 2 * (size_t)NU * KU;
  const size_t buf = (size_t)align32f(nfr * pitch) + (size_t)a.m0q * pitch;
  // two y/f buffers per group when they fit (one barrier per tile), else one
  int nbuf = 2;
  if ((fixed + 2 * nbuf * buf) * 4 > 225 * 1024) nbuf = 1;
  const size_t smem = (fixed + 2 * nbuf * buf) * 4;
  if (smem > 225 * 1024) return NYS_EUNSUPPORTED;
  a.TW = TW;
  a.rpt = 1;
  a.pitch = pitch;
  a.tiles_x = (int)ceil_div(d->W, TW);
  a.ku = KU;
  a.nu = NU;
  a.tcols = tcols;
  a.nbuf = nbuf;
  const long long ntiles = (long long)a.tiles_x * a.vrows;
  const int GR = a.bfrom ? 4 : (d->rho == 3 && d->guide_kind == 0 ? 3 : (d->rho <= 4 ? 4 : (d->rho <= 16 ? 16 : (d->rho <= 32 ? 32 : 64))));
  auto go = [&](auto kern) -> int {
    NYS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    NYS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    // one CTA (two pipeline groups) per SM; each group takes tiles 2*blockIdx.x + g + k*2*grid
    const int grid = (int)std::min<long long>(ceil_div(ntiles, 2), (long long)num_sms());
    count_launch();
    kern<<<grid, K2T_THREADS, smem, s>>>(a);
    NYS_LAUNCH_CHECK();
    return NYS_OK;
  };
#define NYS_HT_GR(RV)                                      \
  switch (GR) {                                            \
    case 3: return go(k_feat_hpass_tc<RV, 3>);             \
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
