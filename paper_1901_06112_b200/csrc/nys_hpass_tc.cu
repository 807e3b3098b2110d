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

  float* Cs = sm;                                  // m0 x rhop
  float* Bh = Cs + align32f(m0 * rhop);            // NU x KU, K-major core matrices
  float* Bl = Bh + NU * KU;
  float* gbase = Bl + NU * KU;                     // per group, per buffer: Fs (nfr x pitch), Ys (m0q x pitch)
  const int buf_floats = align32f(nfr * pitch) + m0q * pitch;
  auto Fs_of = [&](int b) { return gbase + (size_t)(g * nbuf + b) * buf_floats; };
  auto Ys_of = [&](int b) { return Fs_of(b) + align32f(nfr * pitch); };

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

  // 1. features of `tile`: pixel px evaluates b_j for its half of the landmarks
  // and stores b_hi / b_lo into the A operand in TMEM (raw b planes for K3 too)
  auto features = [&](int tile) {
    const int vr = a.v0 + tile / a.tiles_x;
    const int x0 = (tile % a.tiles_x) * TW;
    const int row = clampi(clampi(vr, 0, H - 1), a.rlo, a.rhi - 1);
    const int xs = x0 - R + px;
    const int x = clampi(xs, 0, W - 1);
    float gv[GR];
#pragma unroll
    for (int dd = 0; dd < GR; ++dd)
      gv[dd] = dd < rho ? guide_at(a.g, a.gps, a.f, a.fps, a.gkind, dd, row, x, H, W) : 0.f;
    float* bdst = nullptr;
    if (a.bplanes && !a.phi && px >= R && px < R + TW && xs < ((W + 31) & ~31))
      bdst = a.hp + (long long)(vr - a.v0) * a.rs + (long long)(xs >> 5) * (a.npl * 32) + (long long)(L * NC) * 32 +
             (xs & 31);
    for (int j0 = hh * khalf; j0 < (hh + 1) * khalf; j0 += 4) {
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
      float hi[4], lo[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        hi[e] = umma::to_tf32(bv[e]);
        lo[e] = umma::to_tf32(bv[e] - hi[e]);
      }
      umma::st_32x32b_x4(a_hi + lane_base + (uint32_t)j0, hi[0], hi[1], hi[2], hi[3]);
      umma::st_32x32b_x4(a_lo + lane_base + (uint32_t)j0, lo[0], lo[1], lo[2], lo[3]);
    }
    umma::st_wait();
  };
  // 2. y = M b: 3 x K/8 MMAs (M=128, N=NU, K=8), issued by one thread
  auto issue_mma = [&]() {
    const uint32_t lbo_b = (uint32_t)NU * 16;
    uint32_t acc = 0;
#pragma unroll 1
    for (int pass = 0; pass < 3; ++pass) {
      const uint32_t A = pass == 2 ? a_lo : a_hi;
      const float* B = pass == 1 ? Bl : Bh;
#pragma unroll 1
      for (int kk = 0; kk < KU / 8; ++kk) {
        umma::mma_tf32_ts(tmem, A + (uint32_t)(8 * kk), umma::desc_kmajor(B + kk * 8 * NU, lbo_b, 128), idesc, acc);
        acc = 1;
      }
    }
    umma::commit(bar);
  };
  // 3. accumulator -> y rows in SMEM (warps w, w+4 of the group drain half of
  // the columns of TMEM lanes 32(w%4)..), and the tile's f rows
  auto epilogue = [&](int tile, int b) {
    float* Ys = Ys_of(b);
    float* Fs = Fs_of(b);
    const int nch = NU / 8, c0 = hh * (nch / 2), c1 = c0 + nch / 2;
    for (int c = c0; c < c1; ++c) {
      float v[8];
      umma::ld_32x32b_x8(tmem + lane_base + (uint32_t)(8 * c), v);
      umma::ld_wait();
      if (px < ncols) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int i = 8 * c + e;
          if (i < L) Ys[(size_t)i * pitch + px] = v[e];
        }
      }
      if (a.phi && a.bplanes && px >= R && px < R + TW) {  // phi-form: phi_i = y_i is K3's contraction weight
        const int vr = a.v0 + tile / a.tiles_x;
        const int xs = (tile % a.tiles_x) * TW - R + px;
        if (xs < ((W + 31) & ~31)) {
          float* dst = a.hp + (long long)(vr - a.v0) * a.rs + (long long)(xs >> 5) * (a.npl * 32) +
                       (long long)(L * NC) * 32 + (xs & 31);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int i = 8 * c + e;
            if (i < m0) dst[(size_t)i * 32] = v[e];
          }
        }
      }
    }
    const int vr = a.v0 + tile / a.tiles_x;
    const int x0 = (tile % a.tiles_x) * TW;
    const int row = clampi(clampi(vr, 0, H - 1), a.rlo, a.rhi - 1);
    for (int k = gtid; k < nfr * ncol4; k += K2T_GROUP) {
      const int c = k / ncol4, s = k - c * ncol4;
      const int x = clampi(x0 - R + s, 0, W - 1);
      Fs[(size_t)c * pitch + s] =
          c < n ? __ldg(a.f + (long long)c * a.fps + (long long)row * W + x) : (c == n ? 1.f : 0.f);
    }
  };
  // 4. horizontal FIR of the (m0+1)(n+1) planes, blocked-layout stores
  const int strideL = K2T_GROUP % L, strideR = K2T_GROUP / L;  // item stride in (i, rest) digits
  auto fir = [&](int tile, int b) {
    const float* Ys = Ys_of(b);
    const float* Fs = Fs_of(b);
    const int vr = a.v0 + tile / a.tiles_x;
    const int x0 = (tile % a.tiles_x) * TW;
    // (i, ch, xg) of item it = ((xg * nchunks + ch) * L + i), advanced incrementally by the
    // group stride (no divisions per item)
    int i = gtid % L, ch = (gtid / L) % nchunks, xg = (gtid / L) / nchunks;
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
    for (int it = gtid; it < fir_items; it += K2T_GROUP, advance()) {
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
  uint32_t phase = 0;
  int b = 0;
  if (tile < ntiles) {
    features(tile);
    umma::fence_before();
    group_sync(g);
    if (gtid == 0) {
      umma::fence_after();
      issue_mma();
    }
    umma::mbar_wait(bar, phase);
    phase ^= 1u;
    umma::fence_after();
    epilogue(tile, b);
  }
  for (; tile < ntiles; tile += stride) {
    const int next = tile + stride;
    const bool more = next < ntiles;
    if (more) features(next);
    umma::fence_before();
    group_sync(g);
    umma::fence_after();
    if (more && gtid == 0) issue_mma();
    fir(tile, b);
    if (more) {
      umma::mbar_wait(bar, phase);
      phase ^= 1u;
      umma::fence_after();
      if (nbuf == 1) group_sync(g);  // single buffer: FIR(tile) must be done with Ys / Fs
      b = (b + 1) % nbuf;
      epilogue(next, b);
    }
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem_base, (uint32_t)(2 * a.tcols));
}

int launch_hpass_tc(HArgs& a, const nys_filter_desc* d, cudaStream_t s) {
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
  const size_t fixed = (size_t)align32f(d->m0 * a.rhop) + 2 * (size_t)NU * KU;
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
  const int GR = d->rho <= 4 ? 4 : (d->rho <= 16 ? 16 : (d->rho <= 32 ? 32 : 64));
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
