// K2 / K3: the Nystrom filter proper, B200 (sm_100a) CUDA.
//
// Reference region replaced (reference = /root/reference/pkg/src/nysfilter):
//   filters.py:214-257   fast_filter k-loop, accumulation, denominator guard
//   nystrom.py:43-79     RangeKernel.gram / build_B   (never materialised here)
//   nystrom.py:112-114   extrapolate V = B^T W / alpha (never materialised here)
//   spatial.py:91-109, 194-209  box / FIR row pass then column pass, replicate
//
// Formulation ("y-form"): with b_i(x) = exp(-|p(x)-c_i|^2/2θ^2)
// and M = Σ_k w_k w_k^T / α_k (retained eigenpairs), the reference's
//   zeta(x) = Σ_k α_k v_k(x) [ω * (v_k f)](x)   (v_k = B^T w_k / α_k)
// equals  Σ_i b_i(x) [ω * (y_i f)](x)  with  y = M b  evaluated at the source
// pixel.  K2 evaluates b and y per source pixel (a register-blocked
// [px x m0] x [m0 x (m0+1)] product, the extra column being the lead
// projection s0 = w_1.b) and runs the horizontal pass of the (m0+1)(n+1)
// planes y_i f_c, y_i.  K3 TMA-stages tiles of those planes, runs the vertical
// pass, contracts with b_i(x) recomputed at the centre pixel, and applies the
// guard and division.  Only the horizontally filtered planes touch HBM.
//
// Plane buffer layout: [virtual row][x / 32][plane][32 columns] with plane
// p = i*(n+1) + c; a band has `rows + 2R` virtual rows and virtual row v maps to
// image row clamp(v, 0, H-1), so K3 never clamps (replicate borders,
// spatial.py:85-88).  One TMA box = 32 columns x 4 planes x (TH+2R) rows.
#include "nys_filter_common.cuh"

namespace nys {

// ---------------------------------------------------------------------------
// K3: TMA-staged vertical pass + contraction with b_i(x) + guard + division
// ---------------------------------------------------------------------------
// Tile = 32 columns x K3_TH rows.  256 threads = 4 plane groups x 8 row runs x
// 8 column quads: thread (grp, run, quad) owns the 4 x K3_YR pixels at columns
// 4*quad.., rows K3_YR*run.. and, in channel chunk k, channel c = 4k + grp.
// Stage order per tile: chunk kn (holding the denominator channel n) first,
// then the others; within a chunk landmarks i = 0..m0-1 and the lead group.
// Each stage is one TMA box of (up to) 4 planes x (TH + 2R) rows x 32 columns
// plus, with K2's b planes, the TH x 32 b_i tile.  A thread keeps only the
// accumulators of its current chunk and s0 = u0.b in registers, so the
// unrolled code is one vertical FIR (~0.5k instructions) and stays in the
// instruction cache.
constexpr int K3_THREADS = 256;
constexpr int K3_YR = 4;             // rows per thread
constexpr int K3_TH = 8 * K3_YR;     // tile rows
constexpr int K3_NPX = K3_TH * 32;   // tile pixels
constexpr int K3_NS = 2;             // TMA pipeline depth

struct VArgs {
  const float* f;
  const float* g;
  float* out;
  const float* cst;
  FilterStats* stats;
  long long fps, gps, ops;
  int n, rho, rhop, H, W, m0, R, box, gkind;
  int out0, out_rows, tiles_x, tiles_y, nchunks, u0_off, vec_out, gcache, ntail;
  int rlo, rhi;  // image rows present in f / guide (reads are clamped into them)
  int sc_off;  // cst[sc_off], cst[sc_off + 1]: 1/alpha_1 and eps_den (written with the plan)
  int out64;   // out addresses float64 planes
  float k2;
  float tau, cerr;          // near-guard flag rule (near_guard); tau = cerr = 0 disables it
  unsigned* flag_list;      // global pixel indices queued for nys_filter_finish
  unsigned* chunk_cnt;
  unsigned list_cap;
  float taps[NYS_MAX_TAPS];
  float2 wpair[NYS_MAX_TAPS + 1];  // packed-FIR tap pairs (fill_tap_pairs)
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_addr(unsigned bar_addr, unsigned parity) {  // 32-bit shared address
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar_addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

// vertical FIR of one staged plane: 4 columns x K3_YR rows per thread, row stride rs floats
// RS: staged row stride in floats when known at compile time (full chunks: 4 planes x 32), else 0
template <int RT, int RS = 0>
__device__ __forceinline__ void vfir(const VArgs& a, const float* __restrict__ src, int rs_rt, float (&G)[K3_YR][4]) {
  const int rs = RS > 0 ? RS : rs_rt;
#pragma unroll
  for (int o = 0; o < K3_YR; ++o) G[o][0] = G[o][1] = G[o][2] = G[o][3] = 0.f;
  if constexpr (RT > 0) {
    // packed FIR: rows (2p, 2p+1) of column e accumulate in one f32x2 register
    constexpr int T = 2 * RT + 1;
    static_assert(K3_YR % 2 == 0, "row pairs");
    unsigned long long G2[K3_YR / 2][4];
#pragma unroll
    for (int p = 0; p < K3_YR / 2; ++p) G2[p][0] = G2[p][1] = G2[p][2] = G2[p][3] = 0ull;
#pragma unroll
    for (int s = 0; s < K3_YR + 2 * RT; ++s) {
      const float4 v = *reinterpret_cast<const float4*>(src + s * rs);
#pragma unroll
      for (int p = 0; p < K3_YR / 2; ++p) {
        const int k = s - 2 * p;
        if (k >= 0 && k <= T) {
          const float2 w = a.wpair[k];
          G2[p][0] = ffma2_bc(v.x, w, G2[p][0]);
          G2[p][1] = ffma2_bc(v.y, w, G2[p][1]);
          G2[p][2] = ffma2_bc(v.z, w, G2[p][2]);
          G2[p][3] = ffma2_bc(v.w, w, G2[p][3]);
        }
      }
    }
#pragma unroll
    for (int p = 0; p < K3_YR / 2; ++p)
#pragma unroll
      for (int e = 0; e < 4; ++e) unpack2(G2[p][e], G[2 * p][e], G[2 * p + 1][e]);
  } else if (a.box) {  // running (2R+1)-sum (spatial.py:91-99)
    const int R = a.R;
    float4 sm4 = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int t = 0; t <= 2 * R; ++t) {
      const float4 v = *reinterpret_cast<const float4*>(src + t * rs);
      sm4.x += v.x;
      sm4.y += v.y;
      sm4.z += v.z;
      sm4.w += v.w;
    }
#pragma unroll
    for (int o = 0; o < K3_YR; ++o) {
      if (o > 0) {
        const float4 vi = *reinterpret_cast<const float4*>(src + (o + 2 * R) * rs);
        const float4 vo = *reinterpret_cast<const float4*>(src + (o - 1) * rs);
        sm4.x += vi.x - vo.x;
        sm4.y += vi.y - vo.y;
        sm4.z += vi.z - vo.z;
        sm4.w += vi.w - vo.w;
      }
      G[o][0] = sm4.x;
      G[o][1] = sm4.y;
      G[o][2] = sm4.z;
      G[o][3] = sm4.w;
    }
  } else {
    const int T = 2 * a.R + 1;
    for (int t = 0; t < T; ++t) {
      const float w = a.taps[t];
#pragma unroll
      for (int o = 0; o < K3_YR; ++o) {
        const float4 v = *reinterpret_cast<const float4*>(src + (o + t) * rs);
        G[o][0] = fmaf(w, v.x, G[o][0]);
        G[o][1] = fmaf(w, v.y, G[o][1]);
        G[o][2] = fmaf(w, v.z, G[o][2]);
        G[o][3] = fmaf(w, v.w, G[o][3]);
      }
    }
  }
}

// G1: b_i recomputed from a planar guide tile (rho <= 8); else K2's b planes arrive with the stage.
// A compile-time switch: with G1 the lead projection s0 = u0 . b is accumulated once per pixel by
// the thread that evaluates that pixel's features and handed to the lead stage through shared
// memory, which takes 16 FMAs per stage and 16 accumulator registers out of every thread (the
// four plane groups used to accumulate it redundantly).
template <int RT, bool G1>
__global__ void __launch_bounds__(K3_THREADS, 2) k_vpass(const __grid_constant__ CUtensorMap tmap4,
                                                        const __grid_constant__ CUtensorMap tmapt,
                                                        const __grid_constant__ CUtensorMap tmapb, const VArgs a) {
  extern __shared__ __align__(128) float sm[];
  const int tid = threadIdx.x;
  const int grp = tid >> 6, run = (tid >> 3) & 7, quad = tid & 7;
  const int m0 = a.m0, n = a.n, rho = a.rho, rhop = a.rhop, H = a.H, W = a.W, NC = n + 1;
  const int R = RT > 0 ? RT : a.R;
  const int SR = K3_TH + 2 * R;     // staged rows per plane
  const int nchunks = a.nchunks;
  const int plane_floats = SR * 32;
  // 1: b from a planar guide tile (rho <= 8), 3: b planes from K2.  In the !G1 instantiations it is a
  // constant only for the box kernel: measured, the Gaussian wide-guide kernels are 3.7 % slower
  // with the constant (cfg 4: 2.22 -> 2.30 ms) and the box one 10 % faster (cfg 3: 0.43 -> 0.39 ms)
  // -- instruction scheduling at the 128-register cap, nothing structural.
  const int gmode = G1 ? 1 : (RT == 0 ? 3 : a.gcache);
  const int stage_floats = 4 * plane_floats + (gmode == 3 ? K3_NPX : 0);
  float* stage = sm;                                           // K3_NS x ([SR][4][32] planes, [TH][32] b)
  float* bsh = stage + (size_t)K3_NS * stage_floats;           // gmode 1: 2 x npx
  float* dsh = bsh + (gmode == 1 ? 2 * K3_NPX : 0);            // npx: eta
  float* lsh = dsh + K3_NPX;                                   // npx: eta_lead
  float* ssh = lsh + K3_NPX;                                   // npx: scale of eta (-1: flagged)
  float* Cs = ssh + K3_NPX;                                    // m0 x rhop (gmode 1 only)
  float* U0 = Cs + (gmode == 1 ? (size_t)m0 * rhop : 0);       // m0
  float* gsh = U0 + ((m0 + 3) & ~3);                           // gmode 1: [rho][npx] guide tile
  float* s0sh = gsh + (gmode == 1 ? (size_t)rho * K3_NPX : 0);  // gmode 1: npx, s0 = u0 . b per pixel
  __shared__ __align__(8) unsigned long long full[K3_NS];
  __shared__ float red_min[K3_THREADS / 32];
  __shared__ unsigned long long red_cnt[K3_THREADS / 32];

  const float inv_alpha0 = a.cst[a.sc_off], eps_den = a.cst[a.sc_off + 1];
  if (gmode == 1)  // the centroids only feed the features recomputed from a planar guide tile
    for (int k = tid; k < m0 * rhop; k += K3_THREADS) Cs[k] = a.cst[k];
  for (int k = tid; k < m0; k += K3_THREADS) U0[k] = a.cst[a.u0_off + k];
  if (tid == 0) {
    for (int b = 0; b < K3_NS; ++b) mbar_init(&full[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const unsigned full_addr = smem_u32(&full[0]);
  const int kn = n / 4;  // chunk holding the denominator channel n
  auto chunk_of = [&](int co) { return co == 0 ? kn : (co <= kn ? co - 1 : co); };
  const int L = m0 + 1;
  const int nstages = nchunks * L;
  const int ntiles = a.tiles_x * a.tiles_y;
  const int ntail = a.ntail;  // planes in a partial last chunk (0: all chunks full)

  // TMA for stage s (chunk order s / L, landmark s % L; i == m0 is the lead group) of tile t
  auto issue_at = [&](int tx, int ty, int i, int k, unsigned long long gs) {
    const int buf = (int)(gs % K3_NS);
    const bool tail = ntail && k == nchunks - 1;
    const int nval = tail ? ntail : 4;
    const bool with_b = gmode == 3 && i < m0;
    float* dst = stage + (size_t)buf * stage_floats;
    mbar_expect_tx(&full[buf], (unsigned)(nval * plane_floats * 4 + (with_b ? K3_NPX * 4 : 0)));
    tma_load_4d(dst, tail ? &tmapt : &tmap4, 0, i * NC + 4 * k, tx, ty * K3_TH, &full[buf]);
    if (with_b) tma_load_4d(dst + 4 * plane_floats, &tmapb, 0, L * NC + i, tx, ty * K3_TH + R, &full[buf]);
  };
  auto issue = [&](int t, int s, unsigned long long gs) {  // prologue only: divisions once
    issue_at(t % a.tiles_x, t / a.tiles_x, s % L, chunk_of(s / L), gs);
  };
  // b_i on every tile pixel from the cached guide tile (gmode 1).  K3_NPX / 4 == K3_THREADS: a
  // thread always evaluates the same four pixels, so for rho <= 3 their guide values stay in
  // registers for the whole tile (gq, loaded by load_gq) and a landmark costs one LDS.128.
  static_assert(K3_NPX / 4 == K3_THREADS, "one pixel quad per thread");
  float gq[3][4];
  auto load_gq = [&]() {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const float4 g4 = d < rho ? *reinterpret_cast<const float4*>(gsh + d * K3_NPX + 4 * tid) : make_float4(0.f, 0.f, 0.f, 0.f);
      gq[d][0] = g4.x;
      gq[d][1] = g4.y;
      gq[d][2] = g4.z;
      gq[d][3] = g4.w;
    }
  };
  float s0q[4] = {0.f, 0.f, 0.f, 0.f};  // s0 of this thread's four feature pixels (denominator chunk)
  auto compute_b = [&](int i, float* bb, bool lead_acc) {
    const float u0i = G1 ? U0[i] : 0.f;
    if (rho <= 3) {
      const float4 c4 = *reinterpret_cast<const float4*>(Cs + i * rhop);  // rhop == 4, padded with zeros
      const float cc[3] = {c4.x, c4.y, c4.z};
      float d2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int d = 0; d < 3; ++d)
        if (d < rho) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float t = gq[d][e] - cc[d];
            d2[e] = fmaf(t, t, d2[e]);
          }
        }
      const float bq[4] = {range_kernel_fast(d2[0], a.k2), range_kernel_fast(d2[1], a.k2), range_kernel_fast(d2[2], a.k2),
                           range_kernel_fast(d2[3], a.k2)};
      *reinterpret_cast<float4*>(bb + 4 * tid) = make_float4(bq[0], bq[1], bq[2], bq[3]);
      if (G1 && lead_acc) {
#pragma unroll
        for (int e = 0; e < 4; ++e) s0q[e] = fmaf(u0i, bq[e], s0q[e]);  // landmark order, as the stages had it
        if (i == m0 - 1) *reinterpret_cast<float4*>(s0sh + 4 * tid) = make_float4(s0q[0], s0q[1], s0q[2], s0q[3]);
      }
      return;
    }
    for (int k4 = tid; k4 < K3_NPX / 4; k4 += K3_THREADS) {
      float4 d2 = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int d = 0; d < rho; ++d) {
        const float4 g4 = *reinterpret_cast<const float4*>(gsh + d * K3_NPX + 4 * k4);
        const float c = Cs[i * rhop + d];
        const float tx = g4.x - c, ty = g4.y - c, tz = g4.z - c, tw = g4.w - c;
        d2.x = fmaf(tx, tx, d2.x);
        d2.y = fmaf(ty, ty, d2.y);
        d2.z = fmaf(tz, tz, d2.z);
        d2.w = fmaf(tw, tw, d2.w);
      }
      const float bq[4] = {range_kernel_fast(d2.x, a.k2), range_kernel_fast(d2.y, a.k2), range_kernel_fast(d2.z, a.k2),
                           range_kernel_fast(d2.w, a.k2)};
      *reinterpret_cast<float4*>(bb + 4 * k4) = make_float4(bq[0], bq[1], bq[2], bq[3]);
      if (G1 && lead_acc) {  // (K3_NPX / 4 == K3_THREADS: k4 == tid, one pass)
#pragma unroll
        for (int e = 0; e < 4; ++e) s0q[e] = fmaf(u0i, bq[e], s0q[e]);
        if (i == m0 - 1) *reinterpret_cast<float4*>(s0sh + 4 * k4) = make_float4(s0q[0], s0q[1], s0q[2], s0q[3]);
      }
    }
  };

  const int pxo = run * K3_YR * 32 + quad * 4;  // this thread's first pixel (row-major, 32 wide)
  unsigned long long gs = 0;                    // global stage counter (mbarrier phases)
  if (tid == 0 && blockIdx.x < ntiles)
    for (int s = 0; s < K3_NS && s < nstages; ++s) issue(blockIdx.x, s, s);

  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int ntx = (tile + (int)gridDim.x) % a.tiles_x, nty = (tile + (int)gridDim.x) / a.tiles_x;
    const int x0 = tx * 32, t0 = a.out0 + ty * K3_TH;
    if (gmode == 1) {
      for (int k = tid; k < rho * K3_NPX; k += K3_THREADS) {
        const int d = k / K3_NPX, q = k - d * K3_NPX;
        const int rr = clampi(min(t0 + (q >> 5), H - 1), a.rlo, a.rhi - 1), cx = min(x0 + (q & 31), W - 1);
        gsh[k] = __ldg(a.g + (long long)d * a.gps + (long long)rr * W + cx);
      }
      __syncthreads();
      if (rho <= 3) load_gq();
      s0q[0] = s0q[1] = s0q[2] = s0q[3] = 0.f;
      compute_b(0, bsh, true);
      __syncthreads();
    }
    float s0[K3_YR][4], acc[K3_YR][4], sab[K3_YR][4];  // sab: sum_i b_i |conv(y_i)| (denominator chunk)
#pragma unroll
    for (int o = 0; o < K3_YR; ++o)
#pragma unroll
      for (int e = 0; e < 4; ++e) s0[o][e] = acc[o][e] = sab[o][e] = 0.f;

#pragma unroll 1
    // (co, i) = (s / L, s % L) kept incrementally: a runtime division per stage was 5 % of
    // this kernel's instructions
    int co = 0, i = 0;
    for (int s = 0; s < nstages; ++s, ++gs, i = (i + 1 == L) ? 0 : i + 1, co += (i == 0)) {
      const int k = chunk_of(co);
      const int c = 4 * k + grp;
      const bool tail = ntail && k == nchunks - 1;
      const int buf = (int)(gs % K3_NS);
      const float* sb = stage + (size_t)buf * stage_floats;
      mbar_wait_addr(full_addr + 8u * (unsigned)buf, (unsigned)((gs / K3_NS) & 1));  // (address formed once: the generic-to-
                                                                                      // shared conversion was 2 % of the instructions)
      float G[K3_YR][4];
      if (c < NC) {
        // staged row: [4 or ntail planes][32 columns]; the full-chunk stride is a constant, so the
        // FIR's loads carry immediate offsets (an IMAD per load otherwise)
        if (!tail)
          vfir<RT, 128>(a, sb + grp * 32 + run * K3_YR * 128 + quad * 4, 128, G);
        else
          vfir<RT>(a, sb + grp * 32 + run * K3_YR * ntail * 32 + quad * 4, ntail * 32, G);
      } else {
#pragma unroll
        for (int o = 0; o < K3_YR; ++o) G[o][0] = G[o][1] = G[o][2] = G[o][3] = 0.f;
      }
      if (i < m0) {
        const float* bb = (gmode == 3 ? sb + 4 * plane_floats : bsh + (i & 1) * K3_NPX) + pxo;
        const float u0i = U0[i];
#pragma unroll
        for (int o = 0; o < K3_YR; ++o) {
          const float4 b4 = *reinterpret_cast<const float4*>(bb + o * 32);
          const float bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            acc[o][e] = fmaf(bv[e], G[o][e], acc[o][e]);
            if (co == 0) {
              if constexpr (!G1) s0[o][e] = fmaf(u0i, bv[e], s0[o][e]);
              if (c == n) sab[o][e] = fmaf(bv[e], fabsf(G[o][e]), sab[o][e]);  // only eta's scale is used
            }
          }
        }
        // features of the next stage's landmark (gmode 1): the other b buffer is free
        if (gmode == 1) {
          if (i + 1 < m0) compute_b(i + 1, bsh + ((i + 1) & 1) * K3_NPX, co == 0);
        }
      } else {
        // lead group: zeta_lead = s0 (ω*(s0 f_c)) / α0 ; chunk kn first publishes eta and eta_lead
        float lg[K3_YR][4];
#pragma unroll
        for (int o = 0; o < K3_YR; ++o) {
          float sv[4];
          if constexpr (G1) {
            const float4 s4 = *reinterpret_cast<const float4*>(s0sh + pxo + o * 32);
            sv[0] = s4.x, sv[1] = s4.y, sv[2] = s4.z, sv[3] = s4.w;
          } else {
            sv[0] = s0[o][0], sv[1] = s0[o][1], sv[2] = s0[o][2], sv[3] = s0[o][3];
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) lg[o][e] = sv[e] * G[o][e] * inv_alpha0;
        }
        if (co == 0) {
          if (c == n) {
#pragma unroll
            for (int o = 0; o < K3_YR; ++o) {
              *reinterpret_cast<float4*>(dsh + pxo + o * 32) = make_float4(acc[o][0], acc[o][1], acc[o][2], acc[o][3]);
              *reinterpret_cast<float4*>(lsh + pxo + o * 32) = make_float4(lg[o][0], lg[o][1], lg[o][2], lg[o][3]);
              // near-guard pixels: queued for the FP64 re-evaluation (nys_filter_finish), marked
              // -1 so the tile statistics leave them to it
              const int row = t0 + run * K3_YR + o;
              float sv[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int x = x0 + quad * 4 + e;
                sv[e] = sab[o][e];
                if (row < a.out0 + a.out_rows && row < H && x < W &&
                    near_guard(acc[o][e], sab[o][e], lg[o][e], eps_den, a.tau, a.cerr)) {
                  const unsigned slot = atomicAdd(&a.stats->flagged, 1u);
                  if (slot < a.list_cap) {  // (past the cap the FP32 result and statistics stand)
                    a.flag_list[slot] = (unsigned)((long long)row * W + x);
                    a.chunk_cnt[slot] = 0u;  // nys_filter_finish's per-pixel chunk counter
                    sv[e] = -1.f;
                  }
                }
              }
              *reinterpret_cast<float4*>(ssh + pxo + o * 32) = make_float4(sv[0], sv[1], sv[2], sv[3]);
            }
          }
          __syncthreads();
        }
        if (c < n) {
          const float eps = eps_den;
#pragma unroll
          for (int o = 0; o < K3_YR; ++o) {
            const int row = t0 + run * K3_YR + o;
            if (row >= a.out0 + a.out_rows || row >= H) continue;
            const float4 d4 = *reinterpret_cast<const float4*>(dsh + pxo + o * 32);
            const float4 l4 = *reinterpret_cast<const float4*>(lsh + pxo + o * 32);
            const float dv[4] = {d4.x, d4.y, d4.z, d4.w}, lv[4] = {l4.x, l4.y, l4.z, l4.w};
            float res[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int x = x0 + quad * 4 + e;
              if (fabsf(dv[e]) >= eps) {
                res[e] = acc[o][e] / dv[e];
              } else if (fabsf(lv[e]) >= eps) {
                res[e] = lg[o][e] / lv[e];
              } else {
                res[e] = x < W ? __ldg(a.f + (long long)c * a.fps + (long long)row * W + x) : 0.f;
              }
            }
            if (a.out64) {  // FP64 planes (the reference's Image dtype), e.g. page-locked host memory
              double* d64 = reinterpret_cast<double*>(a.out) + (long long)c * a.ops + (long long)row * W + x0 + quad * 4;
#pragma unroll
              for (int e = 0; e < 4; ++e)
                if (x0 + quad * 4 + e < W) d64[e] = (double)res[e];
              continue;
            }
            float* dst = a.out + (long long)c * a.ops + (long long)row * W + x0 + quad * 4;
            if (a.vec_out && x0 + quad * 4 + 3 < W) {
              *reinterpret_cast<float4*>(dst) = make_float4(res[0], res[1], res[2], res[3]);
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e)
                if (x0 + quad * 4 + e < W) dst[e] = res[e];
            }
          }
        }
#pragma unroll
        for (int o = 0; o < K3_YR; ++o) acc[o][0] = acc[o][1] = acc[o][2] = acc[o][3] = 0.f;
        // first landmark of the next chunk (gmode 1)
        if (gmode == 1 && co + 1 < nchunks) compute_b(0, bsh, false);
      }
      __syncthreads();  // everyone is done with this stage's buffer (and the next b tile is ready)
      if (tid == 0) {
        // keep K3_NS stages in flight, running ahead into this CTA's next tile; stage
        // sn = s + K3_NS is (co2, i2) from the incremental counters (no per-stage division)
        int i2 = i + K3_NS, co2 = co;
        while (i2 >= L) {
          i2 -= L;
          ++co2;
        }
        if (co2 < nchunks)
          issue_at(tx, ty, i2, chunk_of(co2), gs + K3_NS);
        else if (tile + (int)gridDim.x < ntiles && (co2 - nchunks) * L + i2 < nstages)
          issue_at(ntx, nty, i2, chunk_of(co2 - nchunks), gs + K3_NS);
      }
    }
    // guard statistics from the eta tile (deterministic block reduction, atomics across blocks)
    float my_min = INFINITY;
    unsigned long long my_cnt = 0;
    for (int k = tid; k < K3_NPX; k += K3_THREADS) {
      const int row = t0 + (k >> 5), x = x0 + (k & 31);
      if (row < a.out0 + a.out_rows && row < H && x < W && ssh[k] >= 0.f) {
        const float ad = fabsf(dsh[k]);
        my_min = fminf(my_min, ad);
        my_cnt += ad < eps_den ? 1ull : 0ull;
      }
    }
    my_min = warp_min(my_min);
    my_cnt = warp_sum_u64(my_cnt);
    if ((tid & 31) == 0) {
      red_min[tid >> 5] = my_min;
      red_cnt[tid >> 5] = my_cnt;
    }
    __syncthreads();
    if (tid == 0) {
      float mn = INFINITY;
      unsigned long long cnt = 0;
      for (int w = 0; w < K3_THREADS / 32; ++w) {
        mn = fminf(mn, red_min[w]);
        cnt += red_cnt[w];
      }
      if (mn < INFINITY) atomicMin(&a.stats->min_abs_eta_bits, __float_as_uint(mn));
      if (cnt) atomicAdd(&a.stats->guarded, cnt);
    }
    // (the next tile's first barrier orders these reads of dsh before its writes)
  }
}

}  // namespace nys

using namespace nys;

extern "C" {

int nys_filter_vpass(const nys_filter_desc* d, const float* f, int64_t f_plane_stride, const float* guide,
                     int64_t guide_plane_stride, const float* planes, int64_t planes_stride, int out0, int out_rows,
                     float* out, int64_t out_plane_stride, const void* workspace, void* stream) {
  int st = validate_tiled(d);
  if (st) return st;
  if (!f || !planes || !out || !workspace || (d->guide_kind == 0 && !guide)) return NYS_EINVAL;
  if (out0 < 0 || out_rows < 1 || out0 + out_rows > d->H) return NYS_EINVAL;
  const int vrows = out_rows + 2 * d->radius;
  if (planes_stride < plane_row_stride(d->W, buffer_planes(d)) || (planes_stride & 3)) return NYS_EINVAL;
  const FilterLayout L = filter_layout(d);
  const int NC = d->n + 1;
  const int nchunks = (int)ceil_div(NC, 4);
  const int R = d->radius;
  if (K3_TH + 2 * R > 256) return NYS_EUNSUPPORTED;  // TMA box limit
  VArgs a;
  memset(&a, 0, sizeof(a));
  a.f = f;
  a.g = d->guide_kind == 0 ? guide : f;
  a.out = out;
  a.cst = reinterpret_cast<const float*>(workspace);
  a.stats = reinterpret_cast<FilterStats*>((char*)const_cast<void*>(workspace) + L.stats_off_bytes);
  a.fps = f_plane_stride;
  a.gps = d->guide_kind == 0 ? guide_plane_stride : f_plane_stride;
  a.ops = out_plane_stride;
  a.n = d->n;
  a.rho = d->rho;
  a.rhop = L.rhop;
  a.H = d->H;
  a.W = d->W;
  a.m0 = d->m0;
  a.R = R;
  a.box = d->spatial_kind == NYS_SPATIAL_BOX;
  a.gkind = d->guide_kind;
  a.out0 = out0;
  a.out_rows = out_rows;
  a.tiles_x = (int)ceil_div(d->W, 32);
  a.tiles_y = (int)ceil_div(out_rows, K3_TH);
  a.nchunks = nchunks;
  a.ntail = NC % 4;
  a.u0_off = (int)L.off_U0;
  a.out64 = d->out_f64 != 0;
  a.vec_out = ((d->W & 3) == 0) && ((out_plane_stride & 3) == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
  a.rlo = std::max(0, d->row_lo);
  a.rhi = d->row_hi > 0 ? std::min(d->H, d->row_hi) : d->H;
  a.k2 = k2_of(d);
  a.sc_off = (int)L.off_SC;
  refine_params(&a.tau, &a.cerr);
  a.flag_list = reinterpret_cast<unsigned*>((char*)const_cast<void*>(workspace) + L.list_off_bytes);
  a.list_cap = L.list_cap;
  a.chunk_cnt = reinterpret_cast<unsigned*>((char*)const_cast<void*>(workspace) + L.cnt_off_bytes);
  fill_taps(d, a.taps);
  fill_tap_pairs(a.taps, 2 * d->radius + 1, a.wpair);

  // TMA descriptors over the plane buffer: (32 cols, plane, x/32 tile, virtual row),
  // boxes of 32 x 4 x 1 x (TH+2R) planes, 32 x ntail x 1 x (TH+2R) for a partial
  // last chunk, and 32 x 1 x 1 x TH for K2's raw b planes (centre rows only)
  auto enc = encode_fn();
  if (!enc) return NYS_EUNSUPPORTED;
  const int P = buffer_planes(d);
  CUtensorMap tmap4, tmapt, tmapb;
  const cuuint64_t gdim[4] = {32, (cuuint64_t)P, (cuuint64_t)(wpad32(d->W) / 32), (cuuint64_t)vrows};
  const cuuint64_t gstr[3] = {32 * 4, (cuuint64_t)P * 32 * 4, (cuuint64_t)planes_stride * 4};
  const cuuint32_t box4[4] = {32, 4, 1, (cuuint32_t)(K3_TH + 2 * R)};
  const cuuint32_t boxt[4] = {32, (cuuint32_t)std::max(1, a.ntail), 1, (cuuint32_t)(K3_TH + 2 * R)};
  const cuuint32_t boxb[4] = {32, 1, 1, (cuuint32_t)K3_TH};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  auto encode = [&](CUtensorMap* m, const cuuint32_t* box) {
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(planes), gdim, gstr, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  if (!encode(&tmap4, box4) || !encode(&tmapt, boxt) || !encode(&tmapb, boxb)) return NYS_EINVAL;

  a.gcache = use_bplanes(d) ? 3 : 1;  // b planes from K2, or a planar guide tile (rho <= 8)
  const size_t plane_floats = (size_t)(K3_TH + 2 * R) * 32;
  const size_t stage_floats = 4 * plane_floats + (a.gcache == 3 ? K3_NPX : 0);
  const size_t smem = ((size_t)K3_NS * stage_floats + (a.gcache == 1 ? 2 * K3_NPX : 0) + 3 * K3_NPX +
                       (a.gcache == 1 ? (size_t)d->m0 * L.rhop : 0) + ((d->m0 + 3) & ~3) +
                       (a.gcache == 1 ? (size_t)d->rho * K3_NPX + K3_NPX : 0)) *
                      sizeof(float);
  if (smem > 227 * 1024) return NYS_EUNSUPPORTED;
  const long long ntiles = (long long)a.tiles_x * a.tiles_y;
  const int per_sm = smem + 2048 <= 114 * 1024 ? 2 : 1;
  const int grid = (int)std::min<long long>(ntiles, (long long)num_sms() * per_sm);
  cudaStream_t s = (cudaStream_t)stream;
  auto go = [&](auto kern) -> int {
    NYS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    NYS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    count_launch();
    kern<<<grid, K3_THREADS, smem, s>>>(tmap4, tmapt, tmapb, a);
    NYS_LAUNCH_CHECK();
    return NYS_OK;
  };
  const int rsel = a.box ? 0 : d->radius;
  if (a.gcache == 1) {
    switch (rsel) {
      case 9: return go(k_vpass<9, true>);
      case 12: return go(k_vpass<12, true>);
      case 15: return go(k_vpass<15, true>);
      case 18: return go(k_vpass<18, true>);
      default: return go(k_vpass<0, true>);
    }
  }
  switch (rsel) {
    case 9: return go(k_vpass<9, false>);
    case 12: return go(k_vpass<12, false>);
    case 15: return go(k_vpass<15, false>);
    case 18: return go(k_vpass<18, false>);
    default: return go(k_vpass<0, false>);
  }
}

}  // extern "C"
