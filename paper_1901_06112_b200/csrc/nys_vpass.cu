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
constexpr int K3_THREADS = 256;  // 8 column quads x 8 row runs x 4 plane groups
constexpr int K3_NS = 2;         // TMA pipeline depth (stages of up to 4 planes)

struct VArgs {
  const float* f;
  const float* g;
  float* out;
  const float* cst;
  FilterStats* stats;
  long long fps, gps, ops;
  int n, rho, rhop, H, W, m0, R, box, gkind;
  int out0, out_rows, tiles_x, tiles_y, nchunks, u0_off, vec_out, gcache;
  int rlo, rhi;  // image rows present in f / guide (reads are clamped into them)
  float k2, inv_alpha0, eps_den;
  float taps[NYS_MAX_TAPS];
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
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
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

// vertical FIR of one staged plane tile: 4 columns x YR rows per thread
template <int RT, int YR, int RS>
__device__ __forceinline__ void vfir(const VArgs& a, const float* __restrict__ src, float (&G)[YR][4]) {
#pragma unroll
  for (int o = 0; o < YR; ++o) G[o][0] = G[o][1] = G[o][2] = G[o][3] = 0.f;
  if (a.box) {
    const int R = a.R;
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int t = 0; t <= 2 * R; ++t) {
      const float4 v = *reinterpret_cast<const float4*>(src + t * RS);
      s.x += v.x;
      s.y += v.y;
      s.z += v.z;
      s.w += v.w;
    }
    G[0][0] = s.x;
    G[0][1] = s.y;
    G[0][2] = s.z;
    G[0][3] = s.w;
#pragma unroll
    for (int o = 1; o < YR; ++o) {
      const float4 vi = *reinterpret_cast<const float4*>(src + (o + 2 * R) * RS);
      const float4 vo = *reinterpret_cast<const float4*>(src + (o - 1) * RS);
      s.x += vi.x - vo.x;
      s.y += vi.y - vo.y;
      s.z += vi.z - vo.z;
      s.w += vi.w - vo.w;
      G[o][0] = s.x;
      G[o][1] = s.y;
      G[o][2] = s.z;
      G[o][3] = s.w;
    }
    return;
  }
  if constexpr (RT > 0) {
    constexpr int T = 2 * RT + 1;
#pragma unroll
    for (int s = 0; s < YR + 2 * RT; ++s) {
      const float4 v = *reinterpret_cast<const float4*>(src + s * RS);
#pragma unroll
      for (int o = 0; o < YR; ++o) {
        const int t = s - o;
        if (t >= 0 && t < T) {
          const float w = a.taps[t];
          G[o][0] = fmaf(w, v.x, G[o][0]);
          G[o][1] = fmaf(w, v.y, G[o][1]);
          G[o][2] = fmaf(w, v.z, G[o][2]);
          G[o][3] = fmaf(w, v.w, G[o][3]);
        }
      }
    }
  } else {
    const int T = 2 * a.R + 1;
    for (int t = 0; t < T; ++t) {
      const float w = a.taps[t];
#pragma unroll
      for (int o = 0; o < YR; ++o) {
        const float4 v = *reinterpret_cast<const float4*>(src + (o + t) * RS);
        G[o][0] = fmaf(w, v.x, G[o][0]);
        G[o][1] = fmaf(w, v.y, G[o][1]);
        G[o][2] = fmaf(w, v.z, G[o][2]);
        G[o][3] = fmaf(w, v.w, G[o][3]);
      }
    }
  }
}

template <int RT, int YR, int CPT>
__global__ void __launch_bounds__(K3_THREADS) k_vpass(const __grid_constant__ CUtensorMap tmap4,
                                                     const __grid_constant__ CUtensorMap tmap1,
                                                     const __grid_constant__ CUtensorMap tmapb, const VArgs a) {
  extern __shared__ __align__(128) float sm[];
  const int tid = threadIdx.x;
  const int grp = tid >> 6, run = (tid >> 3) & 7, quad = tid & 7;
  const int m0 = a.m0, n = a.n, rho = a.rho, rhop = a.rhop, H = a.H, W = a.W, NC = n + 1;
  const int R = RT > 0 ? RT : a.R;
  const int TH = 8 * YR;           // tile rows
  const int SR = TH + 2 * R;       // staged rows per plane
  const int npx = TH * 32;
  const int nchunks = a.nchunks;
  const int plane_floats = SR * 32;
  float* stage = sm;                                      // K3_NS x 4 x SR x 32
  float* bsh = stage + (size_t)K3_NS * 4 * plane_floats;  // 2 x npx
  float* ssh = bsh + 2 * npx;                             // npx: s0 = u0 . b
  float* dsh = ssh + npx;                                 // npx: eta
  float* lsh = dsh + npx;                                 // npx: eta_lead
  float* Cs = lsh + npx;                                  // m0 x rhop
  float* U0 = Cs + (size_t)m0 * rhop;                     // m0
  // guide cache for the centre-pixel features: planar rho <= 8 -> [rho][npx];
  // 3x3 patch guide -> the f tile with a 1-pixel halo [n][TH+2][34]
  float* gsh = U0 + ((m0 + 3) & ~3);
  const int gmode = a.gcache;  // 0: global loads, 1: planar cache, 2: patch cache, 3: b planes from K2
  __shared__ __align__(8) unsigned long long full[K3_NS];
  __shared__ float red_min[K3_THREADS / 32];
  __shared__ unsigned long long red_cnt[K3_THREADS / 32];

  for (int k = tid; k < m0 * rhop; k += blockDim.x) Cs[k] = a.cst[k];
  for (int k = tid; k < m0; k += blockDim.x) U0[k] = a.cst[a.u0_off + k];
  if (tid == 0) {
    for (int b = 0; b < K3_NS; ++b) mbar_init(&full[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // stage s of a tile: landmark i = s / nchunks (i == m0: lead group), chunk k;
  // the lead group visits the chunk holding plane n first (the guard needs eta_lead)
  const int kn = n / 4;
  auto stage_chunk = [&](int s) {
    const int i = s / nchunks, kk = s - i * nchunks;
    if (i < m0) return kk;
    return kk == 0 ? kn : (kk <= kn ? kk - 1 : kk);
  };
  const int nstages = (m0 + 1) * nchunks;
  unsigned long long gstage = 0;  // running stage counter across tiles (mbarrier phases)
  const int ntiles = a.tiles_x * a.tiles_y;

  // stage = up to 4 consecutive planes of a landmark group: a full chunk is one
  // 4-plane box (SMEM [SR][4][32]); a partial last chunk is nval 1-plane boxes
  // (SMEM [nval][SR][32])
  auto issue = [&](int tx, int ty, int s, unsigned long long gs) {
    const int i = s / nchunks, k = stage_chunk(s);
    const int buf = (int)(gs % K3_NS);
    const int nval = min(4, NC - 4 * k);
    const bool with_b = gmode == 3 && i < m0 && k == 0;  // landmark i's raw b tile rides on its first chunk
    mbar_expect_tx(&full[buf], (unsigned)(nval * plane_floats * 4 + (with_b ? npx * 4 : 0)));
    if (with_b) tma_load_4d(bsh + (i & 1) * npx, &tmapb, 0, (m0 + 1) * NC + i, tx, ty * TH + R, &full[buf]);
    float* dst = stage + (size_t)buf * 4 * plane_floats;
    if (nval == 4) {
      tma_load_4d(dst, &tmap4, 0, i * NC + 4 * k, tx, ty * TH, &full[buf]);
    } else {
      for (int q = 0; q < nval; ++q)
        tma_load_4d(dst + (size_t)q * plane_floats, &tmap1, 0, i * NC + 4 * k + q, tx, ty * TH, &full[buf]);
    }
  };

  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int x0 = tx * 32, t0 = a.out0 + ty * TH;
    if (tid == 0)
      for (int s = 0; s < K3_NS && s < nstages; ++s) issue(tx, ty, s, gstage + s);
    for (int k = tid; k < npx; k += blockDim.x) ssh[k] = 0.f;
    if (gmode == 1) {
      for (int k = tid; k < rho * npx; k += blockDim.x) {
        const int d = k / npx, q = k - d * npx;
        const int rr = clampi(min(t0 + (q >> 5), H - 1), a.rlo, a.rhi - 1), cx = min(x0 + (q & 31), W - 1);
        gsh[k] = __ldg(a.g + (long long)d * a.gps + (long long)rr * W + cx);
      }
    } else if (gmode == 2) {
      for (int k = tid; k < n * (TH + 2) * 34; k += blockDim.x) {
        const int c = k / ((TH + 2) * 34), q = k - c * ((TH + 2) * 34);
        const int yy = clampi(clampi(t0 + q / 34 - 1, 0, H - 1), a.rlo, a.rhi - 1), xx = clampi(x0 + q % 34 - 1, 0, W - 1);
        gsh[k] = __ldg(a.f + (long long)c * a.fps + (long long)yy * W + xx);
      }
    }
    __syncthreads();

    float acc[CPT][YR][4];
#pragma unroll
    for (int c = 0; c < CPT; ++c)
#pragma unroll
      for (int o = 0; o < YR; ++o) acc[c][o][0] = acc[c][o][1] = acc[c][o][2] = acc[c][o][3] = 0.f;

    const int pxo = run * YR * 32 + quad * 4;  // this thread's first pixel in tile order (row-major, 32 wide)
    int s = 0;
    for (int i = 0; i <= m0; ++i) {
      if (i < m0 && gmode != 3) {
        // b_i at every tile pixel (and the lead projection s0 += u0_i b_i)
        float* bb = bsh + (i & 1) * npx;
        const float u0i = U0[i];
        if (gmode == 1) {
          // 4 neighbouring pixels per thread step: independent chains, 128-bit SMEM traffic
#pragma unroll 2
          for (int k4 = tid; k4 < npx / 4; k4 += blockDim.x) {
            float4 d2 = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int d = 0; d < rho; ++d) {
              const float4 g4 = *reinterpret_cast<const float4*>(gsh + d * npx + 4 * k4);
              const float c = Cs[i * rhop + d];
              const float tx = g4.x - c, ty = g4.y - c, tz = g4.z - c, tw = g4.w - c;
              d2.x = fmaf(tx, tx, d2.x);
              d2.y = fmaf(ty, ty, d2.y);
              d2.z = fmaf(tz, tz, d2.z);
              d2.w = fmaf(tw, tw, d2.w);
            }
            const float4 b4 = make_float4(range_kernel(d2.x, a.k2), range_kernel(d2.y, a.k2),
                                          range_kernel(d2.z, a.k2), range_kernel(d2.w, a.k2));
            *reinterpret_cast<float4*>(bb + 4 * k4) = b4;
            float4 s4 = *reinterpret_cast<float4*>(ssh + 4 * k4);
            s4.x = fmaf(u0i, b4.x, s4.x);
            s4.y = fmaf(u0i, b4.y, s4.y);
            s4.z = fmaf(u0i, b4.z, s4.z);
            s4.w = fmaf(u0i, b4.w, s4.w);
            *reinterpret_cast<float4*>(ssh + 4 * k4) = s4;
          }
        } else {
          for (int k = tid; k < npx; k += blockDim.x) {
            float d2 = 0.f;
            if (gmode == 2) {
              const int ty0 = k >> 5, tx0 = k & 31;
              for (int d = 0; d < rho; ++d) {
                const int c = d / 9, q = d - c * 9, dy = q / 3, dx = q - (q / 3) * 3;
                const float t = gsh[(c * (TH + 2) + ty0 + dy) * 34 + tx0 + dx] - Cs[i * rhop + d];
                d2 = fmaf(t, t, d2);
              }
            } else {
              const int rr = clampi(min(t0 + (k >> 5), H - 1), a.rlo, a.rhi - 1);
              const int cx = min(x0 + (k & 31), W - 1);
              for (int d = 0; d < rho; ++d) {
                const float t = guide_at(a.g, a.gps, a.f, a.fps, a.gkind, d, rr, cx, H, W) - Cs[i * rhop + d];
                d2 = fmaf(t, t, d2);
              }
            }
            const float b = range_kernel(d2, a.k2);
            bb[k] = b;
            ssh[k] = fmaf(u0i, b, ssh[k]);
          }
        }
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < CPT; ++kk) {
        if (kk < nchunks) {
          const unsigned long long gs = gstage + s;
          const int buf = (int)(gs % K3_NS);
          mbar_wait(&full[buf], (unsigned)((gs / K3_NS) & 1));
          if (gmode == 3 && i < m0 && kk == 0) {
            const float u0i = U0[i];
            const float* bb = bsh + (i & 1) * npx;
            for (int q = tid; q < npx / 4; q += blockDim.x) {
              const float4 b4 = *reinterpret_cast<const float4*>(bb + 4 * q);
              float4 s4 = *reinterpret_cast<float4*>(ssh + 4 * q);
              s4.x = fmaf(u0i, b4.x, s4.x);
              s4.y = fmaf(u0i, b4.y, s4.y);
              s4.z = fmaf(u0i, b4.z, s4.z);
              s4.w = fmaf(u0i, b4.w, s4.w);
              *reinterpret_cast<float4*>(ssh + 4 * q) = s4;
            }
          }
          const int k = stage_chunk(s);
          const int c = 4 * k + grp;
          float G[YR][4];
          if (c < NC) {
            const float* sb = stage + (size_t)buf * 4 * plane_floats;
            if (4 * k + 4 <= NC)
              vfir<RT, YR, 128>(a, sb + grp * 32 + run * YR * 128 + quad * 4, G);
            else
              vfir<RT, YR, 32>(a, sb + (size_t)grp * plane_floats + pxo, G);
          }
          if (i < m0) {
            const float* bb = bsh + (i & 1) * npx + pxo;
#pragma unroll
            for (int o = 0; o < YR; ++o) {
              const float4 b4 = *reinterpret_cast<const float4*>(bb + o * 32);
              acc[kk][o][0] = fmaf(b4.x, G[o][0], acc[kk][o][0]);
              acc[kk][o][1] = fmaf(b4.y, G[o][1], acc[kk][o][1]);
              acc[kk][o][2] = fmaf(b4.z, G[o][2], acc[kk][o][2]);
              acc[kk][o][3] = fmaf(b4.w, G[o][3], acc[kk][o][3]);
            }
          } else {
            // lead group: zeta_lead = s0 (ω*(s0 f_c)) / α0 ; chunk kn first publishes eta and eta_lead
            float lg[YR][4];
#pragma unroll
            for (int o = 0; o < YR; ++o) {
              const float4 s4 = *reinterpret_cast<const float4*>(ssh + pxo + o * 32);
              lg[o][0] = s4.x * G[o][0] * a.inv_alpha0;
              lg[o][1] = s4.y * G[o][1] * a.inv_alpha0;
              lg[o][2] = s4.z * G[o][2] * a.inv_alpha0;
              lg[o][3] = s4.w * G[o][3] * a.inv_alpha0;
            }
            // numerator set of channel c = 4k + grp: acc[k] (selected without dynamic indexing)
            float A[YR][4];
#pragma unroll
            for (int o = 0; o < YR; ++o)
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                float v = 0.f;
#pragma unroll
                for (int q = 0; q < CPT; ++q) v = (q == k) ? acc[q][o][e] : v;
                A[o][e] = v;
              }
            if (kk == 0) {
              if (c == n) {
#pragma unroll
                for (int o = 0; o < YR; ++o) {
                  *reinterpret_cast<float4*>(dsh + pxo + o * 32) = make_float4(A[o][0], A[o][1], A[o][2], A[o][3]);
                  *reinterpret_cast<float4*>(lsh + pxo + o * 32) = make_float4(lg[o][0], lg[o][1], lg[o][2], lg[o][3]);
                }
              }
              __syncthreads();
            }
            if (c < n) {
              const float eps = a.eps_den;
#pragma unroll
              for (int o = 0; o < YR; ++o) {
                const int row = t0 + run * YR + o;
                if (row >= a.out0 + a.out_rows || row >= H) continue;
                const float4 d4 = *reinterpret_cast<const float4*>(dsh + pxo + o * 32);
                const float4 l4 = *reinterpret_cast<const float4*>(lsh + pxo + o * 32);
                const float dv[4] = {d4.x, d4.y, d4.z, d4.w}, lv[4] = {l4.x, l4.y, l4.z, l4.w};
                float res[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const int x = x0 + quad * 4 + e;
                  if (fabsf(dv[e]) >= eps) {
                    res[e] = A[o][e] / dv[e];
                  } else if (fabsf(lv[e]) >= eps) {
                    res[e] = lg[o][e] / lv[e];
                  } else {
                    res[e] = x < W ? __ldg(a.f + (long long)c * a.fps + (long long)row * W + x) : 0.f;
                  }
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
          }
          __syncthreads();  // everyone is done with this stage's buffer
          if (tid == 0 && s + K3_NS < nstages) issue(tx, ty, s + K3_NS, gstage + s + K3_NS);
          ++s;
        }
      }
    }
    gstage += nstages;
    // guard statistics from the eta tile (deterministic block reduction, atomics across blocks)
    float my_min = INFINITY;
    unsigned long long my_cnt = 0;
    for (int k = tid; k < npx; k += blockDim.x) {
      const int row = t0 + (k >> 5), x = x0 + (k & 31);
      if (row < a.out0 + a.out_rows && row < H && x < W) {
        const float ad = fabsf(dsh[k]);
        my_min = fminf(my_min, ad);
        my_cnt += ad < a.eps_den ? 1ull : 0ull;
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
    __syncthreads();
  }
}

}  // namespace nys

using namespace nys;

extern "C" {

int nys_filter_vpass(const nys_filter_desc* d, const float* f, int64_t f_plane_stride, const float* guide,
                     int64_t guide_plane_stride, const float* planes, int64_t planes_stride, int out0, int out_rows,
                     float* out, int64_t out_plane_stride, const void* workspace, void* stream) {
  int st = validate(d);
  if (st) return st;
  if (!f || !planes || !out || !workspace || (d->guide_kind == 0 && !guide)) return NYS_EINVAL;
  if (out0 < 0 || out_rows < 1 || out0 + out_rows > d->H) return NYS_EINVAL;
  const int vrows = out_rows + 2 * d->radius;
  if (planes_stride < plane_row_stride(d->W, buffer_planes(d)) || (planes_stride & 3)) return NYS_EINVAL;
  const FilterLayout L = filter_layout(d);
  const int NC = d->n + 1;
  const int nchunks = (int)ceil_div(NC, 4);
  // accumulator sets per thread (CPT) and rows per thread (YR) from the channel count
  int YR, CPT;
  if (nchunks <= 1) {
    YR = 8;
    CPT = 1;
  } else if (nchunks <= 2) {
    YR = 8;
    CPT = 2;
  } else if (nchunks <= 5) {
    YR = 8;
    CPT = 5;
  } else if (nchunks <= 8) {
    YR = 4;
    CPT = 8;
  } else {
    YR = 2;
    CPT = 17;
  }
  if (nchunks > CPT) return NYS_EUNSUPPORTED;
  const int TH = 8 * YR;
  const int R = d->radius;
  if (TH + 2 * R > 256) return NYS_EUNSUPPORTED;  // TMA box limit
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
  a.tiles_y = (int)ceil_div(out_rows, TH);
  a.nchunks = nchunks;
  a.u0_off = (int)L.off_U0;
  a.vec_out = ((d->W & 3) == 0) && ((out_plane_stride & 3) == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
  a.rlo = std::max(0, d->row_lo);
  a.rhi = d->row_hi > 0 ? std::min(d->H, d->row_hi) : d->H;
  a.k2 = k2_of(d);
  a.inv_alpha0 = (float)(1.0 / d->alpha0);
  a.eps_den = (float)d->eps_den;
  fill_taps(d, a.taps);

  // TMA descriptors over the plane buffer: (32 cols, plane, x/32 tile, virtual row),
  // boxes of 32 x 4 x 1 x (TH+2R) and 32 x 1 x 1 x (TH+2R)
  auto enc = encode_fn();
  if (!enc) return NYS_EUNSUPPORTED;
  const int P = buffer_planes(d);
  CUtensorMap tmap4, tmap1, tmapb;
  const cuuint64_t gdim[4] = {32, (cuuint64_t)P, (cuuint64_t)(wpad32(d->W) / 32), (cuuint64_t)vrows};
  const cuuint64_t gstr[3] = {32 * 4, (cuuint64_t)P * 32 * 4, (cuuint64_t)planes_stride * 4};
  const cuuint32_t box4[4] = {32, 4, 1, (cuuint32_t)(TH + 2 * R)};
  const cuuint32_t box1[4] = {32, 1, 1, (cuuint32_t)(TH + 2 * R)};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  if (enc(&tmap4, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(planes), gdim, gstr, box4, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
      enc(&tmap1, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(planes), gdim, gstr, box1, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return NYS_EINVAL;
  const cuuint32_t boxb[4] = {32, 1, 1, (cuuint32_t)TH};  // centre rows only
  if (enc(&tmapb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(planes), gdim, gstr, boxb, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return NYS_EINVAL;

  const int npx = TH * 32;
  a.gcache = use_bplanes(d) ? 3 : 1;  // b planes from K2, or a planar guide tile (rho <= 8)
  const size_t gfloats = a.gcache == 1 ? (size_t)d->rho * npx : (a.gcache == 2 ? (size_t)d->n * (TH + 2) * 34 : 0);
  const size_t smem = ((size_t)K3_NS * 4 * (TH + 2 * R) * 32 + 5 * (size_t)npx + (size_t)d->m0 * L.rhop +
                       ((d->m0 + 3) & ~3) + gfloats) *
                      sizeof(float);
  if (smem > 227 * 1024) return NYS_EUNSUPPORTED;
  const long long ntiles = (long long)a.tiles_x * a.tiles_y;
  const int grid = (int)std::min<long long>(ntiles, (long long)num_sms() * 2);
  cudaStream_t s = (cudaStream_t)stream;
  auto go = [&](auto kern) -> int {
    NYS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    NYS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    count_launch();
    kern<<<grid, K3_THREADS, smem, s>>>(tmap4, tmap1, tmapb, a);
    NYS_LAUNCH_CHECK();
    return NYS_OK;
  };
#define NYS_V_CPT(RV)                                   \
  switch (CPT) {                                        \
    case 1: return go(k_vpass<RV, 8, 1>);               \
    case 2: return go(k_vpass<RV, 8, 2>);               \
    case 5: return go(k_vpass<RV, 8, 5>);               \
    case 8: return go(k_vpass<RV, 4, 8>);               \
    default: return go(k_vpass<RV, 2, 17>);             \
  }
  const int rsel = a.box ? 0 : d->radius;
  switch (rsel) {
    case 9: NYS_V_CPT(9)
    case 12: NYS_V_CPT(12)
    case 15: NYS_V_CPT(15)
    case 18: NYS_V_CPT(18)
    default: NYS_V_CPT(0)
  }
#undef NYS_V_CPT
}

}  // extern "C"
