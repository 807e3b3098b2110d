// K2 pieces shared by the SIMT-GEMM kernel (nys_hpass.cu) and the tcgen05
// kernel (nys_hpass_tc.cu): launch arguments and the horizontal FIR item.
#pragma once

#include "nys_filter_common.cuh"

namespace nys {

// ---------------------------------------------------------------------------
// K2: features b, y = M b (+ lead s0), horizontal pass
// ---------------------------------------------------------------------------
constexpr int K2_THREADS = 256;  // two CTAs per SM: one fills in while the other waits at a phase barrier
constexpr int K2_XR = 16;  // output columns per FIR item
constexpr int K2_CC = 4;   // planes per FIR item

struct HArgs {
  const float* f;
  const float* g;
  float* hp;
  const float* cst;
  long long fps, gps, rs;  // rs: plane-buffer row stride (floats)
  int n, rho, rhop, H, W, m0, m0q, R, box, gkind;
  int v0, vrows, TW, pitch, tiles_x, rpt;  // rpt: virtual rows per tile
  int rlo, rhi;  // image rows present in f / guide (reads are clamped into them)
  int npl, bplanes;  // planes per buffer row block; store raw b_i planes after the filtered ones
  int phi;           // phi-form: store y_i (= phi_i) in the feature-plane slots instead of b_i
  int ku, nu, tcols, nbuf;  // tcgen05 path: K (m0 padded to 8), N ((m0+1) padded to 16), TMEM columns per group, y/f buffers
  int sc, kw;               // (unused: the removed tensor-core FIR variant's tile geometry; kept so the struct, and with it
                            // the kernels' parameter layout and register allocation, stay as measured)
  int bfrom;                // wide guides (rho > NYS_MAX_RHO): the features were written as b planes by
                            // k_bplanes_wide; K2 reads them instead of evaluating the guide
  int dbg;  // debug: bit0 skip features, bit1 skip GEMM, bit2 skip FIR math, bit3 skip stores
  float k2;
  float taps[NYS_MAX_TAPS];
  float2 wpair[NYS_MAX_TAPS + 1];  // packed-FIR tap pairs (fill_tap_pairs)
};

// FEXT: Fs holds a row per plane channel of every chunk (f_c, then 1 for the
// y plane, then 0 padding), so a plane value is always one FMUL y * Fs[c]
template <int RT, bool FEXT = false>
__device__ __forceinline__ void hfir(const HArgs& a, const float* __restrict__ yrow,
                                     const float* __restrict__ Fs, int pitch, int xoff, int c0,
                                     float (&acc)[K2_CC][K2_XR]) {
  const int n = a.n;
  const float* fr[K2_CC];
  int mode[K2_CC];  // 0: y*f_c, 1: y, 2: no plane
#pragma unroll
  for (int cc = 0; cc < K2_CC; ++cc) {
    const int c = c0 + cc;
    fr[cc] = Fs + (size_t)(FEXT ? c : min(c, n - 1)) * pitch + xoff;
    mode[cc] = FEXT ? 0 : (c < n ? 0 : (c == n ? 1 : 2));
  }
#pragma unroll
  for (int cc = 0; cc < K2_CC; ++cc)
#pragma unroll
    for (int o = 0; o < K2_XR; ++o) acc[cc][o] = 0.f;
  auto plane_val = [&](int cc, float yv, float fv) {
    if constexpr (FEXT) return yv * fv;
    return mode[cc] == 0 ? yv * fv : (mode[cc] == 1 ? yv : 0.f);
  };

  if (a.box) {  // sliding (2R+1)-sum re-anchored per item (spatial.py:91-99)
    const int R = a.R;
    float s[K2_CC];
#pragma unroll
    for (int cc = 0; cc < K2_CC; ++cc) s[cc] = 0.f;
    for (int t = 0; t <= 2 * R; ++t) {
      const float yv = yrow[t];
#pragma unroll
      for (int cc = 0; cc < K2_CC; ++cc) s[cc] += plane_val(cc, yv, fr[cc][t]);
    }
#pragma unroll
    for (int o = 0; o < K2_XR; ++o) {
      if (o > 0) {
        const float yin = yrow[o + 2 * R], yout = yrow[o - 1];
#pragma unroll
        for (int cc = 0; cc < K2_CC; ++cc)
          s[cc] += plane_val(cc, yin, fr[cc][o + 2 * R]) - plane_val(cc, yout, fr[cc][o - 1]);
      }
#pragma unroll
      for (int cc = 0; cc < K2_CC; ++cc) acc[cc][o] = s[cc];
    }
    return;
  }
  if constexpr (RT > 0) {
    constexpr int T = 2 * RT + 1;
    constexpr int NIN = K2_XR + 2 * RT;
    constexpr int NQ = (NIN + 3) / 4;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const float4 y4 = *reinterpret_cast<const float4*>(yrow + 4 * q);
      float4 f4[K2_CC];
#pragma unroll
      for (int cc = 0; cc < K2_CC; ++cc) f4[cc] = *reinterpret_cast<const float4*>(fr[cc] + 4 * q);
      const float yv[4] = {y4.x, y4.y, y4.z, y4.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int s = 4 * q + e;
        if (s < NIN) {
#pragma unroll
          for (int cc = 0; cc < K2_CC; ++cc) {
            const float fv[4] = {f4[cc].x, f4[cc].y, f4[cc].z, f4[cc].w};
            const float v = plane_val(cc, yv[e], fv[e]);
#pragma unroll
            for (int o = 0; o < K2_XR; ++o) {
              const int t = s - o;
              if (t >= 0 && t < T) acc[cc][o] = fmaf(a.taps[t], v, acc[cc][o]);
            }
          }
        }
      }
    }
  } else {
    const int T = 2 * a.R + 1;
    for (int t = 0; t < T; ++t) {
      const float w = a.taps[t];
#pragma unroll
      for (int o = 0; o < K2_XR; ++o) {
        const float yv = yrow[o + t];
#pragma unroll
        for (int cc = 0; cc < K2_CC; ++cc) acc[cc][o] = fmaf(w, plane_val(cc, yv, fr[cc][o + t]), acc[cc][o]);
      }
    }
  }
}

// One plane of a FIR item: acc[o] = sum_t taps[t] * y[o+t] * fr[o+t], o < K2_XR.
// The caller loops over the item's planes without unrolling, which keeps the
// unrolled body (~0.6k instructions for R = 15) inside the instruction cache.
template <int RT>
__device__ __forceinline__ void hfir_plane(const HArgs& a, const float* __restrict__ yrow,
                                           const float* __restrict__ frow, float (&acc)[K2_XR]) {
#pragma unroll
  for (int o = 0; o < K2_XR; ++o) acc[o] = 0.f;
  if constexpr (RT > 0) {
    // packed FIR: output pairs (2p, 2p+1) accumulate in one f32x2 register,
    // one FFMA2 per (input, pair) -- half the issue slots of scalar FFMA
    constexpr int T = 2 * RT + 1;
    constexpr int NIN = K2_XR + 2 * RT;
    constexpr int NQ = (NIN + 3) / 4;
    static_assert(K2_XR % 2 == 0, "output pairs");
    unsigned long long acc2[K2_XR / 2];
#pragma unroll
    for (int p = 0; p < K2_XR / 2; ++p) acc2[p] = 0ull;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const float4 y4 = *reinterpret_cast<const float4*>(yrow + 4 * q);
      const float4 f4 = *reinterpret_cast<const float4*>(frow + 4 * q);
      // z = y f as two packed multiplies (the LDS.128 results are adjacent register pairs)
      float v4[4];
      mul2(y4.x, y4.y, f4.x, f4.y, v4[0], v4[1]);
      mul2(y4.z, y4.w, f4.z, f4.w, v4[2], v4[3]);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int s = 4 * q + e;
        if (s < NIN) {
#pragma unroll
          for (int p = 0; p < K2_XR / 2; ++p) {
            const int k = s - 2 * p;
            if (k >= 0 && k <= T) acc2[p] = ffma2_bc(v4[e], a.wpair[k], acc2[p]);
          }
        }
      }
    }
#pragma unroll
    for (int p = 0; p < K2_XR / 2; ++p) unpack2(acc2[p], acc[2 * p], acc[2 * p + 1]);
  } else if (a.box) {  // sliding (2R+1)-sum re-anchored per item (spatial.py:91-99)
    const int R = a.R;
    float sum = 0.f;
    for (int t = 0; t <= 2 * R; ++t) sum += yrow[t] * frow[t];
#pragma unroll
    for (int o = 0; o < K2_XR; ++o) {
      if (o > 0) sum += yrow[o + 2 * R] * frow[o + 2 * R] - yrow[o - 1] * frow[o - 1];
      acc[o] = sum;
    }
  } else {
    const int T = 2 * a.R + 1;
    for (int t = 0; t < T; ++t) {
      const float w = a.taps[t];
#pragma unroll
      for (int o = 0; o < K2_XR; ++o) acc[o] = fmaf(w, yrow[o + t] * frow[o + t], acc[o]);
    }
  }
}

// tcgen05 path of K2 (nys_hpass_tc.cu): fills the tile geometry of `a` and
// launches, or returns NYS_EUNSUPPORTED when the shape does not fit it
int launch_hpass_tc(HArgs& a, const nys_filter_desc* d, cudaStream_t s);

}  // namespace nys
