// Shared pieces of the K2/K3 filter kernels (layout, guide access, host helpers).
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "nys_common.cuh"

namespace nys {

// ---------------------------------------------------------------------------
// constants block in the workspace (float offsets)
// ---------------------------------------------------------------------------
// FP64 block (float offset off_D, 8-byte aligned) for the near-guard refinement
// (nys_filter_finish): C64 [m0 x rho], U064 [m0], SC64 {1/alpha_1, eps_den, alpha_1, 0};
// then, past the Cholesky slot, M64 [m0 x m0] (the y-form M, or P^T P in the
// phi-form) and the list of flagged pixels (uint32 global pixel indices).
struct FilterLayout {
  int m0, rho, rhop, m0q;  // rhop: rho padded to 4; m0q: (m0+1) padded to 8
  size_t off_C, off_MT, off_U0, off_SC, off_D, n_floats;  // SC: {1/alpha_1, eps_den} read by K3
  size_t d_C64, d_U064, d_SC64;                           // double offsets from off_D
  size_t stats_off_bytes, chol_off_bytes, m64_off_bytes, list_off_bytes, cnt_off_bytes, part_off_bytes, total_bytes;
  unsigned list_cap;
};
// near-guard refinement: at most kRefineCap queued pixels per filter (the rest keep their FP32
// result and are reported), each pixel's window split over up to kRefineChunks CTAs
constexpr long long kRefineCap = 32768;
constexpr int kRefineChunks = 4;

inline FilterLayout filter_layout(const nys_filter_desc* d) {
  FilterLayout L;
  L.m0 = d->m0;
  L.rho = d->rho;
  L.rhop = (int)ceil_div(d->rho, 4) * 4;
  L.m0q = (int)ceil_div(d->m0 + 1, 8) * 8;
  L.off_C = 0;
  L.off_MT = L.off_C + (size_t)d->m0 * L.rhop;
  L.off_U0 = L.off_MT + (size_t)d->m0 * L.m0q;
  L.off_SC = L.off_U0 + (size_t)ceil_div(d->m0, 4) * 4;
  L.off_D = L.off_SC + 4;  // multiple of 4 floats: 16-byte aligned
  L.d_C64 = 0;
  L.d_U064 = (size_t)d->m0 * d->rho;
  L.d_SC64 = L.d_U064 + d->m0;
  L.n_floats = L.off_D + 2 * (L.d_SC64 + 4);
  L.n_floats = (L.n_floats + 3) & ~size_t(3);
  L.stats_off_bytes = ((L.n_floats * 4 + 255) / 256) * 256;
  L.chol_off_bytes = L.stats_off_bytes + 256;
  L.m64_off_bytes = L.chol_off_bytes + ((size_t)d->m0 * d->m0 * 8 + 255) / 256 * 256;
  L.list_off_bytes = L.m64_off_bytes + ((size_t)d->m0 * d->m0 * 8 + 255) / 256 * 256;
  const long long px = (long long)d->H * d->W;
  L.list_cap = (unsigned)std::min<long long>(px, kRefineCap);
  // per queued pixel: a chunk counter, then kRefineChunks x 2(n+1) FP64 window partial sums
  L.cnt_off_bytes = L.list_off_bytes + ((size_t)L.list_cap * 4 + 255) / 256 * 256;
  L.part_off_bytes = L.cnt_off_bytes + ((size_t)L.list_cap * 4 + 255) / 256 * 256;
  L.total_bytes = L.part_off_bytes + (size_t)L.list_cap * kRefineChunks * 2 * (d->n + 1) * sizeof(double);
  return L;
}

inline int wpitch(int W) { return (int)ceil_div(W, 4) * 4; }
// plane buffer: [virtual row][x / 32][plane][32] -> one K2 tile writes one
// contiguous block, and one K3 TMA box row is 4 planes x 32 columns = 512 B
inline int wpad32(int W) { return (int)ceil_div(W, 32) * 32; }
inline int64_t plane_row_stride(int W, int nplanes) { return (int64_t)wpad32(W) * nplanes; }
// K2 also stores the raw features b_i (one plane per landmark, after the
// (m0+1)(n+1) filtered planes) when recomputing them at the centre pixel in
// K3 would be expensive: high-dimensional guides and the NLM patch guide
inline bool use_bplanes(const nys_filter_desc* d) { return d->guide_kind == 1 || d->rho > 8 || d->phi_form; }
inline int buffer_planes(const nys_filter_desc* d) {
  return (d->m0 + 1) * (d->n + 1) + (use_bplanes(d) ? d->m0 : 0);
}

struct FilterStats {
  unsigned int min_abs_eta_bits;  // float bits, non-negative => integer order
  unsigned int flagged;           // pixels K3 queued for the FP64 near-guard refinement
  unsigned long long guarded;
  unsigned int finish_done;       // k_finish: CTAs done (the last one publishes)
  unsigned int refined_guarded;   // guarded pixels among the refined ones (diagnostics)
  unsigned int gate_timeout;      // the in-stream plan's gate timed out (outputs invalid)
  unsigned int pad;
};
static_assert(sizeof(FilterStats) == 32, "reset_filter_stats writes 8 words");

// K3's near-guard flag rule.  eta (FP32), its
// absolute scale S = sum_i b_i |conv(y_i)| and the lead denominator; a pixel is
// re-evaluated in FP64 when its ratio is ill-conditioned in FP32 (|eta| < tau S)
// or a guard decision could flip within the FP32 error bound cerr * S.
__device__ __forceinline__ bool near_guard(float eta, float S, float eta_lead, float eps, float tau, float cerr) {
  const float ad = fabsf(eta), al = fabsf(eta_lead);
  if (!(ad == ad) || !(al == al)) return true;
  if (ad >= eps) return ad < tau * S || ad - cerr * S < eps;
  return ad + cerr * S >= eps || fabsf(al - eps) <= 1e-3f * eps;
}

// guide coordinate d of pixel (row, x): planar guide or an on-the-fly 3x3 patch
// of f (channel, dy, dx order, edge replicate: filters.py:174-181)
__device__ __forceinline__ float guide_at(const float* __restrict__ g, long long gps,
                                          const float* __restrict__ f, long long fps, int gkind,
                                          int d, int row, int x, int H, int W) {
  if (gkind == 0) return __ldg(g + (long long)d * gps + (long long)row * W + x);
  const int c = d / 9, k = d - c * 9, dy = k / 3 - 1, dx = k - (k / 3) * 3 - 1;
  const int yy = clampi(row + dy, 0, H - 1), xx = clampi(x + dx, 0, W - 1);
  return __ldg(f + (long long)c * fps + (long long)yy * W + xx);
}

// host helpers
inline int num_sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

inline int validate(const nys_filter_desc* d) {
  if (!d) return NYS_EINVAL;
  if (d->n < 1 || d->n > NYS_MAX_CHANNELS_WIDE || d->rho < 1 || d->rho > NYS_MAX_RHO_WIDE) return NYS_EUNSUPPORTED;
  if (d->H < 1 || d->W < 1 || d->m0 < 1 || d->m0 > NYS_MAX_M0) return NYS_EINVAL;
  if (d->spatial_kind == NYS_SPATIAL_GAUSSIAN_RECURSIVE) {
    // radius unused (the recursion spans whole rows / columns); sigma < 1 is
    // served by the FIR path (spatial.py:206-208)
    if (!(d->sigma >= 1.0) || !std::isfinite(d->sigma)) return NYS_EINVAL;
  } else {
    if (d->radius < 0 || d->radius > NYS_MAX_RADIUS) return NYS_EUNSUPPORTED;
    if (d->spatial_kind != NYS_SPATIAL_BOX && d->spatial_kind != NYS_SPATIAL_GAUSSIAN_FIR) return NYS_EUNSUPPORTED;
  }
  if (d->spatial_kind == NYS_SPATIAL_GAUSSIAN_FIR && (!(d->sigma > 0) || d->radius < 1)) return NYS_EINVAL;
  if (!(d->theta > 0)) return NYS_EINVAL;
  if (d->guide_kind != 0 && d->guide_kind != 1) return NYS_EINVAL;
  if (d->guide_kind == 1 && d->rho != 9 * d->n) return NYS_EINVAL;
  return NYS_OK;
}

// K2/K3 (tiled FIR / box) only
inline int validate_tiled(const nys_filter_desc* d) {
  const int st = validate(d);
  if (st) return st;
  return d->spatial_kind == NYS_SPATIAL_GAUSSIAN_RECURSIVE ? NYS_EINVAL : NYS_OK;
}

// FIR tap pairs for the packed (f32x2) FIR: wpair[k] = (w[k], w[k-1]) with
// w[-1] = w[T] = 0, so output pair (o, o+1) takes input s with k = s - o:
// lane 0 accumulates w[s-o] v[s], lane 1 w[s-o-1] v[s] -- the same FMAs, in
// the same order, as the scalar loop (bit-identical results)
inline void fill_tap_pairs(const float* taps, int T, float2* wpair) {
  for (int k = 0; k <= NYS_MAX_TAPS; ++k) wpair[k] = make_float2(0.f, 0.f);
  for (int k = 0; k <= T; ++k) wpair[k] = make_float2(k < T ? taps[k] : 0.f, k >= 1 ? taps[k - 1] : 0.f);
}

// acc(lane0, lane1) += (v * w.x, v * w.y): one FFMA2 (v broadcast from a
// 32-bit register, the weight pair from a uniform register) = two FP32 FMAs
// in one issue slot
__device__ __forceinline__ unsigned long long ffma2_bc(float v, float2 w, unsigned long long acc) {
  unsigned long long vv, ww;
  asm("mov.b64 %0, {%1, %1};" : "=l"(vv) : "f"(v));
  asm("mov.b64 %0, {%1, %2};" : "=l"(ww) : "f"(w.x), "f"(w.y));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(vv), "l"(ww));
  return acc;
}
// (a0 b0, a1 b1) as one packed multiply
__device__ __forceinline__ void mul2(float a0, float a1, float b0, float b1, float& r0, float& r1) {
  unsigned long long a, b, r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(b) : "f"(b0), "f"(b1));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r0), "=f"(r1) : "l"(r));
}
__device__ __forceinline__ void unpack2(unsigned long long v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}

inline void fill_taps(const nys_filter_desc* d, float* taps) {
  const int T = 2 * d->radius + 1;
  for (int t = 0; t < NYS_MAX_TAPS; ++t) taps[t] = 0.f;
  for (int t = 0; t < T; ++t) {
    if (d->spatial_kind == NYS_SPATIAL_BOX) {
      taps[t] = 1.f;
    } else {
      const double u = (double)(t - d->radius);
      taps[t] = (float)std::exp(-(u * u) / (2.0 * d->sigma * d->sigma));  // spatial.py:72-75
    }
  }
}

// Near-guard flag rule constants for K3 (near_guard): tau bounds the FP32
// conditioning |eta| / S of the ratio, cerr * S the FP32 error of eta.  Defaults
// from the full-size cfg 3 sweep; NYS_REFINE_TAU / NYS_REFINE_CERR
// override them (0 / 0 disables the refinement: A/B switch).
inline void refine_params(float* tau, float* cerr) {  // read per launch (A/B within a process)
  const char* et = getenv("NYS_REFINE_TAU");
  const char* ec = getenv("NYS_REFINE_CERR");
  *tau = et ? (float)atof(et) : 0.25f;
  *cerr = ec ? (float)atof(ec) : 1e-3f;
}

inline float k2_of(const nys_filter_desc* d) {
  return (float)(-1.4426950408889634 / (2.0 * d->theta * d->theta));
}

inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

}  // namespace nys
