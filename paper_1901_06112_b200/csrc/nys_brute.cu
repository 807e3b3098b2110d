// Direct evaluation of the kernel filter, Eq. (1) of the paper.
//
// Reference region replaced: filters.py:107-138 (_window_weights,
// brute_force_filter): for every pixel x,
//   out(x) = Σ_d w(d) κ(p(x+d) - p(x)) f(x+d) / Σ_d w(d) κ(p(x+d) - p(x))
// over the (2S+1)^2 window, w = outer(w1, w1) with w1 the unnormalised
// Gaussian taps at S (box: ones; a recursive kernel is evaluated as its FIR
// counterpart at S = ceil(3 sigma)), κ(u) = exp(-|u|^2 / (2 θ^2)), edge
// replicate (np.pad mode="edge").
//
// Compute-bound: (2S+1)^2 (2ρ + n + 3) FP32 ops per pixel (FP32 within a
// window row, FP64 across rows).  One thread per
// output pixel; a CTA stages its (TY+2S) x (TX+2S) halo of the ρ guide and n
// input planes in shared memory when it fits (clamped once at load time), so
// the window loop is shared-memory broadcast/conflict-free reads + FMAs.
// Larger stacks read the (L1-resident) planes directly.
#include "nys_filter_common.cuh"

namespace nys {

constexpr int BF_TX = 32, BF_TY = 8;

struct BruteArgs {
  const float* f;
  long long fps;
  const float* g;
  long long gps;
  float* out;
  long long ops;
  int n, rho, H, W, S;
  float k2;
  float w1[NYS_MAX_TAPS];
};

// RM / NM: compile-time bounds of rho / n (register-resident for the small
// instantiation, local memory for the general one)
template <bool SMEM, int RM, int NM>
__global__ void __launch_bounds__(BF_TX* BF_TY) k_brute(const BruteArgs a) {
  extern __shared__ float bsm[];
  const int S = a.S, T = 2 * S + 1;
  const int tx = threadIdx.x % BF_TX, ty = threadIdx.x / BF_TX;
  const int x0 = blockIdx.x * BF_TX, y0 = blockIdx.y * BF_TY;
  const int x = x0 + tx, y = y0 + ty;
  const int HW = BF_TX + 2 * S, HH = BF_TY + 2 * S;
  const int nplanes = a.rho + a.n;
  if (SMEM) {
    // planes 0..rho-1: guide, rho..rho+n-1: f; halo rows/cols clamped (edge pad)
    for (int k = threadIdx.x; k < nplanes * HH * HW; k += blockDim.x) {
      const int pl = k / (HH * HW), r = k - pl * HH * HW, hy = r / HW, hx = r - hy * HW;
      const int yy = clampi(y0 - S + hy, 0, a.H - 1), xx = clampi(x0 - S + hx, 0, a.W - 1);
      const float* src = pl < a.rho ? a.g + (long long)pl * a.gps : a.f + (long long)(pl - a.rho) * a.fps;
      bsm[k] = __ldg(src + (long long)yy * a.W + xx);
    }
    __syncthreads();
  }
  if (x >= a.W || y >= a.H) return;
  auto at = [&](int pl, int dy, int dx) -> float {  // plane pl at (y+dy, x+dx), dy,dx in [-S,S]
    if (SMEM) return bsm[(pl * HH + ty + S + dy) * HW + tx + S + dx];
    const int yy = clampi(y + dy, 0, a.H - 1), xx = clampi(x + dx, 0, a.W - 1);
    const float* src = pl < a.rho ? a.g + (long long)pl * a.gps : a.f + (long long)(pl - a.rho) * a.fps;
    return __ldg(src + (long long)yy * a.W + xx);
  };
  float pc[RM];
#pragma unroll
  for (int d = 0; d < RM; ++d) pc[d] = d < a.rho ? at(d, 0, 0) : 0.f;
  // FP32 sums along a window row, FP64 across rows (windows reach (2*64+1)^2 terms)
  double num_d[NM], den_d = 0.0;
#pragma unroll
  for (int c = 0; c < NM; ++c) num_d[c] = 0.0;
  for (int iy = 0; iy < T; ++iy) {
    const float wy = a.w1[iy];
    float num[NM];
#pragma unroll
    for (int c = 0; c < NM; ++c) num[c] = 0.f;
    float den = 0.f;
    for (int ix = 0; ix < T; ++ix) {
      float d2 = 0.f;
#pragma unroll
      for (int d = 0; d < RM; ++d) {
        if (d < a.rho) {
          const float u = at(d, iy - S, ix - S) - pc[d];
          d2 = fmaf(u, u, d2);
        }
      }
      const float kv = range_kernel(d2, a.k2) * (wy * a.w1[ix]);
#pragma unroll
      for (int c = 0; c < NM; ++c)
        if (c < a.n) num[c] = fmaf(kv, at(a.rho + c, iy - S, ix - S), num[c]);
      den += kv;
    }
#pragma unroll
    for (int c = 0; c < NM; ++c) num_d[c] += (double)num[c];
    den_d += (double)den;
  }
#pragma unroll
  for (int c = 0; c < NM; ++c)
    if (c < a.n) a.out[(long long)c * a.ops + (long long)y * a.W + x] = (float)(num_d[c] / den_d);
}

}  // namespace nys

using namespace nys;

extern "C" int nys_brute_force_filter(const nys_filter_desc* d, const float* f, int64_t f_plane_stride,
                                      const float* guide, int64_t guide_plane_stride, float* out,
                                      int64_t out_plane_stride, void* stream) {
  int st = validate(d);
  if (!st && (d->rho > NYS_MAX_RHO || d->n > NYS_MAX_CHANNELS)) st = NYS_EUNSUPPORTED;  // register-resident
  if (st) return st;
  if (!f || !out || !guide) return NYS_EINVAL;
  if (d->guide_kind != 0) return NYS_EINVAL;  // the patch guide is materialised first (nys_patch_guide)
  BruteArgs a{};
  a.f = f;
  a.fps = f_plane_stride;
  a.g = guide;
  a.gps = guide_plane_stride;
  a.out = out;
  a.ops = out_plane_stride;
  a.n = d->n;
  a.rho = d->rho;
  a.H = d->H;
  a.W = d->W;
  // window radius S (spatial.py:66-69) and the 1-D weights (filters.py:107-113)
  const bool rec = d->spatial_kind == NYS_SPATIAL_GAUSSIAN_RECURSIVE;
  a.S = rec ? (int)std::ceil(3.0 * d->sigma) : d->radius;
  if (a.S > NYS_MAX_RADIUS) return NYS_EUNSUPPORTED;
  for (int t = 0; t < NYS_MAX_TAPS; ++t) a.w1[t] = 0.f;
  for (int t = 0; t <= 2 * a.S; ++t) {
    const double u = (double)(t - a.S);
    a.w1[t] = d->spatial_kind == NYS_SPATIAL_BOX ? 1.f : (float)std::exp(-(u * u) / (2.0 * d->sigma * d->sigma));
  }
  a.k2 = k2_of(d);
  const dim3 grid((unsigned)ceil_div(d->W, BF_TX), (unsigned)ceil_div(d->H, BF_TY));
  const size_t smem = (size_t)(d->rho + d->n) * (BF_TY + 2 * a.S) * (BF_TX + 2 * a.S) * sizeof(float);
  cudaStream_t s = (cudaStream_t)stream;
  const bool small = d->rho <= 8 && d->n <= 4;
  count_launch();
  if (smem <= 200 * 1024) {
    auto k = small ? k_brute<true, 8, 4> : k_brute<true, NYS_MAX_RHO, NYS_MAX_CHANNELS>;
    NYS_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, BF_TX * BF_TY, smem, s>>>(a);
  } else {
    auto k = small ? k_brute<false, 8, 4> : k_brute<false, NYS_MAX_RHO, NYS_MAX_CHANNELS>;
    k<<<grid, BF_TX * BF_TY, 0, s>>>(a);
  }
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}
