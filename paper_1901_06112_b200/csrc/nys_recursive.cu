// Recursive-Gaussian spatial kernel on the Nystrom filter path.
//
// Reference region replaced (reference = /root/reference/pkg/src/nysfilter):
//   spatial.py:114-146  _vyv_coeffs (host: nys_vyv_coeffs in nys_host.cpp)
//   spatial.py:149-176  _vyv_scan: fifth-order causal + anticausal recursion per
//                       row, forward state initialised with the edge sample,
//                       backward state with the forward output's edge sample
//   spatial.py:179-191  _recursive_planes: row scan, then column scan, then the
//                       squared truncated-FIR mass ((fir_mass(σ))^2)
//   filters.py:223-257  rank loop, accumulation, guard, division (y-form, as K2/K3)
//
// An IIR pass spans a whole row / column, so the tile-local FIR structure of
// K2/K3 does not apply.  The path is four kernels:
//   R1 k_rec_features  per pixel: b(x) and y = M b (+ the lead projection
//                      s0 = u0.b) -> Y [px][m0+1], Bf [px][m0]
//   R2 k_rec_rows      one thread per (row, plane): forward then backward
//                      recursion along the row, in place in Hb [px][Pb]
//   R3 k_rec_cols      one CTA per 1-4 columns, one thread per plane: forward
//                      recursion down the column in place, then the backward
//                      recursion up the column fused with the contraction
//                      Σ_i b_i(x) conv_i(x) (block reduction over landmarks)
//                      -> Z [(n+1)][px], lead terms -> Lz [(n+1)][px]
//   R4 k_rec_finish    mass^2 scale, guard, division, min|eta| / guarded count
// The planes are processed in landmark bands (Pb = (n+1) * groups per band)
// so the plane buffer fits the caller's scratch; Z accumulates across bands.
// The recursions run in FP64 (their poles sit close to 1: the direct form in
// FP32 would amplify rounding); planes are stored as FP32 between passes.
#include <string>

#include "nys_filter_common.cuh"

namespace nys {

struct RecCoeffs {
  double g, a1, a2, a3, a4, a5;
};

constexpr int REC_ROW_THREADS = 128;
constexpr int REC_RB = 16;    // rows per contraction batch in R3
constexpr int REC_COL_MAX_THREADS = 1024;  // R3 CTA: cpb * roundup32(Pb) threads (64 registers)
constexpr int REC_BATCH = 8;  // loads issued ahead of the recursion

struct RecScratch {
  size_t off_Y, off_B, off_Z, off_L, off_H, total;
};

inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

inline RecScratch rec_scratch(const nys_filter_desc* d, int groups_per_band) {
  const size_t px = (size_t)d->H * d->W;
  RecScratch s;
  s.off_Y = 0;
  s.off_B = s.off_Y + align256(px * (d->m0 + 1) * 4);
  s.off_Z = s.off_B + align256(px * d->m0 * 4);
  s.off_L = s.off_Z + align256(px * (d->n + 1) * 4);
  s.off_H = s.off_L + align256(px * (d->n + 1) * 4);
  s.total = s.off_H + align256(px * (size_t)(d->n + 1) * groups_per_band * 4);
  return s;
}

// one step of the reference recursion (spatial.py:161, 171):
//   cur = gain * x - (a1 w1 + a2 w2 + a3 w3 + a4 w4 + a5 w5)
struct RecState {
  double w1, w2, w3, w4, w5;
  __device__ __forceinline__ void init(double v) { w1 = w2 = w3 = w4 = w5 = v; }
  __device__ __forceinline__ double step(const RecCoeffs& c, double x) {
    const double t = fma(c.a5, w5, fma(c.a4, w4, fma(c.a3, w3, c.a2 * w2)));
    const double cur = fma(c.g, x, -fma(c.a1, w1, t));
    w5 = w4;
    w4 = w3;
    w3 = w2;
    w2 = w1;
    w1 = cur;
    return cur;
  }
};

// ---------------------------------------------------------------------------
// R1: features b(x) and y = M b at every pixel (nystrom.py:43-79, 112-114 in
// the y-form).  MT = [M | u0] transposed in the workspace (FilterLayout).
// ---------------------------------------------------------------------------
template <int BS, bool CSM, bool PLANAR>
__global__ void __launch_bounds__(BS) k_rec_features(
    const float* __restrict__ f, long long fps, const float* __restrict__ g, long long gps, int gkind, int rho,
    int H, int W, int m0, const float* __restrict__ consts, int rhop, int m0q, long long off_MT, float k2,
    float* __restrict__ Y, float* __restrict__ Bf, int phi) {
  // phi-form: the stored contraction weights are y (= phi) instead of b.
  // b and y are staged in shared memory ([value][pixel], pitch BS+1: the
  // transposed read-out below is bank-conflict free) so the block writes its
  // contiguous [px][m0] / [px][m0+1] output rows with coalesced stores.
  // CSM: centroids and [M | u0]^T also live in shared memory (broadcast LDS
  // instead of dependent L1 loads in the m0 x (m0+1) product).
  constexpr int PT = BS + 1;
  extern __shared__ float rsm[];
  float* sg = rsm;                                   // [rho][BS]
  float* sb = sg + (size_t)rho * BS;                 // [m0][PT]
  float* sy = sb + (size_t)m0 * PT;                  // [m0+1][PT]
  float* sc = rsm + ((((size_t)rho * BS + (size_t)(2 * m0 + 1) * PT) + 3) & ~(size_t)3);  // CSM, 16-byte aligned:
                                                     // [m0][rhop] centroids, then [m0][m0q] MT
  const int t = threadIdx.x;
  const long long npx = (long long)H * W;
  const long long px0 = (long long)blockIdx.x * BS;
  const long long px = px0 + t;
  const bool ok = px < npx;
  const int row = ok ? (int)(px / W) : 0, x = ok ? (int)(px - (long long)row * W) : 0;
  const float* C = consts;
  const float* MT = consts + off_MT;
  if (CSM) {
    for (int k = t; k < m0 * rhop; k += BS) sc[k] = __ldg(C + k);
    for (int k = t; k < m0 * m0q; k += BS) sc[m0 * rhop + k] = __ldg(MT + k);
    C = sc;
    MT = sc + m0 * rhop;
  }
  for (int k = 0; k < rho; ++k) sg[k * BS + t] = ok ? guide_at(g, gps, f, fps, gkind, k, row, x, H, W) : 0.f;
  if (CSM) __syncthreads();
  for (int j = 0; j < m0; ++j) {
    float d2 = 0.f;
    const float* cj = C + (size_t)j * rhop;
    for (int k = 0; k < rho; ++k) {
      const float dd = sg[k * BS + t] - cj[k];
      d2 = fmaf(dd, dd, d2);
    }
    sb[j * PT + t] = range_kernel(d2, k2);
  }
  for (int i0 = 0; i0 <= m0; i0 += 8) {
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
#pragma unroll 4
    for (int j = 0; j < m0; ++j) {
      const float bj = sb[j * PT + t];
      const float4 lo = *reinterpret_cast<const float4*>(MT + (size_t)j * m0q + i0);
      const float4 hi = *reinterpret_cast<const float4*>(MT + (size_t)j * m0q + i0 + 4);
      acc[0] = fmaf(bj, lo.x, acc[0]);
      acc[1] = fmaf(bj, lo.y, acc[1]);
      acc[2] = fmaf(bj, lo.z, acc[2]);
      acc[3] = fmaf(bj, lo.w, acc[3]);
      acc[4] = fmaf(bj, hi.x, acc[4]);
      acc[5] = fmaf(bj, hi.y, acc[5]);
      acc[6] = fmaf(bj, hi.z, acc[6]);
      acc[7] = fmaf(bj, hi.w, acc[7]);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (i0 + e <= m0) sy[(i0 + e) * PT + t] = acc[e];
  }
  if (PLANAR) {  // planar [value][px]: one coalesced store per value
    if (ok) {
      for (int j = 0; j < m0; ++j) Bf[(long long)j * npx + px] = phi ? sy[j * PT + t] : sb[j * PT + t];
      for (int i = 0; i <= m0; ++i) Y[(long long)i * npx + px] = sy[i * PT + t];
    }
    return;
  }
  __syncthreads();
  const int cnt = (int)min((long long)BS, npx - px0);
  for (int e = t; e < cnt * m0; e += BS) {
    const int i = e / m0, j = e - i * m0;
    Bf[px0 * m0 + e] = phi ? sy[j * PT + i] : sb[j * PT + i];
  }
  const int G = m0 + 1;
  for (int e = t; e < cnt * G; e += BS) {
    const int i = e / G, j = e - i * G;
    Y[px0 * G + e] = sy[j * PT + i];
  }
}

// ---------------------------------------------------------------------------
// R2: row recursion (spatial.py:184-185, _vyv_scan over rows) for the planes
// of landmark band [g0, g0+nb): plane q = c*nb + (g - g0), input y_g f_c
// (c < n) or y_g (c == n).  Forward pass writes Hb, backward pass rewrites it.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(REC_ROW_THREADS) k_rec_rows(
    const float* __restrict__ f, long long fps, const float* __restrict__ Y, int n, int H, int W, int m0, int g0,
    int nb, RecCoeffs cf, float* __restrict__ Hb) {
  const int Pb = (n + 1) * nb;
  const int q = blockIdx.x * REC_ROW_THREADS + threadIdx.x;
  const int row = blockIdx.y;
  if (q >= Pb) return;
  const int c = q / nb, g = g0 + (q - c * nb);
  const long long base = (long long)row * W;
  const float* __restrict__ yr = Y + base * (m0 + 1) + g;
  const float* __restrict__ fr = f + (long long)(c < n ? c : 0) * fps + base;
  float* __restrict__ hr = Hb + base * Pb + q;
  const bool mulf = c < n;
  RecState s;
  {
    const double v0 = mulf ? (double)__ldg(yr) * (double)__ldg(fr) : (double)__ldg(yr);
    s.init(v0);
  }
  double last = 0.0;
  for (int x0 = 0; x0 < W; x0 += REC_BATCH) {
    double v[REC_BATCH];
#pragma unroll
    for (int e = 0; e < REC_BATCH; ++e) {
      const int x = min(x0 + e, W - 1);
      const double yy = (double)__ldg(yr + (long long)x * (m0 + 1));
      v[e] = mulf ? yy * (double)__ldg(fr + x) : yy;
    }
#pragma unroll
    for (int e = 0; e < REC_BATCH; ++e) {
      if (x0 + e < W) {
        last = s.step(cf, v[e]);
        hr[(long long)(x0 + e) * Pb] = (float)last;
      }
    }
  }
  s.init((double)(float)last);  // backward state: the (stored) forward output's edge sample
  for (int x0 = W - 1; x0 >= 0; x0 -= REC_BATCH) {
    float v[REC_BATCH];
#pragma unroll
    for (int e = 0; e < REC_BATCH; ++e) v[e] = hr[(long long)max(x0 - e, 0) * Pb];
#pragma unroll
    for (int e = 0; e < REC_BATCH; ++e)
      if (x0 - e >= 0) hr[(long long)(x0 - e) * Pb] = (float)s.step(cf, (double)v[e]);
  }
}

// ---------------------------------------------------------------------------
// R3: column recursion (spatial.py:186-188) + contraction (filters.py:227-238
// in the y-form).  A CTA covers `cpb` adjacent columns (so each row step reads
// cpb*Pb contiguous floats); thread (column cb, plane q).  The forward pass
// rewrites Hb in place; the backward pass only feeds the contraction.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(REC_COL_MAX_THREADS, 1) k_rec_cols(const float* __restrict__ Y, const float* __restrict__ Bf,
                                                      int n, int H, int W, int m0, int g0, int nb, int cpb,
                                                      RecCoeffs cf, float inv_alpha0, int accumulate,
                                                      float* __restrict__ Hb, float* __restrict__ Z,
                                                      float* __restrict__ Lz) {
  extern __shared__ float csm[];  // [REC_RB][cpb][Pb] products b_g * conv
  const int Pb = (n + 1) * nb;
  const int Pbp = (Pb + 31) & ~31;
  const int cb = threadIdx.x / Pbp, q = threadIdx.x - cb * Pbp;
  const int x = blockIdx.x * cpb + cb;
  const bool active = q < Pb && cb < cpb && x < W;
  const int c = active ? q / nb : 0, g = g0 + (active ? q - c * nb : 0);
  const long long rs = (long long)W * Pb;  // row stride of Hb
  const long long npx = (long long)H * W;
  float* __restrict__ col = Hb + (long long)x * Pb + q;
  RecState s;
  double last = 0.0;
  if (active) {
    s.init((double)col[0]);
    for (int r0 = 0; r0 < H; r0 += REC_BATCH) {
      float v[REC_BATCH];
#pragma unroll
      for (int e = 0; e < REC_BATCH; ++e) v[e] = col[(long long)min(r0 + e, H - 1) * rs];
#pragma unroll
      for (int e = 0; e < REC_BATCH; ++e)
        if (r0 + e < H) {
          last = s.step(cf, (double)v[e]);
          col[(long long)(r0 + e) * rs] = (float)last;
        }
    }
    s.init((double)(float)last);
  }
  const bool has_lead = g0 <= m0 && m0 < g0 + nb;
  const int lead_l = m0 - g0;
  const int nl = min(nb, m0 - g0);  // landmark (non-lead) groups in the band
  const int ncols = min(cpb, W - (int)blockIdx.x * cpb);
  for (int rtop = H - 1; rtop >= 0; rtop -= REC_RB) {
    const int cnt = min(REC_RB, rtop + 1);
    if (active) {
#pragma unroll 1
     for (int h = 0; h < REC_RB; h += REC_BATCH) {
      float v[REC_BATCH];
#pragma unroll
      for (int e2 = 0; e2 < REC_BATCH; ++e2) v[e2] = h + e2 < cnt ? col[(long long)(rtop - h - e2) * rs] : 0.f;
#pragma unroll
      for (int e2 = 0; e2 < REC_BATCH; ++e2) {
        const int e = h + e2;
        if (e < cnt) {
          const int row = rtop - e;
          const float val = (float)s.step(cf, (double)v[e2]);
          const long long p = (long long)row * W + x;
          float prod;
          if (g < m0)
            prod = __ldg(Bf + p * m0 + g) * val;
          else
            prod = __ldg(Y + p * (m0 + 1) + m0) * val * inv_alpha0;  // s0 conv(s0 f)/α0
          csm[(e * cpb + cb) * Pb + q] = prod;
        }
      }
     }
    }
    __syncthreads();
    for (int o = threadIdx.x; o < ncols * (n + 1) * cnt; o += blockDim.x) {
      const int e = o % cnt, rest = o / cnt, cc = rest % (n + 1), cbo = rest / (n + 1);
      const float* sp = csm + (e * cpb + cbo) * Pb + cc * nb;
      float acc = 0.f;
      for (int l = 0; l < nl; ++l) acc += sp[l];
      const long long p = (long long)(rtop - e) * W + blockIdx.x * cpb + cbo;
      float* zp = Z + cc * npx + p;
      *zp = accumulate ? *zp + acc : acc;
      if (has_lead) Lz[cc * npx + p] = sp[lead_l];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// R4: (fir_mass)^2 scale (spatial.py:189-191), guard and division
// (filters.py:241-257), min|eta| and the guarded-pixel count.
// ---------------------------------------------------------------------------
__global__ void k_rec_finish(const float* __restrict__ f, long long fps, const float* __restrict__ Z,
                             const float* __restrict__ Lz, int n, int H, int W, float mass2, float eps,
                             float* __restrict__ out, long long ops, FilterStats* __restrict__ stats) {
  const long long npx = (long long)H * W;
  float my_min = INFINITY;
  unsigned long long my_cnt = 0;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < npx; p += (long long)gridDim.x * blockDim.x) {
    const float eta = Z[(long long)n * npx + p] * mass2;
    const float eta_l = Lz[(long long)n * npx + p] * mass2;
    const float ae = fabsf(eta);
    my_min = fminf(my_min, ae);
    const bool guarded = ae < eps;
    my_cnt += guarded ? 1ull : 0ull;
    const int row = (int)(p / W), x = (int)(p - (long long)row * W);
    for (int c = 0; c < n; ++c) {
      float r;
      if (!guarded)
        r = (Z[(long long)c * npx + p] * mass2) / eta;
      else if (fabsf(eta_l) >= eps)
        r = (Lz[(long long)c * npx + p] * mass2) / eta_l;
      else
        r = __ldg(f + (long long)c * fps + p);
      out[(long long)c * ops + (long long)row * W + x] = r;
    }
  }
  // block reduction, then one atomic per block
  __shared__ float smin[32];
  __shared__ unsigned long long scnt[32];
  my_min = warp_min(my_min);
  my_cnt = warp_sum_u64(my_cnt);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    smin[wid] = my_min;
    scnt[wid] = my_cnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float mn = INFINITY;
    unsigned long long cn = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      mn = fminf(mn, smin[w]);
      cn += scnt[w];
    }
    atomicMin(&stats->min_abs_eta_bits, __float_as_uint(mn));
    if (cn) atomicAdd(&stats->guarded, cn);
  }
}

}  // namespace nys

using namespace nys;

namespace {

int rec_groups_fit(const nys_filter_desc* d, size_t scratch_bytes) {
  // largest landmark band (groups of n+1 planes incl. the lead group) with
  // Pb <= 1024 threads per CTA whose plane buffer fits the scratch
  const int G = d->m0 + 1;
  int nb = std::min(G, REC_COL_MAX_THREADS / (d->n + 1));
  while (nb >= 1 && rec_scratch(d, nb).total > scratch_bytes) --nb;
  return nb;
}

int rec_validate(const nys_filter_desc* d) {
  const int st = validate(d);
  if (!st && (d->rho > NYS_MAX_RHO || d->n > NYS_MAX_CHANNELS)) return NYS_EUNSUPPORTED;  // register-resident R1
  if (st) return st;
  if (d->spatial_kind != NYS_SPATIAL_GAUSSIAN_RECURSIVE) return NYS_EINVAL;
  if (d->n + 1 > REC_COL_MAX_THREADS) return NYS_EUNSUPPORTED;
  return NYS_OK;
}

}  // namespace

extern "C" {

size_t nys_filter_recursive_scratch_bytes(const nys_filter_desc* d, int groups_per_band) {
  if (rec_validate(d) != NYS_OK) return 0;
  const int G = d->m0 + 1;
  int nb = groups_per_band <= 0 ? G : std::min(groups_per_band, G);
  nb = std::min(nb, REC_COL_MAX_THREADS / (d->n + 1));
  return rec_scratch(d, nb).total;
}

int nys_filter_recursive(const nys_filter_desc* d, const float* f, int64_t f_plane_stride, const float* guide,
                         int64_t guide_plane_stride, float* out, int64_t out_plane_stride, void* scratch,
                         size_t scratch_bytes, const void* workspace, void* stream) {
  int st = rec_validate(d);
  if (st) return st;
  if (!f || !out || !scratch || !workspace || (d->guide_kind == 0 && !guide)) return NYS_EINVAL;
  if (d->row_lo != 0 || (d->row_hi != 0 && d->row_hi != d->H)) return NYS_EUNSUPPORTED;  // whole columns only
  double cfv[6];
  st = nys_vyv_coeffs(d->sigma, cfv);
  if (st) return st;
  const RecCoeffs cf{cfv[0], cfv[1], cfv[2], cfv[3], cfv[4], cfv[5]};
  // squared truncated-FIR mass at radius ceil(3 sigma) (spatial.py:78-82, 189-191)
  const int Rm = (int)std::ceil(3.0 * d->sigma);
  double mass = 0.0;
  for (int t = -Rm; t <= Rm; ++t) mass += std::exp(-((double)t * t) / (2.0 * d->sigma * d->sigma));
  const FilterLayout L = filter_layout(d);
  const int nb_max = rec_groups_fit(d, scratch_bytes);
  if (nb_max < 1) return NYS_EINVAL;
  const RecScratch S = rec_scratch(d, nb_max);
  char* sc = static_cast<char*>(scratch);
  float* Y = reinterpret_cast<float*>(sc + S.off_Y);
  float* Bf = reinterpret_cast<float*>(sc + S.off_B);
  float* Z = reinterpret_cast<float*>(sc + S.off_Z);
  float* Lz = reinterpret_cast<float*>(sc + S.off_L);
  float* Hb = reinterpret_cast<float*>(sc + S.off_H);
  const float* consts = static_cast<const float*>(workspace);
  cudaStream_t s = (cudaStream_t)stream;
  const long long npx = (long long)d->H * d->W;
  const float* g = d->guide_kind == 0 ? guide : f;

  {
    // (2 m0 + 1 + rho) x (BS + 1) floats of SMEM (+ centroids and MT when m0 <= 96):
    // 128-pixel blocks up to m0 = 96, 64 beyond
    const int BS = d->m0 <= 96 ? 128 : 64;
    const bool csm = d->m0 <= 96;
    const size_t smem = ((size_t)d->rho * BS + (size_t)(2 * d->m0 + 1) * (BS + 1) +
                         (csm ? (size_t)d->m0 * (L.rhop + L.m0q) + 4 : 0)) * sizeof(float);
    auto k = csm ? k_rec_features<128, true, false> : k_rec_features<64, false, false>;
    NYS_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    count_launch();
    k<<<(unsigned)ceil_div(npx, BS), BS, smem, s>>>(f, f_plane_stride, g, guide_plane_stride, d->guide_kind, d->rho,
                                                    d->H, d->W, d->m0, consts + L.off_C, L.rhop, L.m0q,
                                                    (long long)(L.off_MT - L.off_C), k2_of(d), Y, Bf, d->phi_form);
    NYS_LAUNCH_CHECK();
  }
  const int G = d->m0 + 1;
  const int nbands = (int)ceil_div(G, nb_max);
  const int nb_even = (int)ceil_div(G, nbands);  // balanced bands
  for (int b = 0, g0 = 0; b < nbands; ++b, g0 += nb_even) {
    const int nb = std::min(nb_even, G - g0);
    const int Pb = (d->n + 1) * nb;
    count_launch();
    k_rec_rows<<<dim3((unsigned)ceil_div(Pb, REC_ROW_THREADS), (unsigned)d->H), REC_ROW_THREADS, 0, s>>>(
        f, f_plane_stride, Y, d->n, d->H, d->W, d->m0, g0, nb, cf, Hb);
    NYS_LAUNCH_CHECK();
    const int Pbp = (int)ceil_div(Pb, 32) * 32;
    const int cpb = 1;  // measured: more columns per CTA lowers occupancy (latency-bound walk)
    const size_t smem = (size_t)REC_RB * cpb * Pb * sizeof(float);
    NYS_CUDA_TRY(cudaFuncSetAttribute(k_rec_cols, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    count_launch();
    k_rec_cols<<<(unsigned)ceil_div(d->W, cpb), cpb * Pbp, smem, s>>>(Y, Bf, d->n, d->H, d->W, d->m0, g0, nb, cpb, cf,
                                                      (float)(1.0 / d->alpha0), b > 0 ? 1 : 0, Hb, Z, Lz);
    NYS_LAUNCH_CHECK();
  }
  count_launch();
  const int grid = (int)std::min<long long>(ceil_div(npx, 256), (long long)num_sms() * 8);
  k_rec_finish<<<grid, 256, 0, s>>>(f, f_plane_stride, Z, Lz, d->n, d->H, d->W, (float)(mass * mass),
                                    (float)d->eps_den, out, out_plane_stride,
                                    reinterpret_cast<FilterStats*>((char*)workspace + L.stats_off_bytes));
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

}  // extern "C"
