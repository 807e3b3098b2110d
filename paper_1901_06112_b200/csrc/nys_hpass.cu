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
// spatial.py:85-88).  K2's output tile is one contiguous block (streaming HBM
// writes); K3 reads 4 planes x 32 columns = 512 B per row with one TMA box.
#include <cstdlib>

#include "nys_hpass.cuh"

namespace nys {

constexpr double NYS_TC_MAX_NORM = 1.0e3;  // tensor-core y = M b up to this ||M||_inf (nys_filter_hpass)

template <int RT, int GR>
__global__ void __launch_bounds__(K2_THREADS, 2) k_feat_hpass(const HArgs a) {
  extern __shared__ __align__(128) float sm[];
  const int R = RT > 0 ? RT : a.R;
  const int m0 = a.m0, m0q = a.m0q, n = a.n, rho = a.rho, rhop = a.rhop, W = a.W, H = a.H;
  const int NC = n + 1, L = m0 + 1, pitch = a.pitch, TW = a.TW;
  const int RPT = a.rpt;
  float* Cs = sm;                                  // m0 x rhop
  float* MT = Cs + (size_t)m0 * rhop;              // m0 x m0q   MT[j][i] = M[i][j], MT[j][m0] = u0[j]
  float* Fs = MT + (size_t)m0 * m0q;               // RPT x n x pitch
  float* Bs = Fs + (size_t)RPT * n * pitch;        // RPT x m0 x pitch
  float* Ys = Bs + (size_t)RPT * m0 * pitch;       // RPT x m0q x pitch

  const size_t ncst = (size_t)m0 * rhop + (size_t)m0 * m0q;
  for (size_t k = threadIdx.x; k < ncst; k += blockDim.x) sm[k] = a.cst[k];

  const int ncols = TW + 2 * R;
  const int nq = (ncols + 3) / 4;          // pixel quads with features
  const int ncol4 = nq * 4;
  const int nchunks = (NC + K2_CC - 1) / K2_CC;
  const int XG = TW / K2_XR;
  const int fir_items = RPT * L * nchunks * XG;
  const int nic = m0q / 8;
  const int gemm_items = RPT * nq * nic;
  const int row_tiles = (a.vrows + RPT - 1) / RPT;
  const int ntiles = a.tiles_x * row_tiles;

  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int vb = a.v0 + (tile / a.tiles_x) * RPT;  // first virtual row of the tile
    const int x0 = (tile % a.tiles_x) * TW;
    __syncthreads();  // previous tile's readers are done (and constants staged)
    for (int k = threadIdx.x; k < RPT * n * ncol4; k += blockDim.x) {
      const int r = k / (n * ncol4), rem = k - r * (n * ncol4);
      const int c = rem / ncol4, s = rem - c * ncol4;
      const int row = clampi(clampi(vb + r, 0, H - 1), a.rlo, a.rhi - 1);
      const int x = clampi(x0 - R + s, 0, W - 1);
      Fs[((size_t)r * n + c) * pitch + s] = __ldg(a.f + (long long)c * a.fps + (long long)row * W + x);
    }
    // b_j(x) for every column of the tile incl. the 2R halo (difference-form distances)
    for (int k = threadIdx.x; k < ((a.dbg & 1) ? 0 : RPT * ncol4); k += blockDim.x) {
      const int r = k / ncol4, s = k - r * ncol4;
      const int row = clampi(clampi(vb + r, 0, H - 1), a.rlo, a.rhi - 1);
      const int x = clampi(x0 - R + s, 0, W - 1);
      float gv[GR];
#pragma unroll
      for (int d = 0; d < GR; ++d) gv[d] = d < rho ? guide_at(a.g, a.gps, a.f, a.fps, a.gkind, d, row, x, H, W) : 0.f;
      float* brow = Bs + (size_t)r * m0 * pitch + s;
      for (int j = 0; j < m0; ++j) {
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
        brow[(size_t)j * pitch] = range_kernel(d2, a.k2);
      }
    }
    __syncthreads();
    // [px x m0] x [m0 x m0q]: 4 pixels x 8 outputs per item, FP32 FMA
    for (int it = threadIdx.x; it < ((a.dbg & 2) ? 0 : gemm_items); it += blockDim.x) {
      const int q = it % nq, rem = it / nq;
      const int ic = rem % nic, r = rem / nic;
      float acc[4][8];
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int ii = 0; ii < 8; ++ii) acc[p][ii] = 0.f;
      const float* bcol = Bs + (size_t)r * m0 * pitch + 4 * q;
      const float* mcol = MT + 8 * ic;
#pragma unroll 4
      for (int j = 0; j < m0; ++j) {
        const float4 b4 = *reinterpret_cast<const float4*>(bcol + (size_t)j * pitch);
        const float4 ma = *reinterpret_cast<const float4*>(mcol + (size_t)j * m0q);
        const float4 mb = *reinterpret_cast<const float4*>(mcol + (size_t)j * m0q + 4);
        const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
        const float mm[8] = {ma.x, ma.y, ma.z, ma.w, mb.x, mb.y, mb.z, mb.w};
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int ii = 0; ii < 8; ++ii) acc[p][ii] = fmaf(mm[ii], bb[p], acc[p][ii]);
      }
      float* yout = Ys + (size_t)r * m0q * pitch + 4 * q;
#pragma unroll
      for (int ii = 0; ii < 8; ++ii)
        *reinterpret_cast<float4*>(yout + (size_t)(8 * ic + ii) * pitch) =
            make_float4(acc[0][ii], acc[1][ii], acc[2][ii], acc[3][ii]);
    }
    __syncthreads();
    for (int it = threadIdx.x; it < fir_items; it += blockDim.x) {
      const int i = it % L;
      int rest = it / L;
      const int ch = rest % nchunks;
      rest /= nchunks;
      const int xg = rest % XG;
      const int r = rest / XG;
      const int xo = x0 + xg * K2_XR;
      if (xo >= W || vb + r >= a.v0 + a.vrows) continue;
      float acc[K2_CC][K2_XR];
      if (a.dbg & 4) {
#pragma unroll
        for (int cc = 0; cc < K2_CC; ++cc)
#pragma unroll
          for (int o = 0; o < K2_XR; ++o) acc[cc][o] = Ys[((size_t)r * m0q + i) * pitch + o + cc];
      } else {
        hfir<RT>(a, Ys + ((size_t)r * m0q + i) * pitch + xg * K2_XR, Fs + (size_t)r * n * pitch, pitch, xg * K2_XR,
                 ch * K2_CC, acc);
      }
      if (a.dbg & 8) {
        if (acc[0][0] == 1234.5f) a.hp[0] = acc[1][1];
        continue;
      }
      float* dst0 = a.hp + (long long)(vb + r - a.v0) * a.rs + (long long)(xo >> 5) * (a.npl * 32) + (xo & 31);
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
    if (a.bplanes) {
      // raw b_i of the tile's output columns (K3 reads them at the centre pixel)
      for (int it = threadIdx.x; it < RPT * m0 * XG; it += blockDim.x) {
        const int i = it % m0, rest = it / m0, xg = rest % XG, r = rest / XG;
        const int xo = x0 + xg * K2_XR;
        if (xo >= W || vb + r >= a.v0 + a.vrows) continue;
        const float* src = (a.phi ? Ys + ((size_t)r * m0q + i) * pitch : Bs + ((size_t)r * m0 + i) * pitch) + R +
                           xg * K2_XR;  // phi-form: the contraction weights are phi = y
        float* dst = a.hp + (long long)(vb + r - a.v0) * a.rs + (long long)(xo >> 5) * (a.npl * 32) +
                     (long long)(L * NC + i) * 32 + (xo & 31);
#pragma unroll
        for (int q4 = 0; q4 < K2_XR / 4; ++q4)
          reinterpret_cast<float4*>(dst)[q4] = make_float4(src[4 * q4], src[4 * q4 + 1], src[4 * q4 + 2], src[4 * q4 + 3]);
      }
    }
  }
}

}  // namespace nys

using namespace nys;

extern "C" {

int nys_filter_hpass(const nys_filter_desc* d, const float* f, int64_t f_plane_stride, const float* guide,
                     int64_t guide_plane_stride, int out0, int out_rows, float* planes, int64_t planes_stride,
                     const void* workspace, void* stream) {
  int st = validate_tiled(d);
  if (st) return st;
  if (!f || !planes || !workspace || (d->guide_kind == 0 && !guide)) return NYS_EINVAL;
  if (out0 < 0 || out_rows < 1 || out0 + out_rows > d->H) return NYS_EINVAL;
  if (planes_stride < plane_row_stride(d->W, buffer_planes(d)) || (planes_stride & 3)) return NYS_EINVAL;
  if (reinterpret_cast<uintptr_t>(planes) & 15) return NYS_EINVAL;
  const FilterLayout L = filter_layout(d);
  HArgs a;
  memset(&a, 0, sizeof(a));
  a.f = f;
  a.g = d->guide_kind == 0 ? guide : f;
  a.hp = planes;
  a.cst = reinterpret_cast<const float*>(workspace);
  a.fps = f_plane_stride;
  a.gps = d->guide_kind == 0 ? guide_plane_stride : f_plane_stride;
  a.rs = planes_stride;
  a.n = d->n;
  a.rho = d->rho;
  a.rhop = L.rhop;
  a.H = d->H;
  a.W = d->W;
  a.m0 = d->m0;
  a.m0q = L.m0q;
  a.R = d->radius;
  a.box = d->spatial_kind == NYS_SPATIAL_BOX;
  a.gkind = d->guide_kind;
  a.v0 = out0 - d->radius;
  a.vrows = out_rows + 2 * d->radius;
  a.rlo = std::max(0, d->row_lo);
  a.npl = buffer_planes(d);
  a.bplanes = use_bplanes(d);
  a.phi = d->phi_form;
  a.rhi = d->row_hi > 0 ? std::min(d->H, d->row_hi) : d->H;
  a.k2 = k2_of(d);
  fill_taps(d, a.taps);
  fill_tap_pairs(a.taps, 2 * d->radius + 1, a.wpair);
  if (const char* e = getenv("NYS_DBG_K2")) a.dbg = atoi(e);
  cudaStream_t s = (cudaStream_t)stream;
  {
    // The tensor-core product (3xTF32: ~3x the rounding error of FP32 FMA, from
    // the split representation and the accumulator) is used while the mixing
    // matrix is well conditioned.  ||M||_inf >= ||M||_2 = 1/alpha_min bounds the
    // cancellation in y = M b; beyond NYS_TC_MAX_NORM the CUDA-core FP32 FMA
    // GEMM keeps ill-conditioned landmark sets inside the parity budget.
    double normM = 0.0;
    for (int i = 0; i < d->m0; ++i) {
      double rs = 0.0;
      for (int j = 0; j < d->m0; ++j) rs += std::fabs(d->M[(size_t)i * d->m0 + j]);
      normM = std::max(normM, rs);
    }
    const char* e = getenv("NYS_K2_SIMT");  // debug: force the CUDA-core GEMM kernel
    if (!(e && atoi(e)) && normM <= NYS_TC_MAX_NORM) {
      const int rc = launch_hpass_tc(a, d, s);
      if (rc != NYS_EUNSUPPORTED) return rc;
    }
  }
  // tile shape (TW columns x RPT rows): minimise a per-output-pixel cost model
  // of the three barrier-separated phases (features, y GEMM, FIR), each of
  // which runs ceil(items / 512) rounds, under the shared-memory budget
  const size_t cst_floats = (size_t)d->m0 * L.rhop + (size_t)d->m0 * L.m0q;
  const size_t per_col = (size_t)(d->n + d->m0 + L.m0q);
  auto pitch_for = [&](int tw) {
    int p = (int)ceil_div(tw + 2 * d->radius + 4, 4) * 4;
    p += ((4 - p % 32) + 32) % 32;  // pitch = 4 (mod 32): LDS.128 across rows is conflict-free
    return p;
  };
  auto smem_for = [&](int tw, int rpt) { return (cst_floats + (size_t)rpt * per_col * pitch_for(tw)) * 4; };
  const int R = d->radius, T = 2 * R + 1, NC = d->n + 1, Lm = d->m0 + 1;
  const int nchunks = (int)ceil_div(NC, K2_CC);
  const double fir_item = d->spatial_kind == NYS_SPATIAL_BOX ? 4.0 * (16 + 2 * R) * 3 : 64.0 * T + 4.0 * (16 + 2 * R);
  const double gemm_item = 36.0 * d->m0;
  const double feat_px = d->m0 * (2.0 * d->rho + 6.0);
  const int wcap = (int)std::min<int64_t>(256, ceil_div(d->W, K2_XR) * K2_XR);
  int TW = K2_XR, RPT = 1;
  double best = 1e300;
  for (int rpt = 1; rpt <= 4; rpt *= 2) {
    if (rpt > out_rows + 2 * R) break;
    for (int tw = K2_XR; tw <= wcap; tw += K2_XR) {
      if (smem_for(tw, rpt) > 110 * 1024) break;
      const int nq = (int)ceil_div(tw + 2 * R, 4);
      const double fr = (double)ceil_div((int64_t)rpt * Lm * nchunks * (tw / K2_XR), K2_THREADS) * fir_item;
      const double gr = (double)ceil_div((int64_t)rpt * nq * (L.m0q / 8), K2_THREADS) * gemm_item;
      const double er = (double)ceil_div((int64_t)rpt * nq * 4, K2_THREADS) * feat_px;
      const double cost = (fr + gr + er + 2000.0) / ((double)rpt * std::min(tw, d->W));
      if (cost < best) {
        best = cost;
        TW = tw;
        RPT = rpt;
      }
    }
  }
  const size_t smem = smem_for(TW, RPT);
  if (smem > 220 * 1024) return NYS_EUNSUPPORTED;
  a.TW = TW;
  a.rpt = RPT;
  a.pitch = pitch_for(TW);
  a.tiles_x = (int)ceil_div(d->W, TW);
  const long long ntiles = (long long)a.tiles_x * ceil_div(a.vrows, RPT);
  const int grid = (int)std::min<long long>(ntiles, (long long)num_sms() * 2);
  const int GR = d->rho <= 4 ? 4 : (d->rho <= 16 ? 16 : (d->rho <= 32 ? 32 : 64));
  auto go = [&](auto kern) -> int {
    NYS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    NYS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    count_launch();
    kern<<<grid, K2_THREADS, smem, s>>>(a);
    NYS_LAUNCH_CHECK();
    return NYS_OK;
  };
#define NYS_H_GR(RV)                                       \
  switch (GR) {                                            \
    case 4: return go(k_feat_hpass<RV, 4>);                \
    case 16: return go(k_feat_hpass<RV, 16>);              \
    case 32: return go(k_feat_hpass<RV, 32>);              \
    default: return go(k_feat_hpass<RV, 64>);              \
  }
  const int rsel = a.box ? 0 : d->radius;
  switch (rsel) {
    case 9: NYS_H_GR(9)
    case 12: NYS_H_GR(12)
    case 15: NYS_H_GR(15)
    case 18: NYS_H_GR(18)
    default: NYS_H_GR(0)
  }
#undef NYS_H_GR
}

}  // extern "C"
