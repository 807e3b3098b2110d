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
// pixel.  K2 evaluates b and y per source pixel and runs the horizontal pass
// of the (m0+1)(n+1) planes y_i f_c, y_i (plus the rank-1 lead planes
// s0 f_c, s0 with s0 = w_0.b, needed by the guard).  K3 runs the vertical pass
// and contracts with b_i(x) recomputed at the centre pixel, then applies the
// guard and division.  Only the horizontally filtered planes touch HBM.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "nys_common.cuh"

namespace nys {

// ---------------------------------------------------------------------------
// constants block in the workspace (float offsets)
// ---------------------------------------------------------------------------
struct FilterLayout {
  int m0, rho, m0p;  // m0p: m0 rounded up to 16 (zero-padded rows of M^T)
  size_t off_C, off_MT, off_U0, n_floats;
  size_t stats_off_bytes, total_bytes;
};

static FilterLayout filter_layout(const nys_filter_desc* d) {
  FilterLayout L;
  L.m0 = d->m0;
  L.rho = d->rho;
  L.m0p = (int)ceil_div(d->m0, 16) * 16;
  L.off_C = 0;
  L.off_MT = L.off_C + (size_t)d->m0 * d->rho;
  L.off_U0 = L.off_MT + (size_t)d->m0 * L.m0p;
  L.n_floats = L.off_U0 + (size_t)L.m0p;
  L.stats_off_bytes = ((L.n_floats * 4 + 255) / 256) * 256;
  L.total_bytes = L.stats_off_bytes + 256;
  return L;
}

struct FilterStats {
  unsigned int min_abs_eta_bits;  // float bits, non-negative => integer order
  unsigned int pad;
  unsigned long long guarded;
};

// ---------------------------------------------------------------------------
// kernel arguments (passed by value; taps land in the constant bank, so the
// unrolled FIR issues FFMA with a c[0x0][...] operand)
// ---------------------------------------------------------------------------
struct HArgs {
  const float* f;
  const float* g;
  float* hp;
  const float* cst;
  long long fps, gps, hps;
  int n, rho, H, W, m0, m0p, R, box, gkind;
  int row0, rows, TW, pitch, tiles_x;
  float k2;
  float taps[NYS_MAX_TAPS];
};

struct VArgs {
  const float* f;
  const float* g;
  const float* hp;
  float* out;
  const float* cst;
  FilterStats* stats;
  long long fps, gps, hps, ops;
  int n, rho, H, W, m0, R, box, gkind;
  int hp_row0, out0, out_rows, nchunks, runs, tiles_x, tiles_y;
  long long u0_off;  // float offset of u0 in the constants block
  float k2, inv_alpha0, eps_den;
  float taps[NYS_MAX_TAPS];
};

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

// ---------------------------------------------------------------------------
// K2: features + y = M b + horizontal pass
// ---------------------------------------------------------------------------
constexpr int H_THREADS = 256;
constexpr int H_XR = 8;   // output columns per thread item (one 32 B sector)
constexpr int H_CC = 4;   // planes per thread item

template <int RT>
__device__ __forceinline__ void hfir_item(const HArgs& a, const float* __restrict__ yrow,
                                          const float* __restrict__ Fs, int pitch, int xoff,
                                          int c0, float (&acc)[H_CC][H_XR]) {
  const int n = a.n;
  const float* fr[H_CC];
  float mode[H_CC];  // 0: y*f, 1: y, 2: unused plane
#pragma unroll
  for (int cc = 0; cc < H_CC; ++cc) {
    const int c = c0 + cc;
    fr[cc] = Fs + (size_t)min(c, n - 1) * pitch + xoff;
    mode[cc] = c < n ? 0.f : (c == n ? 1.f : 2.f);
  }
#pragma unroll
  for (int cc = 0; cc < H_CC; ++cc)
#pragma unroll
    for (int o = 0; o < H_XR; ++o) acc[cc][o] = 0.f;

  if (a.box) {
    // sliding (2R+1)-sum, re-anchored per item (spatial.py:91-99)
    const int R = a.R;
    float s[H_CC];
#pragma unroll
    for (int cc = 0; cc < H_CC; ++cc) s[cc] = 0.f;
    for (int t = 0; t <= 2 * R; ++t) {
      const float yv = yrow[t];
#pragma unroll
      for (int cc = 0; cc < H_CC; ++cc) s[cc] += mode[cc] == 0.f ? yv * fr[cc][t] : (mode[cc] == 1.f ? yv : 0.f);
    }
#pragma unroll
    for (int o = 0; o < H_XR; ++o) {
      if (o > 0) {
        const float yin = yrow[o + 2 * R], yout = yrow[o - 1];
#pragma unroll
        for (int cc = 0; cc < H_CC; ++cc) {
          const float vin = mode[cc] == 0.f ? yin * fr[cc][o + 2 * R] : (mode[cc] == 1.f ? yin : 0.f);
          const float vout = mode[cc] == 0.f ? yout * fr[cc][o - 1] : (mode[cc] == 1.f ? yout : 0.f);
          s[cc] += vin - vout;
        }
      }
#pragma unroll
      for (int cc = 0; cc < H_CC; ++cc) acc[cc][o] = s[cc];
    }
    return;
  }
  if constexpr (RT > 0) {
    constexpr int T = 2 * RT + 1;
#pragma unroll
    for (int s = 0; s < H_XR + 2 * RT; ++s) {
      const float yv = yrow[s];
#pragma unroll
      for (int cc = 0; cc < H_CC; ++cc) {
        const float v = mode[cc] == 0.f ? yv * fr[cc][s] : (mode[cc] == 1.f ? yv : 0.f);
#pragma unroll
        for (int o = 0; o < H_XR; ++o) {
          const int t = s - o;
          if (t >= 0 && t < T) acc[cc][o] = fmaf(a.taps[t], v, acc[cc][o]);
        }
      }
    }
  } else {
    const int T = 2 * a.R + 1;
    for (int t = 0; t < T; ++t) {
      const float w = a.taps[t];
#pragma unroll
      for (int o = 0; o < H_XR; ++o) {
        const float yv = yrow[o + t];
#pragma unroll
        for (int cc = 0; cc < H_CC; ++cc) {
          const float v = mode[cc] == 0.f ? yv * fr[cc][o + t] : (mode[cc] == 1.f ? yv : 0.f);
          acc[cc][o] = fmaf(w, v, acc[cc][o]);
        }
      }
    }
  }
}

template <int RT>
__global__ void __launch_bounds__(H_THREADS) k_feat_hpass(const HArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int R = RT > 0 ? RT : a.R;
  const int m0 = a.m0, m0p = a.m0p, n = a.n, rho = a.rho, W = a.W, H = a.H;
  const int NC = n + 1, L = m0 + 1, pitch = a.pitch, TW = a.TW;
  const int ncols = TW + 2 * R;
  float* Cs = sm;                                  // m0*rho
  float* MT = Cs + (size_t)m0 * rho;               // m0 x m0p   (MT[j*m0p+i] = M[i][j])
  float* U0 = MT + (size_t)m0 * m0p;               // m0p
  float* Fs = U0 + m0p;                            // n x pitch
  float* Ys = Fs + (size_t)n * pitch;              // L x pitch
  float* Bs = Ys + (size_t)L * pitch;              // m0 x pitch

  const size_t ncst = (size_t)m0 * rho + (size_t)m0 * m0p + m0p;
  for (size_t k = threadIdx.x; k < ncst; k += blockDim.x) sm[k] = a.cst[k];

  const int nchunks = (NC + H_CC - 1) / H_CC;
  const int nxr = TW / H_XR;
  const int items = L * nchunks * nxr;
  const int ntiles = a.tiles_x * a.rows;

  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int row = a.row0 + tile / a.tiles_x;
    const int x0 = (tile % a.tiles_x) * TW;
    __syncthreads();  // previous tile's readers done (and constants staged)
    for (int k = threadIdx.x; k < n * ncols; k += blockDim.x) {
      const int c = k / ncols, s = k - c * ncols;
      const int x = clampi(x0 - R + s, 0, W - 1);
      Fs[(size_t)c * pitch + s] = __ldg(a.f + (long long)c * a.fps + (long long)row * W + x);
    }
    // features b_j(x) for every column of the tile incl. the 2R halo
    for (int s = threadIdx.x; s < ncols; s += blockDim.x) {
      const int x = clampi(x0 - R + s, 0, W - 1);
      float gv[NYS_MAX_RHO];
      const bool small = rho <= 32;
      if (small) {
#pragma unroll
        for (int d = 0; d < 32; ++d)
          if (d < rho) gv[d] = guide_at(a.g, a.gps, a.f, a.fps, a.gkind, d, row, x, H, W);
      }
      for (int j = 0; j < m0; ++j) {
        float d2 = 0.f;
        if (small) {
#pragma unroll
          for (int d = 0; d < 32; ++d)
            if (d < rho) {
              const float t = gv[d] - Cs[j * rho + d];
              d2 = fmaf(t, t, d2);
            }
        } else {
          for (int d = 0; d < rho; ++d) {
            const float t = guide_at(a.g, a.gps, a.f, a.fps, a.gkind, d, row, x, H, W) - Cs[j * rho + d];
            d2 = fmaf(t, t, d2);
          }
        }
        Bs[(size_t)j * pitch + s] = range_kernel(d2, a.k2);
      }
      // y = M b (16 rows at a time) and the lead projection s0 = u0 . b
      for (int i0 = 0; i0 < m0; i0 += 16) {
        float y[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) y[q] = 0.f;
        for (int j = 0; j < m0; ++j) {
          const float bj = Bs[(size_t)j * pitch + s];
          const float4* mr = reinterpret_cast<const float4*>(MT + (size_t)j * m0p + i0);
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const float4 mm = mr[q4];
            y[4 * q4 + 0] = fmaf(mm.x, bj, y[4 * q4 + 0]);
            y[4 * q4 + 1] = fmaf(mm.y, bj, y[4 * q4 + 1]);
            y[4 * q4 + 2] = fmaf(mm.z, bj, y[4 * q4 + 2]);
            y[4 * q4 + 3] = fmaf(mm.w, bj, y[4 * q4 + 3]);
          }
        }
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (i0 + q < m0) Ys[(size_t)(i0 + q) * pitch + s] = y[q];
      }
      float s0 = 0.f;
      for (int j = 0; j < m0; ++j) s0 = fmaf(U0[j], Bs[(size_t)j * pitch + s], s0);
      Ys[(size_t)m0 * pitch + s] = s0;
    }
    __syncthreads();

    const bool vec = ((W & 3) == 0) && ((a.hps & 3) == 0);
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
      const int i = it % L;
      const int rest = it / L;
      const int ch = rest % nchunks;
      const int xr = rest / nchunks;
      const int xo = x0 + xr * H_XR;
      if (xo >= W) continue;
      float acc[H_CC][H_XR];
      hfir_item<RT>(a, Ys + (size_t)i * pitch + xr * H_XR, Fs, pitch, xr * H_XR, ch * H_CC, acc);
#pragma unroll
      for (int cc = 0; cc < H_CC; ++cc) {
        const int c = ch * H_CC + cc;
        if (c >= NC) break;
        float* dst = a.hp + (long long)(i * NC + c) * a.hps + (long long)(row - a.row0) * W + xo;
        if (vec && xo + H_XR <= W) {
          reinterpret_cast<float4*>(dst)[0] = make_float4(acc[cc][0], acc[cc][1], acc[cc][2], acc[cc][3]);
          reinterpret_cast<float4*>(dst)[1] = make_float4(acc[cc][4], acc[cc][5], acc[cc][6], acc[cc][7]);
        } else {
#pragma unroll
          for (int o = 0; o < H_XR; ++o)
            if (xo + o < W) dst[o] = acc[cc][o];
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K3: vertical pass + contraction with b_i(x) + guard + division
// ---------------------------------------------------------------------------
constexpr int V_YR = 8;  // output rows per thread
constexpr int V_CC = 4;  // planes per thread

template <int RT>
__device__ __forceinline__ void vfir(const VArgs& a, const float* __restrict__ col, int r0,
                                     float (&G)[V_YR]) {
  const int H = a.H, W = a.W, hp0 = a.hp_row0;
#pragma unroll
  for (int o = 0; o < V_YR; ++o) G[o] = 0.f;
  if (a.box) {
    const int R = a.R;
    float s = 0.f;
    for (int t = 0; t <= 2 * R; ++t)
      s += __ldg(col + (long long)(clampi(r0 - R + t, 0, H - 1) - hp0) * W);
    G[0] = s;
#pragma unroll
    for (int o = 1; o < V_YR; ++o) {
      s += __ldg(col + (long long)(clampi(r0 + o + R, 0, H - 1) - hp0) * W) -
           __ldg(col + (long long)(clampi(r0 + o - 1 - R, 0, H - 1) - hp0) * W);
      G[o] = s;
    }
    return;
  }
  if constexpr (RT > 0) {
    constexpr int T = 2 * RT + 1;
#pragma unroll
    for (int s = 0; s < V_YR + 2 * RT; ++s) {
      const float v = __ldg(col + (long long)(clampi(r0 - RT + s, 0, H - 1) - hp0) * W);
#pragma unroll
      for (int o = 0; o < V_YR; ++o) {
        const int t = s - o;
        if (t >= 0 && t < T) G[o] = fmaf(a.taps[t], v, G[o]);
      }
    }
  } else {
    const int R = a.R, T = 2 * R + 1;
    for (int t = 0; t < T; ++t) {
      const float w = a.taps[t];
#pragma unroll
      for (int o = 0; o < V_YR; ++o)
        G[o] = fmaf(w, __ldg(col + (long long)(clampi(r0 + o - R + t, 0, H - 1) - hp0) * W), G[o]);
    }
  }
}

template <int RT>
__global__ void __launch_bounds__(256) k_vpass(const VArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int m0 = a.m0, n = a.n, rho = a.rho, H = a.H, W = a.W, NC = n + 1;
  const int nchunks = a.nchunks, runs = a.runs;
  const int run = warp / nchunks, ch = warp - run * nchunks;
  const int tile_rows = runs * V_YR;
  const int npx = 32 * tile_rows;
  float* Cs = sm;                       // m0*rho
  float* U0 = Cs + (size_t)m0 * rho;    // m0
  float* bsh = U0 + m0;                 // 2 x npx (double buffer)
  float* ssh = bsh + 2 * npx;           // npx: s0 = u0.b per pixel
  float* dsh = ssh + npx;               // npx: eta (den)
  float* lsh = dsh + npx;               // npx: eta_lead
  __shared__ float red_min[32];
  __shared__ unsigned long long red_cnt[32];

  for (int k = threadIdx.x; k < m0 * rho; k += blockDim.x) Cs[k] = a.cst[k];
  for (int k = threadIdx.x; k < m0; k += blockDim.x) U0[k] = a.cst[a.u0_off + k];

  const int ntiles = a.tiles_x * a.tiles_y;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int xbase = tx * 32;
    const int r_base = a.out0 + ty * tile_rows;
    const int x = xbase + lane;
    const int xc = min(x, W - 1);
    const int r0 = r_base + run * V_YR;
    __syncthreads();
    for (int k = threadIdx.x; k < npx; k += blockDim.x) ssh[k] = 0.f;

    float acc[V_CC][V_YR];
#pragma unroll
    for (int cc = 0; cc < V_CC; ++cc)
#pragma unroll
      for (int o = 0; o < V_YR; ++o) acc[cc][o] = 0.f;

    for (int i = 0; i < m0; ++i) {
      float* bb = bsh + (i & 1) * npx;
      // b_i at every pixel of the tile (and the lead projection s0 += u0_i b_i)
      for (int k = threadIdx.x; k < npx; k += blockDim.x) {
        const int rr = min(r_base + (k >> 5), H - 1);
        const int cx = min(xbase + (k & 31), W - 1);
        float d2 = 0.f;
        for (int d = 0; d < rho; ++d) {
          const float t = guide_at(a.g, a.gps, a.f, a.fps, a.gkind, d, rr, cx, H, W) - Cs[i * rho + d];
          d2 = fmaf(t, t, d2);
        }
        const float b = range_kernel(d2, a.k2);
        bb[k] = b;
        ssh[k] = fmaf(U0[i], b, ssh[k]);
      }
      __syncthreads();
#pragma unroll
      for (int cc = 0; cc < V_CC; ++cc) {
        const int c = ch * V_CC + cc;
        if (c < NC) {
          float G[V_YR];
          vfir<RT>(a, a.hp + (long long)(i * NC + c) * a.hps + xc, r0, G);
#pragma unroll
          for (int o = 0; o < V_YR; ++o) acc[cc][o] = fmaf(bb[(run * V_YR + o) * 32 + lane], G[o], acc[cc][o]);
        }
      }
    }
    __syncthreads();  // ssh complete
    // rank-1 lead planes (k = 0 eigenpair): zeta_lead = s0 (ω*(s0 f)) / α0
    float lg[V_CC][V_YR];
#pragma unroll
    for (int cc = 0; cc < V_CC; ++cc) {
      const int c = ch * V_CC + cc;
      if (c < NC) {
        float G[V_YR];
        vfir<RT>(a, a.hp + (long long)(m0 * NC + c) * a.hps + xc, r0, G);
#pragma unroll
        for (int o = 0; o < V_YR; ++o) lg[cc][o] = ssh[(run * V_YR + o) * 32 + lane] * G[o] * a.inv_alpha0;
      } else {
#pragma unroll
        for (int o = 0; o < V_YR; ++o) lg[cc][o] = 0.f;
      }
    }
    if (ch == n / V_CC) {
      const int nsel = n % V_CC;
      static_assert(V_CC == 4, "selection below assumes 4 planes per thread");
#pragma unroll
      for (int o = 0; o < V_YR; ++o) {
        const float dv = nsel == 0 ? acc[0][o] : (nsel == 1 ? acc[1][o] : (nsel == 2 ? acc[2][o] : acc[3][o]));
        const float lv = nsel == 0 ? lg[0][o] : (nsel == 1 ? lg[1][o] : (nsel == 2 ? lg[2][o] : lg[3][o]));
        dsh[(run * V_YR + o) * 32 + lane] = dv;
        lsh[(run * V_YR + o) * 32 + lane] = lv;
      }
    }
    __syncthreads();

    float my_min = INFINITY;
    unsigned long long my_cnt = 0;
    const float eps = a.eps_den;
#pragma unroll
    for (int o = 0; o < V_YR; ++o) {
      const int row = r0 + o;
      const bool valid = x < W && row < H && row < a.out0 + a.out_rows;
      const float den = dsh[(run * V_YR + o) * 32 + lane];
      const float lden = lsh[(run * V_YR + o) * 32 + lane];
      const bool guarded = fabsf(den) < eps;
      if (valid && ch == 0) {
        my_min = fminf(my_min, fabsf(den));
        my_cnt += guarded ? 1ull : 0ull;
      }
#pragma unroll
      for (int cc = 0; cc < V_CC; ++cc) {
        const int c = ch * V_CC + cc;
        if (valid && c < n) {
          float v;
          if (!guarded) {
            v = acc[cc][o] / den;
          } else if (fabsf(lden) >= eps) {
            v = lg[cc][o] / lden;
          } else {
            v = __ldg(a.f + (long long)c * a.fps + (long long)row * W + x);
          }
          a.out[(long long)c * a.ops + (long long)row * W + x] = v;
        }
      }
    }
    // block reduction of the guard statistics (deterministic; atomics only across blocks)
    my_min = warp_min(my_min);
    my_cnt = warp_sum_u64(my_cnt);
    if (lane == 0) {
      red_min[warp] = my_min;
      red_cnt[warp] = my_cnt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      float mn = INFINITY;
      unsigned long long cnt = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        mn = fminf(mn, red_min[w]);
        cnt += red_cnt[w];
      }
      if (mn < INFINITY) atomicMin(&a.stats->min_abs_eta_bits, __float_as_uint(mn));
      if (cnt) atomicAdd(&a.stats->guarded, cnt);
    }
  }
}

// ---------------------------------------------------------------------------
// patch-guide materialisation (filters.py:174-181)
// ---------------------------------------------------------------------------
__global__ void k_patch_guide(const float* __restrict__ f, long long fps, int n, int H, int W, int r,
                              float* __restrict__ out, long long ops) {
  const int side = 2 * r + 1;
  const long long m = (long long)H * W;
  const int dim = n * side * side;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < m * dim;
       idx += (long long)gridDim.x * blockDim.x) {
    const int d = (int)(idx / m);
    const long long p = idx - d * m;
    const int y = (int)(p / W), x = (int)(p - (long long)y * W);
    const int c = d / (side * side), k = d - c * side * side, dy = k / side - r, dx = k % side - r;
    out[(long long)d * ops + p] =
        __ldg(f + (long long)c * fps + (long long)clampi(y + dy, 0, H - 1) * W + clampi(x + dx, 0, W - 1));
  }
}

__global__ void k_reset_stats(FilterStats* s) {
  s->min_abs_eta_bits = 0x7f800000u;  // +inf
  s->guarded = 0ull;
}

__global__ void k_copy_stats(const FilterStats* s, double* out) {
  out[0] = (double)__uint_as_float(s->min_abs_eta_bits);
  reinterpret_cast<long long*>(out)[1] = (long long)s->guarded;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int g_num_sms = 0;
static int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

static int validate(const nys_filter_desc* d) {
  if (!d) return NYS_EINVAL;
  if (d->n < 1 || d->n > NYS_MAX_CHANNELS || d->rho < 1 || d->rho > NYS_MAX_RHO) return NYS_EUNSUPPORTED;
  if (d->H < 1 || d->W < 1 || d->m0 < 1 || d->m0 > NYS_MAX_M0) return NYS_EINVAL;
  if (d->radius < 0 || d->radius > NYS_MAX_RADIUS) return NYS_EUNSUPPORTED;
  if (d->spatial_kind != NYS_SPATIAL_BOX && d->spatial_kind != NYS_SPATIAL_GAUSSIAN_FIR) return NYS_EUNSUPPORTED;
  if (d->spatial_kind == NYS_SPATIAL_GAUSSIAN_FIR && (!(d->sigma > 0) || d->radius < 1)) return NYS_EINVAL;
  if (!(d->theta > 0)) return NYS_EINVAL;
  if (d->guide_kind != 0 && d->guide_kind != 1) return NYS_EINVAL;
  if (d->guide_kind == 1 && d->rho != 9 * d->n) return NYS_EINVAL;
  return NYS_OK;
}

static void fill_taps(const nys_filter_desc* d, float* taps) {
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

static float k2_of(const nys_filter_desc* d) {
  return (float)(-1.4426950408889634 / (2.0 * d->theta * d->theta));
}

template <typename K>
static int set_smem(K kernel, size_t bytes) {
  NYS_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return NYS_OK;
}

}  // namespace nys

using namespace nys;

extern "C" {

size_t nys_filter_planes_bytes(const nys_filter_desc* d, int rows) {
  if (!d) return 0;
  return (size_t)(d->m0 + 1) * (d->n + 1) * (size_t)rows * (size_t)d->W * sizeof(float);
}

size_t nys_filter_workspace_bytes(const nys_filter_desc* d) {
  if (validate(d) != NYS_OK) return 0;
  return filter_layout(d).total_bytes;
}

int nys_filter_prepare(const nys_filter_desc* d, void* workspace, size_t workspace_bytes, void* stream) {
  int st = validate(d);
  if (st) return st;
  if (!d->centroids || !d->M || !d->u0 || !workspace) return NYS_EINVAL;
  const FilterLayout L = filter_layout(d);
  if (workspace_bytes < L.total_bytes) return NYS_EINVAL;
  std::vector<float> h(L.n_floats, 0.f);
  for (int j = 0; j < d->m0 * d->rho; ++j) h[L.off_C + j] = (float)d->centroids[j];
  for (int i = 0; i < d->m0; ++i)
    for (int j = 0; j < d->m0; ++j) h[L.off_MT + (size_t)j * L.m0p + i] = (float)d->M[(size_t)i * d->m0 + j];
  for (int j = 0; j < d->m0; ++j) h[L.off_U0 + j] = (float)d->u0[j];
  cudaStream_t s = (cudaStream_t)stream;
  NYS_CUDA_TRY(cudaMemcpyAsync(workspace, h.data(), L.n_floats * sizeof(float), cudaMemcpyHostToDevice, s));
  // pageable source: make sure the copy has consumed `h` before it goes away
  NYS_CUDA_TRY(cudaStreamSynchronize(s));
  count_launch(); k_reset_stats<<<1, 1, 0, s>>>(reinterpret_cast<FilterStats*>((char*)workspace + L.stats_off_bytes));
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

int nys_filter_hpass(const nys_filter_desc* d, const float* f, int64_t f_plane_stride, const float* guide,
                     int64_t guide_plane_stride, int row0, int rows, float* planes, int64_t planes_stride,
                     const void* workspace, void* stream) {
  int st = validate(d);
  if (st) return st;
  if (!f || !planes || !workspace || (d->guide_kind == 0 && !guide)) return NYS_EINVAL;
  if (row0 < 0 || rows < 1 || row0 + rows > d->H) return NYS_EINVAL;
  if (planes_stride < (int64_t)rows * d->W) return NYS_EINVAL;
  const FilterLayout L = filter_layout(d);
  HArgs a;
  memset(&a, 0, sizeof(a));
  a.f = f;
  a.g = d->guide_kind == 0 ? guide : f;
  a.hp = planes;
  a.cst = reinterpret_cast<const float*>(workspace);
  a.fps = f_plane_stride;
  a.gps = d->guide_kind == 0 ? guide_plane_stride : f_plane_stride;
  a.hps = planes_stride;
  a.n = d->n;
  a.rho = d->rho;
  a.H = d->H;
  a.W = d->W;
  a.m0 = d->m0;
  a.m0p = L.m0p;
  a.R = d->radius;
  a.box = d->spatial_kind == NYS_SPATIAL_BOX;
  a.gkind = d->guide_kind;
  a.row0 = row0;
  a.rows = rows;
  a.k2 = k2_of(d);
  fill_taps(d, a.taps);
  // tile width: as wide as the shared-memory budget allows (<= 256 columns)
  const size_t cst_floats = (size_t)d->m0 * d->rho + (size_t)d->m0 * L.m0p + L.m0p;
  const size_t per_col = (size_t)(d->n + (d->m0 + 1) + d->m0);
  const size_t budget = 200 * 1024;
  int TW = 256;
  auto smem_for = [&](int tw) {
    int pitch = tw + 2 * d->radius;
    pitch |= 1;  // odd pitch: rows of Ys map to distinct banks
    return std::make_pair(pitch, (cst_floats + per_col * (size_t)pitch) * sizeof(float));
  };
  while (TW > H_XR && smem_for(TW).second > budget) TW -= H_XR;
  if (smem_for(TW).second > budget) return NYS_EUNSUPPORTED;
  TW = std::min<int>(TW, (int)ceil_div(d->W, H_XR) * H_XR);
  const auto pr = smem_for(TW);
  a.TW = TW;
  a.pitch = pr.first;
  a.tiles_x = (int)ceil_div(d->W, TW);
  const long long ntiles = (long long)a.tiles_x * rows;
  const int grid = (int)std::min<long long>(ntiles, (long long)num_sms() * 8);
  cudaStream_t s = (cudaStream_t)stream;
#define NYS_H_CASE(RV)                                                     \
  case RV:                                                                 \
    st = set_smem(k_feat_hpass<RV>, pr.second);                            \
    if (st) return st;                                                     \
    count_launch(); k_feat_hpass<RV><<<grid, H_THREADS, pr.second, s>>>(a);                \
    break;
  const int rsel = a.box ? 0 : d->radius;
  switch (rsel) {
    NYS_H_CASE(9)
    NYS_H_CASE(12)
    NYS_H_CASE(15)
    NYS_H_CASE(18)
    default:
      st = set_smem(k_feat_hpass<0>, pr.second);
      if (st) return st;
      count_launch(); k_feat_hpass<0><<<grid, H_THREADS, pr.second, s>>>(a);
  }
#undef NYS_H_CASE
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

int nys_filter_vpass(const nys_filter_desc* d, const float* f, int64_t f_plane_stride, const float* guide,
                     int64_t guide_plane_stride, const float* planes, int64_t planes_stride, int planes_row0,
                     int out0, int out_rows, float* out, int64_t out_plane_stride, const void* workspace,
                     void* stream) {
  int st = validate(d);
  if (st) return st;
  if (!f || !planes || !out || !workspace || (d->guide_kind == 0 && !guide)) return NYS_EINVAL;
  if (out0 < 0 || out_rows < 1 || out0 + out_rows > d->H) return NYS_EINVAL;
  if (planes_row0 > std::max(0, out0 - d->radius)) return NYS_EINVAL;
  const FilterLayout L = filter_layout(d);
  VArgs a;
  memset(&a, 0, sizeof(a));
  a.f = f;
  a.g = d->guide_kind == 0 ? guide : f;
  a.hp = planes;
  a.out = out;
  a.cst = reinterpret_cast<const float*>(workspace);
  a.stats = reinterpret_cast<FilterStats*>((char*)const_cast<void*>(workspace) + L.stats_off_bytes);
  a.fps = f_plane_stride;
  a.gps = d->guide_kind == 0 ? guide_plane_stride : f_plane_stride;
  a.hps = planes_stride;
  a.ops = out_plane_stride;
  a.n = d->n;
  a.rho = d->rho;
  a.H = d->H;
  a.W = d->W;
  a.m0 = d->m0;
  a.R = d->radius;
  a.box = d->spatial_kind == NYS_SPATIAL_BOX;
  a.gkind = d->guide_kind;
  a.hp_row0 = planes_row0;
  a.u0_off = (long long)L.off_U0;
  a.out0 = out0;
  a.out_rows = out_rows;
  a.nchunks = (int)ceil_div(d->n + 1, V_CC);
  a.runs = std::max(1, 8 / a.nchunks);
  a.tiles_x = (int)ceil_div(d->W, 32);
  a.tiles_y = (int)ceil_div(out_rows, a.runs * V_YR);
  a.k2 = k2_of(d);
  a.inv_alpha0 = (float)(1.0 / d->alpha0);
  a.eps_den = (float)d->eps_den;
  fill_taps(d, a.taps);
  const int threads = 32 * a.runs * a.nchunks;
  if (threads > 256) return NYS_EUNSUPPORTED;
  const int npx = 32 * a.runs * V_YR;
  const size_t smem = ((size_t)d->m0 * d->rho + d->m0 + 5 * (size_t)npx) * sizeof(float);
  const long long ntiles = (long long)a.tiles_x * a.tiles_y;
  const int grid = (int)std::min<long long>(ntiles, (long long)num_sms() * 8);
  cudaStream_t s = (cudaStream_t)stream;
#define NYS_V_CASE(RV)                                            \
  case RV:                                                        \
    st = set_smem(k_vpass<RV>, smem);                             \
    if (st) return st;                                            \
    count_launch(); k_vpass<RV><<<grid, threads, smem, s>>>(a);                   \
    break;
  const int rsel = a.box ? 0 : d->radius;
  switch (rsel) {
    NYS_V_CASE(9)
    NYS_V_CASE(12)
    NYS_V_CASE(15)
    NYS_V_CASE(18)
    default:
      st = set_smem(k_vpass<0>, smem);
      if (st) return st;
      count_launch(); k_vpass<0><<<grid, threads, smem, s>>>(a);
  }
#undef NYS_V_CASE
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

int nys_filter_stats(const nys_filter_desc* d, const void* workspace, void* stats_out, void* stream) {
  int st = validate(d);
  if (st) return st;
  if (!workspace || !stats_out) return NYS_EINVAL;
  const FilterLayout L = filter_layout(d);
  count_launch(); k_copy_stats<<<1, 1, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const FilterStats*>((const char*)workspace + L.stats_off_bytes),
      reinterpret_cast<double*>(stats_out));
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

int nys_patch_guide(const float* f, int64_t f_plane_stride, int n, int H, int W, int r, float* out,
                    int64_t out_plane_stride, void* stream) {
  if (!f || !out || n < 1 || H < 1 || W < 1 || r < 0) return NYS_EINVAL;
  const long long total = (long long)H * W * n * (2 * r + 1) * (2 * r + 1);
  const int grid = (int)std::min<long long>(ceil_div(total, 256), (long long)num_sms() * 16);
  count_launch(); k_patch_guide<<<grid, 256, 0, (cudaStream_t)stream>>>(f, f_plane_stride, n, H, W, r, out, out_plane_stride);
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

}  // extern "C"
