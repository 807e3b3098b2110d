// K0 / K1 / K1f: k-means landmark selection in range space, B200 (sm_100a) CUDA.
//
// Reference region replaced (/root/reference/pkg/src/nysfilter/landmarks.py):
//   _plus_plus_init   60-73   -> k_pp_update (FP64 D^2, bit-exact per point) + k_pp_select
//   _assign (loop)    37-57   -> k_assign   (FP32 differenced distances, first index on ties)
//   Lloyd update      108-119 -> k_reduce + k_finalize (+ k_repair for empty clusters)
//   final _assign     121-129 -> k_exact    (FP64 differenced form, quant_error)
//
// Determinism: every reduction uses a fixed shape (per-thread sequential runs,
// fixed butterfly warp sums, warps and blocks combined in index order); no
// floating-point atomics.  The k-means++ uniforms come from the host (numpy
// default_rng(seed)), so the seed sequence matches the reference exactly as
// long as the D^2 prefix sums cross u*total at the same index (they differ
// from numpy's sequential cumsum only by FP64 rounding).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "nys_kmeans_dev.cuh"

namespace nys {

// ---------------------------------------------------------------------------
// k-means++ (landmarks.py:60-73)
// ---------------------------------------------------------------------------
__global__ void k_gather(const float* __restrict__ pts, long long ps, int rho, const long long* __restrict__ idxp,
                         long long idx_const, double* __restrict__ dst) {
  const long long idx = idxp ? *idxp : idx_const;
  for (int d = threadIdx.x; d < rho; d += blockDim.x) dst[d] = (double)pts[d * ps + idx];
}

// d2 = min(d2, |x - c|^2) over the contiguous chunk of block b; ppart[b] = Σ chunk
__global__ void __launch_bounds__(256) k_pp_update(const float* __restrict__ pts, long long ps, long long m,
                                                   int rho, const double* __restrict__ c, int init,
                                                   double* __restrict__ d2, double* __restrict__ ppart,
                                                   long long chunk, const KState* st) {
  __shared__ double sh[32];
  __shared__ double cs[NYS_MAX_RHO_WIDE];
  if (st && st->zero_draw >= 0) return;
  for (int d = threadIdx.x; d < rho; d += blockDim.x) cs[d] = c[d];
  __syncthreads();
  const long long lo = blockIdx.x * chunk, hi = min(m, lo + chunk);
  double s = 0.0;
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double v = d2_exact(pts, ps, i, rho, cs);
    const double nv = init ? v : fmin(d2[i], v);
    d2[i] = nv;
    s += nv;
  }
  const double t = block_sum(s, sh);
  if (threadIdx.x == 0) ppart[blockIdx.x] = t;
}

// exclusive prefix over per-block sums + the in-chunk scan that finds the first
// index whose running D^2 prefix exceeds u * total  (Generator.choice semantics)
__device__ long long pp_find(const double* __restrict__ d2, long long m, const double* __restrict__ ppart,
                             int nb, long long chunk, double target, double* sh, long long* shi) {
  // one thread resolves the owning block (nb <= 592 sequential adds)
  if (threadIdx.x == 0) {
    double pre = 0.0;
    int b = -1, last_pos = -1;
    for (int k = 0; k < nb; ++k) {
      if (ppart[k] > 0.0) last_pos = k;
      if (pre + ppart[k] > target) {
        b = k;
        break;
      }
      pre += ppart[k];
    }
    if (b < 0) {  // rounding pushed target past the end: take the last positive block
      b = last_pos;
      pre = 0.0;
      for (int k = 0; k < b; ++k) pre += ppart[k];
      target = pre + ppart[b] * (1.0 - 1e-16);
    }
    sh[0] = (double)b;
    sh[1] = target - pre;
  }
  __syncthreads();
  const int b = (int)sh[0];
  const double t = sh[1];
  const long long lo = b * chunk, hi = min(m, lo + chunk);
  const long long len = hi - lo;
  const long long per = ceil_div(len, (long long)blockDim.x);
  const long long s0 = lo + threadIdx.x * per, s1 = min(hi, s0 + per);
  double mine = 0.0;
  for (long long i = s0; i < s1; ++i) mine += d2[i];
  double* runs = sh + 2;
  runs[threadIdx.x] = mine;
  __syncthreads();
  if (threadIdx.x == 0) {
    double pre = 0.0;
    int owner = -1;
    for (int k = 0; k < (int)blockDim.x; ++k) {
      if (pre + runs[k] > t) {
        owner = k;
        break;
      }
      pre += runs[k];
    }
    if (owner < 0) {
      for (int k = (int)blockDim.x - 1; k >= 0; --k)
        if (runs[k] > 0.0) {
          owner = k;
          break;
        }
      pre = 0.0;
      for (int k = 0; k < owner; ++k) pre += runs[k];
    }
    long long idx = -1;
    const long long a0 = lo + (long long)owner * per, a1 = min(hi, a0 + per);
    double acc = pre;
    long long lastpos = -1;
    for (long long i = a0; i < a1; ++i) {
      if (d2[i] > 0.0) lastpos = i;
      acc += d2[i];
      if (acc > t) {
        idx = i;
        break;
      }
    }
    if (idx < 0) idx = lastpos;
    *shi = idx;
  }
  __syncthreads();
  return *shi;
}

__global__ void __launch_bounds__(1024) k_pp_select(const float* __restrict__ pts, long long ps, long long m, int rho,
                                                    const double* __restrict__ d2, const double* __restrict__ ppart,
                                                    int nb, long long chunk, double u, int draw,
                                                    double* __restrict__ cdst, long long* __restrict__ seed_idx,
                                                    KState* st) {
  __shared__ double sh[2 + 1024];
  __shared__ long long shi;
  if (st->zero_draw >= 0) return;
  // total in fixed order
  double v = 0.0;
  for (int k = threadIdx.x; k < nb; k += blockDim.x) v += ppart[k];
  const double total = block_sum(v, sh);
  __syncthreads();
  if (threadIdx.x == 0) sh[0] = total;
  __syncthreads();
  const double tot = sh[0];
  __syncthreads();
  if (!(tot > 0.0)) {
    if (threadIdx.x == 0) st->zero_draw = draw;
    return;
  }
  const long long idx = pp_find(d2, m, ppart, nb, chunk, u * tot, sh, &shi);
  if (threadIdx.x == 0 && seed_idx) seed_idx[draw] = idx;
  for (int d = threadIdx.x; d < rho; d += blockDim.x) cdst[d] = (double)pts[d * ps + idx];
}

// ---------------------------------------------------------------------------
// Lloyd assignment (landmarks.py:47-57 semantics, FP32 differenced distances)
// ---------------------------------------------------------------------------
template <int GR>
__global__ void __launch_bounds__(256) k_assign(const float* __restrict__ pts, long long ps, long long m, int rho,
                                                const float* __restrict__ Cf, int m0, int* __restrict__ labels,
                                                int first, double* __restrict__ part, int S, const KState* st) {
  extern __shared__ __align__(16) double dsm[];
  if (st && st->converged) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int slots = m0 * (rho + 1);
  double* wacc = dsm;                                  // nw x slots
  float* Cs = reinterpret_cast<float*>(dsm + (size_t)nw * slots);
  for (int k = threadIdx.x; k < nw * slots; k += blockDim.x) wacc[k] = 0.0;
  for (int k = threadIdx.x; k < m0 * rho; k += blockDim.x) Cs[k] = Cf[k];
  __syncthreads();
  double* my = wacc + (size_t)w * slots;
  double near_sum = 0.0;
  long long changed = 0;
  const long long chunk = ceil_div(m, (long long)gridDim.x);
  const long long lo = blockIdx.x * chunk, hi = min(m, lo + chunk);
  for (long long base = lo + (long long)w * 32; base < hi; base += (long long)nw * 32) {
    const long long i = base + lane;
    const bool valid = i < hi;
    float x[GR];
#pragma unroll
    for (int d = 0; d < GR; ++d) x[d] = (valid && d < rho) ? __ldg(pts + d * ps + i) : 0.f;
    float best = INFINITY;
    int arg = 0;
    for (int j = 0; j < m0; ++j) {
      float d2 = 0.f;
#pragma unroll
      for (int d = 0; d < GR; ++d)
        if (d < rho) {
          const float t = x[d] - Cs[j * rho + d];
          d2 = fmaf(t, t, d2);
        }
      if (d2 < best) {  // strict: first index wins ties (np.argmin)
        best = d2;
        arg = j;
      }
    }
    if (valid) {
      near_sum += (double)best;
      const int old = labels[i];
      if (first || old != arg) ++changed;
      labels[i] = arg;
    }
    // per-cluster coordinate sums: reduce each label group of the warp with a
    // fixed butterfly (zeros elsewhere), lane 0 owns this warp's accumulators
    unsigned rem = __ballot_sync(0xffffffffu, valid);
    while (rem) {
      const int leader = __ffs(rem) - 1;
      const int L = __shfl_sync(0xffffffffu, arg, leader);
      const unsigned grp = __ballot_sync(0xffffffffu, valid && arg == L);
      const bool in = (grp >> lane) & 1u;
#pragma unroll
      for (int d = 0; d < GR; ++d)
        if (d < rho) {
          const double s = warp_sum(in ? (double)x[d] : 0.0);
          if (lane == 0) my[L * (rho + 1) + d] += s;
        }
      if (lane == 0) my[L * (rho + 1) + rho] += (double)__popc(grp);
      rem &= ~grp;
    }
  }
  near_sum = warp_sum(near_sum);
  const double ch = warp_sum((double)changed);
  __shared__ double extra[2][32];
  if (lane == 0) {
    extra[0][w] = near_sum;
    extra[1][w] = ch;
  }
  __syncthreads();
  double* out = part + (size_t)blockIdx.x * S;
  for (int k = threadIdx.x; k < slots; k += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < nw; ++q) s += wacc[(size_t)q * slots + k];
    out[k] = s;
  }
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int q = 0; q < nw; ++q) {
      a += extra[0][q];
      b += extra[1][q];
    }
    out[slots] = a;
    out[slots + 1] = b;
  }
}

// Wide guides (rho > NYS_MAX_RHO): the same assignment with the coordinates read from the
// planar points inside the centroid loop (L1-resident) instead of registers.
__global__ void __launch_bounds__(256) k_assign_wide(const float* __restrict__ pts, long long ps, long long m, int rho,
                                                     const float* __restrict__ Cf, int m0, int* __restrict__ labels,
                                                     int first, double* __restrict__ part, int S, const KState* st) {
  extern __shared__ __align__(16) double dsm[];
  if (st && st->converged) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int slots = m0 * (rho + 1);
  double* wacc = dsm;                                  // nw x slots
  float* Cs = reinterpret_cast<float*>(dsm + (size_t)nw * slots);
  for (int k = threadIdx.x; k < nw * slots; k += blockDim.x) wacc[k] = 0.0;
  for (int k = threadIdx.x; k < m0 * rho; k += blockDim.x) Cs[k] = Cf[k];
  __syncthreads();
  double* my = wacc + (size_t)w * slots;
  double near_sum = 0.0;
  long long changed = 0;
  const long long chunk = ceil_div(m, (long long)gridDim.x);
  const long long lo = blockIdx.x * chunk, hi = min(m, lo + chunk);
  for (long long base = lo + (long long)w * 32; base < hi; base += (long long)nw * 32) {
    const long long i = base + lane;
    const bool valid = i < hi;
    const long long ii = valid ? i : lo;
    float best = INFINITY;
    int arg = 0;
    for (int j = 0; j < m0; ++j) {
      float d2 = 0.f;
      for (int d = 0; d < rho; ++d) {
        const float t = __ldg(pts + d * ps + ii) - Cs[j * rho + d];
        d2 = fmaf(t, t, d2);
      }
      if (d2 < best) {  // strict: first index wins ties (np.argmin)
        best = d2;
        arg = j;
      }
    }
    if (valid) {
      near_sum += (double)best;
      const int old = labels[i];
      if (first || old != arg) ++changed;
      labels[i] = arg;
    }
    unsigned rem = __ballot_sync(0xffffffffu, valid);
    while (rem) {
      const int leader = __ffs(rem) - 1;
      const int Lb = __shfl_sync(0xffffffffu, arg, leader);
      const unsigned grp = __ballot_sync(0xffffffffu, valid && arg == Lb);
      const bool in = (grp >> lane) & 1u;
      for (int d = 0; d < rho; ++d) {
        const double sd = warp_sum(in ? (double)__ldg(pts + d * ps + ii) : 0.0);
        if (lane == 0) my[Lb * (rho + 1) + d] += sd;
      }
      if (lane == 0) my[Lb * (rho + 1) + rho] += (double)__popc(grp);
      rem &= ~grp;
    }
  }
  near_sum = warp_sum(near_sum);
  const double ch = warp_sum((double)changed);
  __shared__ double extra[2][32];
  if (lane == 0) {
    extra[0][w] = near_sum;
    extra[1][w] = ch;
  }
  __syncthreads();
  double* out = part + (size_t)blockIdx.x * S;
  for (int k = threadIdx.x; k < slots; k += blockDim.x) {
    double sv = 0.0;
    for (int q = 0; q < nw; ++q) sv += wacc[(size_t)q * slots + k];
    out[k] = sv;
  }
  if (threadIdx.x == 0) {
    double a0 = 0.0, b0 = 0.0;
    for (int q = 0; q < nw; ++q) {
      a0 += extra[0][q];
      b0 += extra[1][q];
    }
    out[slots] = a0;
    out[slots + 1] = b0;
  }
}

// Wide guides: the exact (FP64 differenced) nearest distance straight, no FP32 screen
__global__ void __launch_bounds__(256) k_exact_wide(const float* __restrict__ pts, long long ps, long long m, int rho,
                                                    const double* __restrict__ C, int m0, long long* __restrict__ asg,
                                                    double* __restrict__ part) {
  __shared__ double sh[32];
  const long long chunk = ceil_div(m, (long long)gridDim.x);
  const long long lo = min(m, blockIdx.x * chunk), hi = min(m, lo + chunk);
  double s = 0.0;
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    double best = INFINITY;
    int arg = 0;
    for (int j = 0; j < m0; ++j) {
      const double v = d2_exact(pts, ps, i, rho, C + (size_t)j * rho);
      if (v < best) {
        best = v;
        arg = j;
      }
    }
    if (asg) asg[i] = arg;
    s += fmax(best, 0.0);
  }
  const double t = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// tot[k] = Σ_b part[b][k] in block order
__global__ void k_reduce(const double* __restrict__ part, int nb, int S, double* __restrict__ tot,
                         const KState* st) {
  if (st && st->converged) return;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= S) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += part[(size_t)b * S + k];
  tot[k] = s;
}

// Lloyd bookkeeping for iteration `it` (landmarks.py:101-119)
__global__ void k_finalize(const double* __restrict__ tot, int m0, int rho, int it, double* __restrict__ C,
                           double* __restrict__ Cprev, float* __restrict__ Cf, double* __restrict__ errors,
                           KState* st) {
  if (st->converged) return;
  const int slots = m0 * (rho + 1);
  const long long changed = (long long)tot[slots + 1];
  __syncthreads();
  if (threadIdx.x == 0) {
    errors[it] = tot[slots];
    st->iters = it + 1;
    st->changed = changed;
  }
  if (it > 0 && changed == 0) {
    if (threadIdx.x == 0) st->converged = 1;
    return;
  }
  for (int k = threadIdx.x; k < m0 * rho; k += blockDim.x) Cprev[k] = C[k];
  __syncthreads();
  for (int k = threadIdx.x; k < m0 * rho; k += blockDim.x) {
    const int j = k / rho, d = k - j * rho;
    const double cnt = tot[j * (rho + 1) + rho];
    if (cnt > 0.0) C[k] = tot[j * (rho + 1) + d] / cnt;
    Cf[k] = (float)C[k];
  }
  if (threadIdx.x == 0) {
    int ne = 0;
    for (int j = 0; j < m0; ++j) ne += tot[j * (rho + 1) + rho] > 0.0 ? 0 : 1;
    st->n_empty = ne;
  }
}

// empty-cluster repair (landmarks.py:114-119): for each empty j in ascending
// order take the point farthest from its (pre-update) centroid, excluding
// points already taken; first index on ties.  Rare; one block.
__global__ void __launch_bounds__(1024) k_repair(const float* __restrict__ pts, long long ps, long long m, int rho,
                                                 const int* __restrict__ labels, const double* __restrict__ tot,
                                                 int m0, double* __restrict__ C, const double* __restrict__ Cprev,
                                                 float* __restrict__ Cf, long long* __restrict__ excl, KState* st) {
  __shared__ double bv[1024];
  __shared__ long long bi[1024];
  if (st->converged || st->n_empty == 0) return;
  int nex = 0;
  for (int j = 0; j < m0; ++j) {
    if (tot[j * (rho + 1) + rho] > 0.0) continue;
    double best = -INFINITY;
    long long arg = m;
    for (long long i = threadIdx.x; i < m; i += blockDim.x) {
      bool ex = false;
      for (int q = 0; q < nex; ++q) ex |= (excl[q] == i);
      double v;
      if (ex) {
        v = -1.0;
      } else {
        v = d2_exact(pts, ps, i, rho, Cprev + (size_t)labels[i] * rho);
      }
      if (v > best) {
        best = v;
        arg = i;
      }
    }
    bv[threadIdx.x] = best;
    bi[threadIdx.x] = arg;
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = -INFINITY;
      long long a = m;
      for (int k = 0; k < (int)blockDim.x; ++k)
        if (bv[k] > b || (bv[k] == b && bi[k] < a)) {
          b = bv[k];
          a = bi[k];
        }
      excl[nex] = a;
      for (int d = 0; d < rho; ++d) {
        C[j * rho + d] = (double)pts[d * ps + a];
        Cf[j * rho + d] = pts[d * ps + a];
      }
      st->repairs += 1;
    }
    ++nex;
    __syncthreads();
  }
}

// Final exact assignment (landmarks.py:121-129): FP64 differenced distances in
// numpy's summation order, evaluated only where an FP32 bound cannot rule the
// centroid out.  With G_j = |c_j|^2 - 2 x.c~_j (FP32, c~ the FP32-rounded
// centroid, one FFMA per dimension) and F_j = G_j + |x|^2, the FP64 value E_j obeys
//   |F_j - E_j| <= (2 rho + 8) 2^-24 (|x|^2 + |c_j|^2)
// (operand rounding of c_j, FP32 products and sums, cancellation included), so
//   delta_j = A + B_j,  A = r |x|^2 + 2^-60,  B_j = r |c_j|^2,  r = (rho + 4) 2^-20
// over-covers it by 8x (the FP32 rounding of the bounds themselves included).
// The FP64 argmin j* satisfies F_j* - delta_j* <= E_j* <= E_k <= F_k + delta_k,
// so only centroids with G_j - B_j <= min_k (G_k + B_k) + 2A can be it (ties
// included); FP64 runs for those alone, in ascending j with a strict <, which
// returns exactly the brute-force FP64 label and value.  (G_j +- B_j are rounded
// once more in FP32; the 8x slack covers it.)
template <int GR, int RX>
__global__ void __launch_bounds__(256) k_exact(const float* __restrict__ pts, long long ps, long long m, int rho,
                                               const double* __restrict__ C, int m0, long long* __restrict__ asg,
                                               double* __restrict__ part) {
  extern __shared__ __align__(16) double csm[];
  __shared__ double sh[32];
  if (RX > 0) rho = RX;  // compile-time rho for the common small dimensions
  const int rhop = (rho + 3) & ~3;
  float* cf = reinterpret_cast<float*>(csm + (((size_t)m0 * rho + 1) & ~size_t(1)));  // m0 x rhop: -2 c~ (exact), 16 B aligned
  float* cn = cf + (size_t)m0 * rhop;  // |c_j|^2: start of the chain
  float* cb = cn + m0;                 // B_j = r |c_j|^2
  const double r = (double)(rho + 4) * 0x1p-20;
  for (int k = threadIdx.x; k < m0 * rho; k += blockDim.x) csm[k] = C[k];
  for (int k = threadIdx.x; k < m0 * rhop; k += blockDim.x) {
    const int j = k / rhop, d = k - j * rhop;
    cf[k] = d < rho ? -2.f * (float)C[(size_t)j * rho + d] : 0.f;
  }
  for (int j = threadIdx.x; j < m0; j += blockDim.x) {
    double t = 0.0;
    for (int d = 0; d < rho; ++d) t += C[(size_t)j * rho + d] * C[(size_t)j * rho + d];
    cn[j] = (float)t;
    cb[j] = __double2float_ru(r * t);
  }
  __syncthreads();
  const long long chunk = ceil_div(m, (long long)gridDim.x);
  const long long lo = min(m, blockIdx.x * chunk), hi = min(m, lo + chunk);
  double s = 0.0;
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    float x[GR];
    float xn = 0.f;
#pragma unroll
    for (int d = 0; d < GR; ++d) {
      x[d] = d < rho ? __ldg(pts + d * ps + i) : 0.f;
      xn = fmaf(x[d], x[d], xn);
    }
    auto chain = [&](int j, float start) {  // start - 2 x.c~_j
      const float* c = cf + (size_t)j * rhop;
      float acc = start;
#pragma unroll
      for (int d4 = 0; d4 < (GR + 3) / 4; ++d4) {
        if (4 * d4 < rho) {
          const float4 c4 = reinterpret_cast<const float4*>(c)[d4];
          const float cc[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (4 * d4 + e < GR && 4 * d4 + e < rho) acc = fmaf(x[4 * d4 + e], cc[e], acc);
        }
      }
      return acc;
    };
    // one pass: U = min (G_k + B_k) and the two smallest G_j - B_j; when the second of
    // those exceeds U + 2A only the first centroid can be the FP64 argmin
    float U = INFINITY, L1 = INFINITY, L2 = INFINITY;
    int j1 = 0;
    for (int j = 0; j < m0; ++j) {
      const float g = chain(j, cn[j]), b = cb[j];
      U = fminf(U, g + b);
      const float lb = g - b;
      if (lb < L1) {
        L2 = L1;
        L1 = lb;
        j1 = j;
      } else {
        L2 = fminf(L2, lb);
      }
    }
    const float thr = U + (float)(2.0 * (r * (double)xn + 0x1p-60));
    double best = INFINITY;
    int arg = 0;
    if (!(L2 <= thr)) {
      if (L1 <= thr) {
        best = d2_exact_regs<GR>(x, rho, csm + (size_t)j1 * rho);
        arg = j1;
      }
    } else {
      for (int j = 0; j < m0; ++j) {
        if (chain(j, cn[j]) - cb[j] <= thr) {
          const double v = d2_exact_regs<GR>(x, rho, csm + (size_t)j * rho);
          if (v < best) {
            best = v;
            arg = j;
          }
        }
      }
    }
    if (asg) asg[i] = arg;
    s += fmax(best, 0.0);
  }
  const double t = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

static int launch_exact(const float* pts, long long ps, long long m, int rho, const double* C, int m0, long long* asg,
                        double* part, int max_nb, int* nb_out, cudaStream_t s) {
  const size_t smem = (((size_t)m0 * rho + 1) & ~size_t(1)) * 8 + (size_t)m0 * ((rho + 3) & ~3) * 4 + (size_t)m0 * 8;
  auto go = [&](auto kern) -> int {
    // latency-bound loops: as many resident warps as the registers allow
    int per_sm = 0;
    NYS_CUDA_TRY(coop_blocks_per_sm((const void*)kern, 256, smem, &per_sm));
    const int nb = (int)std::max<long long>(
        1, std::min<long long>({ceil_div(m, 256LL), (long long)std::max(per_sm, 1) * sms(), (long long)max_nb}));
    *nb_out = nb;
    count_launch();
    kern<<<nb, 256, smem, s>>>(pts, ps, m, rho, C, m0, asg, part);
    NYS_LAUNCH_CHECK();
    return NYS_OK;
  };
  if (rho > NYS_MAX_RHO) {
    const int nb = (int)std::max<long long>(1, std::min<long long>(ceil_div(m, 256LL), (long long)max_nb));
    *nb_out = nb;
    count_launch();
    k_exact_wide<<<nb, 256, 0, s>>>(pts, ps, m, rho, C, m0, asg, part);
    NYS_LAUNCH_CHECK();
    return NYS_OK;
  }
  switch (rho) {
    case 1: return go(k_exact<4, 1>);
    case 2: return go(k_exact<4, 2>);
    case 3: return go(k_exact<4, 3>);
    case 4: return go(k_exact<4, 4>);
    default: break;
  }
  switch (rho) {  // exact compile-time dimensions of the BASELINE guides
    case 16: return go(k_exact<16, 16>);
    case 27: return go(k_exact<32, 27>);
    case 31: return go(k_exact<32, 31>);
    default: break;
  }
  if (rho <= 16) return go(k_exact<16, 0>);
  if (rho <= 32) return go(k_exact<32, 0>);
  return go(k_exact<64, 0>);
}

__global__ void k_sum_parts(const double* __restrict__ part, int nb, double* __restrict__ out) {
  __shared__ double sh[32];
  double v = 0.0;
  for (int k = threadIdx.x; k < nb; k += blockDim.x) v += part[k];
  const double t = block_sum(v, sh);
  if (threadIdx.x == 0) out[0] = t;
}

__global__ void k_init_state(KState* st, long long* seed_idx, long long first, double* C, int rho, int m0) {
  st->converged = 0;
  st->iters = 0;
  st->n_empty = 0;
  st->zero_draw = -1;
  st->changed = 0;
  st->repairs = 0;
  if (seed_idx) seed_idx[0] = first;
}

// everything the seeding needs before its first draw, in one launch: state reset, first
// pick, first centroid, the owner flag and the host's uniforms (passed by value, so no
// pageable host->device copy sits between the launches)
struct SeedPrologue {
  KState* st;
  long long* seeds;
  long long first;
  double* C;
  const float* pts;
  long long ps;
  int rho, m0;
  int* flag;
  double* unif_dst;
  unsigned long long* lloyd_gacc;  // Lloyd's first delta buffer (gstride words) and max|x| word
  int gstride;
  unsigned* lloyd_maxabs;
  double unif[NYS_MAX_M0];
};
__global__ void k_seed_prologue(const SeedPrologue p) {
  const int t = threadIdx.x;
  if (t == 0) {
    p.st->converged = 0;
    p.st->iters = 0;
    p.st->n_empty = 0;
    p.st->zero_draw = -1;
    p.st->changed = 0;
    p.st->repairs = 0;
    if (p.seeds) p.seeds[0] = p.first;
    *p.flag = 0;
  }
  for (int d = t; d < p.rho; d += blockDim.x) p.C[d] = (double)p.pts[d * p.ps + p.first];
  for (int k = t; k < p.m0 - 1; k += blockDim.x) p.unif_dst[k] = p.unif[k];
  for (int k = t; k < p.gstride; k += blockDim.x) p.lloyd_gacc[k] = 0ull;  // the seeding never touches these
  if (t < 7) p.lloyd_maxabs[t] = 0u;  // max|x| and the bounding box words of the cell-pruned search
}

__global__ void k_c_to_f(const double* __restrict__ C, float* __restrict__ Cf, int n) {
  for (int k = threadIdx.x; k < n; k += blockDim.x) Cf[k] = (float)C[k];
}

__global__ void k_write_stats(const KState* st, long long* out) {
  out[0] = st->iters;
  out[1] = st->zero_draw;
  out[2] = st->changed;
  out[3] = st->repairs;
}

// farthest point for the multi-GPU repair (value, local index) -- single block
__global__ void __launch_bounds__(1024) k_farthest(const float* __restrict__ pts, long long ps, long long m, int rho,
                                                   const double* __restrict__ C, const int* __restrict__ labels,
                                                   const long long* __restrict__ excl, int nex, double* out) {
  __shared__ double bv[1024];
  __shared__ long long bi[1024];
  double best = -INFINITY;
  long long arg = m;
  for (long long i = threadIdx.x; i < m; i += blockDim.x) {
    bool ex = false;
    for (int q = 0; q < nex; ++q) ex |= (excl[q] == i);
    const double v = ex ? -1.0 : d2_exact(pts, ps, i, rho, C + (size_t)labels[i] * rho);
    if (v > best) {
      best = v;
      arg = i;
    }
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = arg;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = -INFINITY;
    long long a = m;
    for (int k = 0; k < (int)blockDim.x; ++k)
      if (bv[k] > b || (bv[k] == b && bi[k] < a)) {
        b = bv[k];
        a = bi[k];
      }
    out[0] = b;
    out[1] = (double)a;
  }
}

__global__ void __launch_bounds__(1024) k_pick(const double* __restrict__ d2, long long m, const double* __restrict__ ppart,
                                               int nb, long long chunk, double target, long long* out) {
  __shared__ double sh[2 + 1024];
  __shared__ long long shi;
  double v = 0.0;
  for (int k = threadIdx.x; k < nb; k += blockDim.x) v += ppart[k];
  const double total = block_sum(v, sh);
  __syncthreads();
  if (threadIdx.x == 0) sh[0] = total;
  __syncthreads();
  const double tot = sh[0];
  __syncthreads();
  if (!(tot > 0.0) || target >= tot) {
    if (threadIdx.x == 0) *out = -1;
    return;
  }
  const long long idx = pp_find(d2, m, ppart, nb, chunk, target, sh, &shi);
  if (threadIdx.x == 0) *out = idx;
}

// ---------------------------------------------------------------------------
// row-band-sharded k-means, device resident (parallel.py): per k-means++ draw the
// ranks all-gather their D^2 totals and every rank resolves the draw from them with
// the same arithmetic; the owner writes the chosen point (+ its global index) into a
// candidate vector that an all-reduce(sum) then hands to everyone.  No host wait.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_pp_owner_pick(const float* __restrict__ pts, long long ps, long long m,
                                                        int rho, const double* __restrict__ d2,
                                                        const double* __restrict__ ppart, int nb, long long chunk,
                                                        const double* __restrict__ totals, int world, int rank,
                                                        long long my_offset, double u, int draw,
                                                        double* __restrict__ cand, KState* st) {
  __shared__ double sh[2 + 1024];
  __shared__ long long shi;
  __shared__ int owner_sh;
  __shared__ double local_target;
  for (int d = threadIdx.x; d <= rho; d += blockDim.x) cand[d] = 0.0;
  if (st->zero_draw >= 0) return;
  if (threadIdx.x == 0) {
    double total = 0.0;
    for (int r = 0; r < world; ++r) total += totals[r];  // rank order: identical on every rank
    int owner = -1;
    double t = 0.0;
    if (total > 0.0) {
      const double target = u * total;
      double pre = 0.0;
      int last_pos = -1;
      for (int r = 0; r < world; ++r) {
        if (totals[r] > 0.0) last_pos = r;
        if (pre + totals[r] > target) {
          owner = r;
          t = target - pre;
          break;
        }
        pre += totals[r];
      }
      if (owner < 0) {  // rounding pushed the target past the end (parallel.distributed_kmeans)
        owner = last_pos;
        t = totals[owner] * (1.0 - 1e-16);
      }
    } else {
      st->zero_draw = draw;  // sum(D^2) == 0: the reference switches to integers(m) (host fallback)
    }
    owner_sh = owner;
    local_target = t;
  }
  __syncthreads();
  if (owner_sh != rank) return;
  const long long idx = pp_find(d2, m, ppart, nb, chunk, local_target, sh, &shi);
  for (int d = threadIdx.x; d < rho; d += blockDim.x) cand[d] = (double)pts[d * ps + idx];
  if (threadIdx.x == 0) cand[rho] = (double)(my_offset + idx);
}

// One Lloyd assignment over the local points (full search, the FP32 difference form of the
// single-device kernels, first index on ties) with the cluster sums as EXACT fixed-point
// integers (x * 2^sexp rounded once per point, warp_accumulate_fx): per-block partials, then
// k_reduce_fx -- integer sums, so any order (blocks here, ranks in the all-reduce) gives the
// same bits, and the centroids equal the single-device cooperative kernel's.
template <int GR>
__global__ void __launch_bounds__(256) k_assign_fx(const float* __restrict__ pts, long long ps, long long m, int rho,
                                                   const float* __restrict__ Cf, int m0, int* __restrict__ labels,
                                                   int first, double scale, unsigned long long* __restrict__ bpart,
                                                   double* __restrict__ bobj, const KState* st) {
  extern __shared__ __align__(16) unsigned long long fsm[];
  if (st->converged) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int ns = m0 * rho;
  unsigned long long* wacc = fsm;                              // nw x ns
  int* wcnt = reinterpret_cast<int*>(wacc + (size_t)nw * ns);  // nw x m0
  float* Cs = reinterpret_cast<float*>(wcnt + (size_t)nw * m0);
  for (int k = threadIdx.x; k < nw * ns; k += blockDim.x) wacc[k] = 0ull;
  for (int k = threadIdx.x; k < nw * m0; k += blockDim.x) wcnt[k] = 0;
  for (int k = threadIdx.x; k < m0 * rho; k += blockDim.x) Cs[k] = Cf[k];
  __syncthreads();
  unsigned long long* myacc = wacc + (size_t)w * ns;
  int* mycnt = wcnt + (size_t)w * m0;
  double near_sum = 0.0;
  long long changed = 0;
  const long long chunk = ceil_div(m, (long long)gridDim.x);
  const long long lo = blockIdx.x * chunk, hi = min(m, lo + chunk);
  for (long long base = lo + (long long)w * 32; base < hi; base += (long long)nw * 32) {
    const long long i = base + lane;
    const bool valid = i < hi;
    float x[GR];
#pragma unroll
    for (int d = 0; d < GR; ++d) x[d] = (valid && d < rho) ? __ldg(pts + d * ps + i) : 0.f;
    float best = INFINITY;
    int arg = 0;
    for (int j = 0; j < m0; ++j) {
      float d2 = 0.f;
#pragma unroll
      for (int d = 0; d < GR; ++d)
        if (d < rho) {
          const float t = x[d] - Cs[j * rho + d];
          d2 = fmaf(t, t, d2);
        }
      if (d2 < best) {  // strict: first index wins ties (np.argmin)
        best = d2;
        arg = j;
      }
    }
    if (valid) {
      near_sum += (double)best;
      const int old = labels[i];
      if (first || old != arg) ++changed;
      labels[i] = arg;
    }
    warp_accumulate_fx<GR>(x, rho, arg, valid, scale, 1, myacc, mycnt);
  }
  near_sum = warp_sum(near_sum);
  const double ch = warp_sum((double)changed);
  __shared__ double extra[2][32];
  if (lane == 0) {
    extra[0][w] = near_sum;
    extra[1][w] = ch;
  }
  __syncthreads();
  const int S = ns + m0;
  unsigned long long* out = bpart + (size_t)blockIdx.x * S;
  for (int k = threadIdx.x; k < ns; k += blockDim.x) {
    unsigned long long v = 0ull;
    for (int q = 0; q < nw; ++q) v += wacc[(size_t)q * ns + k];
    out[k] = v;
  }
  for (int k = threadIdx.x; k < m0; k += blockDim.x) {
    long long v = 0;
    for (int q = 0; q < nw; ++q) v += wcnt[(size_t)q * m0 + k];
    out[ns + k] = (unsigned long long)v;
  }
  if (threadIdx.x == 0) {
    double a0 = 0.0, b0 = 0.0;
    for (int q = 0; q < nw; ++q) {
      a0 += extra[0][q];
      b0 += extra[1][q];
    }
    bobj[2 * blockIdx.x] = a0;
    bobj[2 * blockIdx.x + 1] = b0;
  }
}

// totals over the blocks: tot[0 .. S) integer sums and counts, tot[S] the changed count;
// obj[0] the objective (block order)
__global__ void k_reduce_fx(const unsigned long long* __restrict__ bpart, const double* __restrict__ bobj, int nb,
                            int S, unsigned long long* __restrict__ tot, double* __restrict__ obj, const KState* st) {
  if (st->converged) return;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < S) {
    unsigned long long v = 0ull;
    for (int b = 0; b < nb; ++b) v += bpart[(size_t)b * S + k];
    tot[k] = v;
  }
  if (k == S) {
    double o = 0.0, c = 0.0;
    for (int b = 0; b < nb; ++b) {
      o += bobj[2 * b];
      c += bobj[2 * b + 1];
    }
    obj[0] = o;
    tot[S] = (unsigned long long)(long long)c;
  }
}

// the reference's update and break rule on the all-reduced fixed-point totals
// (landmarks.py:101-119); empty clusters are left to the host fallback (k_mark_empty)
__global__ void k_finalize_fx(const long long* __restrict__ tot, const double* __restrict__ obj, int m0, int rho,
                              int it, double inv_scale, double* __restrict__ C, float* __restrict__ Cf,
                              double* __restrict__ errors, KState* st) {
  if (st->converged) return;
  const int ns = m0 * rho;
  const long long changed = tot[ns + m0];
  __syncthreads();
  if (threadIdx.x == 0) {
    errors[it] = obj[0];
    st->iters = it + 1;
    st->changed = changed;
  }
  if (it > 0 && changed == 0) {
    if (threadIdx.x == 0) st->converged = 1;
    return;
  }
  for (int k = threadIdx.x; k < ns; k += blockDim.x) {
    const int j = k / rho;
    const double cnt = (double)tot[ns + j];
    if (cnt > 0.0) C[k] = ((double)tot[k] * inv_scale) / cnt;
    Cf[k] = (float)C[k];
  }
  if (threadIdx.x == 0) {
    int ne = 0;
    for (int j = 0; j < m0; ++j) ne += tot[ns + j] > 0 ? 0 : 1;
    st->n_empty = ne;
  }
}

__global__ void k_state_init_sharded(KState* st) {
  st->converged = 0;
  st->iters = 0;
  st->n_empty = 0;
  st->zero_draw = -1;
  st->changed = 0;
  st->repairs = 0;
}

// after k_finalize on the all-reduced totals: an empty cluster needs the global farthest point,
// which the device-resident path does not resolve -- mark the run (repairs = -1) for the
// host-orchestrated fallback and stop iterating
__global__ void k_mark_empty(KState* st) {
  if (!st->converged && st->n_empty > 0) {
    st->repairs = -1;
    st->converged = 1;
  }
}

// ---------------------------------------------------------------------------
// host orchestration
// ---------------------------------------------------------------------------
static int launch_assign(const float* pts, long long ps, long long m, int rho, const float* Cf, int m0, int* labels,
                         int first, double* part, int nb, int S, const KState* st, cudaStream_t s) {
  const int slots = m0 * (rho + 1);
  // warps per block limited by the per-warp FP64 accumulators in shared memory
  const size_t budget = 160 * 1024;
  int nw = 8;
  while (nw > 1 && (size_t)nw * slots * 8 + (size_t)m0 * rho * 4 > budget) --nw;
  const size_t smem = (size_t)nw * slots * 8 + (size_t)m0 * rho * 4;
  if (smem > 220 * 1024) return NYS_EUNSUPPORTED;
#define NYS_A_CASE(G)                                                                                        \
  NYS_CUDA_TRY(cudaFuncSetAttribute(k_assign<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
  count_launch(); k_assign<G><<<nb, nw * 32, smem, s>>>(pts, ps, m, rho, Cf, m0, labels, first, part, S, st);
  if (rho <= 4) {
    NYS_A_CASE(4)
  } else if (rho <= 16) {
    NYS_A_CASE(16)
  } else if (rho <= 32) {
    NYS_A_CASE(32)
  } else if (rho <= NYS_MAX_RHO) {
    NYS_A_CASE(64)
  } else {
    NYS_CUDA_TRY(cudaFuncSetAttribute(k_assign_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    count_launch();
    k_assign_wide<<<nb, nw * 32, smem, s>>>(pts, ps, m, rho, Cf, m0, labels, first, part, S, st);
  }
#undef NYS_A_CASE
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

static int check_common(const float* pts, int64_t m, int rho, int m0, void* ws, size_t wsb) {
  if (!pts || m < 1 || rho < 1 || rho > NYS_MAX_RHO_WIDE || m0 < 1 || m0 > NYS_MAX_M0 || m0 > m) return NYS_EINVAL;
  if (!ws || wsb < klayout(m, rho, m0).total) return NYS_EINVAL;
  return NYS_OK;
}

static int run_lloyd_and_final(const float* pts, int64_t ps, int64_t m, int rho, int m0, int max_iter,
                               double* C, double* errors, int64_t* stats, double* qe, int64_t* asg,
                               char* ws, const KLayout& L, cudaStream_t s, bool prezeroed = false) {
  KState* st = reinterpret_cast<KState*>(ws + L.off_state);
  int* labels = reinterpret_cast<int*>(ws + L.off_labels);
  double* part = reinterpret_cast<double*>(ws + L.off_part);
  double* tot = reinterpret_cast<double*>(ws + L.off_tot);
  float* Cf = reinterpret_cast<float*>(ws + L.off_cf);
  double* Cprev = reinterpret_cast<double*>(ws + L.off_cprev);
  long long* excl = reinterpret_cast<long long*>(ws + L.off_excl);
  int rc = launch_lloyd_coop(pts, ps, m, rho, m0, max_iter, C, errors, ws, L, s, prezeroed);
  if (rc != NYS_OK && rc != NYS_EUNSUPPORTED) return rc;
  if (rc == NYS_EUNSUPPORTED) {  // step-wise (wide guides, or no cooperative launch)
    count_launch(); k_c_to_f<<<1, 256, 0, s>>>(C, Cf, m0 * rho);
    NYS_LAUNCH_CHECK();
    for (int it = 0; it < max_iter; ++it) {
      rc = launch_assign(pts, ps, m, rho, Cf, m0, labels, it == 0, part, L.nb_assign, L.S, st, s);
      if (rc) return rc;
      count_launch(); k_reduce<<<(int)ceil_div(L.S, 256), 256, 0, s>>>(part, L.nb_assign, L.S, tot, st);
      count_launch(); k_finalize<<<1, 256, 0, s>>>(tot, m0, rho, it, C, Cprev, Cf, errors, st);
      count_launch(); k_repair<<<1, 1024, 0, s>>>(pts, ps, m, rho, labels, tot, m0, C, Cprev, Cf, excl, st);
      NYS_LAUNCH_CHECK();
    }
  }
  if (qe || asg) {  // the final exact pass; callers that pass neither run nys_kmeans_exact later
    double* ppart = reinterpret_cast<double*>(ws + L.off_arg);
    int nbx = 0;
    int rc2 = launch_exact(pts, ps, m, rho, C, m0, reinterpret_cast<long long*>(asg), ppart, L.nb_exact, &nbx, s);
    if (rc2) return rc2;
    if (qe) {
      count_launch();
      k_sum_parts<<<1, 256, 0, s>>>(ppart, nbx, qe);
    }
  }
  count_launch(); k_write_stats<<<1, 1, 0, s>>>(st, reinterpret_cast<long long*>(stats));
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

}  // namespace nys

using namespace nys;

extern "C" {

int nys_abi_version(void) { return 100; }

size_t nys_kmeans_workspace_bytes(int64_t m, int rho, int m0) {
  if (m < 1 || rho < 1 || m0 < 1) return 0;
  return klayout(m, rho, m0).total;
}

int nys_kmeans_run(const float* points, int64_t plane_stride, int64_t m, int rho, int m0, int max_iter,
                   int64_t first_index, const double* uniforms, double* centroids_out, double* errors_out,
                   int64_t* stats_out, double* quant_error_out, int64_t* assignment_out,
                   int64_t* seed_indices_out, void* workspace, size_t workspace_bytes, void* stream) {
  int rc = check_common(points, m, rho, m0, workspace, workspace_bytes);
  if (rc) return rc;
  if (max_iter < 1 || first_index < 0 || first_index >= m || !centroids_out || !errors_out || !stats_out ||
      (m0 > 1 && !uniforms))
    return NYS_EINVAL;
  const KLayout L = klayout(m, rho, m0);
  char* ws = reinterpret_cast<char*>(workspace);
  cudaStream_t s = (cudaStream_t)stream;
  KState* st = reinterpret_cast<KState*>(ws + L.off_state);
  double* d2 = reinterpret_cast<double*>(ws + L.off_d2);
  double* ppart = reinterpret_cast<double*>(ws + L.off_ppart);
  long long* seeds = reinterpret_cast<long long*>(seed_indices_out);
  double* unif = reinterpret_cast<double*>(ws + L.off_unif);
  {
    SeedPrologue p;
    p.st = st;
    p.seeds = seeds;
    p.first = first_index;
    p.C = centroids_out;
    p.pts = points;
    p.ps = plane_stride;
    p.rho = rho;
    p.m0 = m0;
    p.flag = seed_flag(ws, L);
    p.unif_dst = unif;
    p.lloyd_gacc = reinterpret_cast<unsigned long long*>(ws + L.off_tot);
    p.gstride = m0 * rho + m0;
    p.lloyd_maxabs = reinterpret_cast<unsigned*>(ws + L.off_idx);
    for (int k = 0; k < m0 - 1; ++k) p.unif[k] = uniforms[k];
    count_launch();
    k_seed_prologue<<<1, 64, 0, s>>>(p);
    NYS_LAUNCH_CHECK();
  }
  rc = launch_seed_coop(points, plane_stride, m, rho, m0, unif, centroids_out, seeds, ws, L, s);
  if (rc != NYS_OK && rc != NYS_EUNSUPPORTED) return rc;
  const bool prezeroed = rc == NYS_OK;  // only the cooperative seeding is known to leave Lloyd's words alone
  if (rc == NYS_EUNSUPPORTED) {  // step-wise fallback: two launches per draw
    for (int j = 1; j < m0; ++j) {
      count_launch(); k_pp_update<<<L.nb_seed, 256, 0, s>>>(points, plane_stride, m, rho, centroids_out + (size_t)(j - 1) * rho,
                                            j == 1, d2, ppart, L.seed_chunk, st);
      count_launch(); k_pp_select<<<1, 1024, 0, s>>>(points, plane_stride, m, rho, d2, ppart, L.nb_seed, L.seed_chunk,
                                     uniforms[j - 1], j, centroids_out + (size_t)j * rho, seeds, st);
      NYS_LAUNCH_CHECK();
    }
  }
  return run_lloyd_and_final(points, plane_stride, m, rho, m0, max_iter, centroids_out, errors_out, stats_out,
                             quant_error_out, assignment_out, ws, L, s, prezeroed);
}

int nys_kmeans_run_seeded(const float* points, int64_t plane_stride, int64_t m, int rho, int m0, int max_iter,
                          const int64_t* seed_indices, double* centroids_out, double* errors_out,
                          int64_t* stats_out, double* quant_error_out, int64_t* assignment_out, void* workspace,
                          size_t workspace_bytes, void* stream) {
  int rc = check_common(points, m, rho, m0, workspace, workspace_bytes);
  if (rc) return rc;
  if (max_iter < 1 || !seed_indices || !centroids_out || !errors_out || !stats_out) return NYS_EINVAL;
  for (int j = 0; j < m0; ++j)
    if (seed_indices[j] < 0 || seed_indices[j] >= m) return NYS_EINVAL;
  const KLayout L = klayout(m, rho, m0);
  char* ws = reinterpret_cast<char*>(workspace);
  cudaStream_t s = (cudaStream_t)stream;
  KState* st = reinterpret_cast<KState*>(ws + L.off_state);
  count_launch(); k_init_state<<<1, 1, 0, s>>>(st, nullptr, 0, centroids_out, rho, m0);
  for (int j = 0; j < m0; ++j) {
    count_launch();
    k_gather<<<1, 64, 0, s>>>(points, plane_stride, rho, nullptr, seed_indices[j], centroids_out + (size_t)j * rho);
  }
  NYS_LAUNCH_CHECK();
  return run_lloyd_and_final(points, plane_stride, m, rho, m0, max_iter, centroids_out, errors_out, stats_out,
                             quant_error_out, assignment_out, ws, L, s);
}

int nys_kmeanspp_update(const float* points, int64_t plane_stride, int64_t m, int rho, const double* c, int init,
                        double* d2, double* sum_out, void* workspace, size_t workspace_bytes, void* stream) {
  if (!points || !c || !d2 || !sum_out || m < 1 || rho < 1 || rho > NYS_MAX_RHO_WIDE) return NYS_EINVAL;
  const KLayout L = klayout(m, rho, 1);
  if (!workspace || workspace_bytes < L.total) return NYS_EINVAL;
  char* ws = reinterpret_cast<char*>(workspace);
  double* ppart = reinterpret_cast<double*>(ws + L.off_ppart);
  cudaStream_t s = (cudaStream_t)stream;
  count_launch(); k_pp_update<<<L.nb_seed, 256, 0, s>>>(points, plane_stride, m, rho, c, init, d2, ppart, L.seed_chunk, nullptr);
  count_launch(); k_sum_parts<<<1, 256, 0, s>>>(ppart, L.nb_seed, sum_out);
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

int nys_kmeanspp_pick(const double* d2, int64_t m, double target, int64_t* index_out, void* workspace,
                      size_t workspace_bytes, void* stream) {
  if (!d2 || !index_out || m < 1) return NYS_EINVAL;
  const KLayout L = klayout(m, 1, 1);
  if (!workspace || workspace_bytes < L.total) return NYS_EINVAL;
  // the per-block sums of the last nys_kmeanspp_update on this workspace
  char* ws = reinterpret_cast<char*>(workspace);
  double* ppart = reinterpret_cast<double*>(ws + L.off_ppart);
  count_launch(); k_pick<<<1, 1024, 0, (cudaStream_t)stream>>>(d2, m, ppart, L.nb_seed, L.seed_chunk, target,
                                                reinterpret_cast<long long*>(index_out));
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

int nys_kmeans_assign(const float* points, int64_t plane_stride, int64_t m, int rho, const double* centroids, int m0,
                      int32_t* labels, int first_pass, double* acc_out, void* workspace, size_t workspace_bytes,
                      void* stream) {
  int rc = check_common(points, m, rho, m0, workspace, workspace_bytes);
  if (rc) return rc;
  if (!centroids || !labels || !acc_out) return NYS_EINVAL;
  const KLayout L = klayout(m, rho, m0);
  char* ws = reinterpret_cast<char*>(workspace);
  cudaStream_t s = (cudaStream_t)stream;
  float* Cf = reinterpret_cast<float*>(ws + L.off_cf);
  double* part = reinterpret_cast<double*>(ws + L.off_part);
  count_launch(); k_c_to_f<<<1, 256, 0, s>>>(centroids, Cf, m0 * rho);
  rc = launch_assign(points, plane_stride, m, rho, Cf, m0, labels, first_pass, part, L.nb_assign, L.S, nullptr, s);
  if (rc) return rc;
  count_launch(); k_reduce<<<(int)ceil_div(L.S, 256), 256, 0, s>>>(part, L.nb_assign, L.S, acc_out, nullptr);
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

int nys_kmeans_exact(const float* points, int64_t plane_stride, int64_t m, int rho, const double* centroids, int m0,
                     int64_t* assignment_out, double* sum_out, void* workspace, size_t workspace_bytes,
                     void* stream) {
  int rc = check_common(points, m, rho, m0, workspace, workspace_bytes);
  if (rc) return rc;
  if (!centroids || !sum_out) return NYS_EINVAL;
  const KLayout L = klayout(m, rho, m0);
  char* ws = reinterpret_cast<char*>(workspace);
  cudaStream_t s = (cudaStream_t)stream;
  double* ppart = reinterpret_cast<double*>(ws + L.off_arg);
  int nbx = 0;
  rc = launch_exact(points, plane_stride, m, rho, centroids, m0, reinterpret_cast<long long*>(assignment_out), ppart,
                    L.nb_exact, &nbx, s);
  if (rc) return rc;
  count_launch(); k_sum_parts<<<1, 256, 0, s>>>(ppart, nbx, sum_out);
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

int nys_kmeans_farthest(const float* points, int64_t plane_stride, int64_t m, int rho, const double* centroids, int m0,
                        const int32_t* labels, const int64_t* excluded, int n_excl, double* out, void* workspace,
                        size_t workspace_bytes, void* stream) {
  int rc = check_common(points, m, rho, m0, workspace, workspace_bytes);
  if (rc) return rc;
  if (!centroids || !labels || !out || (n_excl > 0 && !excluded)) return NYS_EINVAL;
  count_launch(); k_farthest<<<1, 1024, 0, (cudaStream_t)stream>>>(points, plane_stride, m, rho, centroids, labels,
                                                    reinterpret_cast<const long long*>(excluded), n_excl, out);
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

int nys_kmeans_state_init(void* workspace, size_t workspace_bytes, int64_t m, int rho, int m0, void* stream) {
  if (!workspace || m < 1 || rho < 1 || m0 < 1 || workspace_bytes < klayout(m, rho, m0).total) return NYS_EINVAL;
  const KLayout L = klayout(m, rho, m0);
  count_launch();
  k_state_init_sharded<<<1, 1, 0, (cudaStream_t)stream>>>(reinterpret_cast<KState*>((char*)workspace + L.off_state));
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

int nys_kmeans_state_read(const void* workspace, int64_t m, int rho, int m0, int64_t* stats_out, void* stream) {
  if (!workspace || !stats_out || m < 1 || rho < 1 || m0 < 1) return NYS_EINVAL;
  const KLayout L = klayout(m, rho, m0);
  count_launch();
  k_write_stats<<<1, 1, 0, (cudaStream_t)stream>>>(reinterpret_cast<const KState*>((const char*)workspace + L.off_state),
                                                  reinterpret_cast<long long*>(stats_out));
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

int nys_kmeanspp_owner_pick(const float* points, int64_t plane_stride, int64_t m, int rho, int m0, const double* d2,
                            const double* totals, int world, int rank, int64_t my_offset, double u, int draw,
                            double* cand_out, void* workspace, size_t workspace_bytes, void* stream) {
  if (!points || !d2 || !totals || !cand_out || m < 1 || rho < 1 || rho > NYS_MAX_RHO_WIDE || m0 < 1 || world < 1 ||
      rank < 0 || rank >= world)
    return NYS_EINVAL;
  const KLayout L = klayout(m, rho, m0);
  if (!workspace || workspace_bytes < L.total) return NYS_EINVAL;
  char* ws = reinterpret_cast<char*>(workspace);
  // ppart: the per-block sums of the last nys_kmeanspp_update on this workspace (their offset
  // and block shape depend on m only)
  const double* ppart = reinterpret_cast<const double*>(ws + L.off_ppart);
  count_launch();
  k_pp_owner_pick<<<1, 1024, 0, (cudaStream_t)stream>>>(points, plane_stride, m, rho, d2, ppart, L.nb_seed,
                                                         L.seed_chunk, totals, world, rank, my_offset, u, draw,
                                                         cand_out, reinterpret_cast<KState*>(ws + L.off_state));
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

int nys_kmeans_lloyd_local(const float* points, int64_t plane_stride, int64_t m, int rho, const double* centroids,
                           int m0, int it, int sexp, int64_t* tot_out, double* obj_out, void* workspace,
                           size_t workspace_bytes, void* stream) {
  int rc = check_common(points, m, rho, m0, workspace, workspace_bytes);
  if (rc) return rc;
  if (!centroids || !tot_out || !obj_out || it < 0) return NYS_EINVAL;
  const KLayout L = klayout(m, rho, m0);
  char* ws = reinterpret_cast<char*>(workspace);
  cudaStream_t s = (cudaStream_t)stream;
  KState* st = reinterpret_cast<KState*>(ws + L.off_state);
  float* Cf = reinterpret_cast<float*>(ws + L.off_cf);
  int* labels = reinterpret_cast<int*>(ws + L.off_labels);
  unsigned long long* bpart = reinterpret_cast<unsigned long long*>(ws + L.off_part);  // nb x (m0 rho + m0) <= nb x S
  double* bobj = reinterpret_cast<double*>(ws + L.off_arg);                            // nb x 2
  if (it == 0) {
    count_launch();
    k_c_to_f<<<1, 256, 0, s>>>(centroids, Cf, m0 * rho);  // later iterations: k_finalize_fx keeps Cf
  }
  const int ns = m0 * rho;
  int nw = 8;
  while (nw > 1 && (size_t)nw * (ns * 8 + m0 * 4) + (size_t)ns * 4 > 160 * 1024) --nw;
  const size_t smem = (size_t)nw * (ns * 8 + m0 * 4) + (size_t)ns * 4;
  const double scale = std::ldexp(1.0, sexp);
  const int nb = L.nb_assign;
#define NYS_AFX(G)                                                                                             \
  NYS_CUDA_TRY(cudaFuncSetAttribute(k_assign_fx<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
  count_launch();                                                                                              \
  k_assign_fx<G><<<nb, nw * 32, smem, s>>>(points, plane_stride, m, rho, Cf, m0, labels, it == 0, scale, bpart, bobj, st);
  if (rho <= 4) {
    NYS_AFX(4)
  } else if (rho <= 16) {
    NYS_AFX(16)
  } else if (rho <= 32) {
    NYS_AFX(32)
  } else {
    NYS_AFX(64)
  }
#undef NYS_AFX
  const int S = ns + m0;
  count_launch();
  k_reduce_fx<<<(int)ceil_div(S + 1, 256), 256, 0, s>>>(bpart, bobj, nb, S, reinterpret_cast<unsigned long long*>(tot_out),
                                                        obj_out, st);
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

int nys_kmeans_lloyd_update(int64_t m, int rho, int m0, int it, int sexp, const int64_t* tot, const double* obj,
                            double* centroids, double* errors, void* workspace, size_t workspace_bytes, void* stream) {
  if (!tot || !obj || !centroids || !errors || !workspace || m < 1 || rho < 1 || m0 < 1 || it < 0) return NYS_EINVAL;
  const KLayout L = klayout(m, rho, m0);
  if (workspace_bytes < L.total) return NYS_EINVAL;
  char* ws = reinterpret_cast<char*>(workspace);
  cudaStream_t s = (cudaStream_t)stream;
  KState* st = reinterpret_cast<KState*>(ws + L.off_state);
  count_launch();
  k_finalize_fx<<<1, 256, 0, s>>>(reinterpret_cast<const long long*>(tot), obj, m0, rho, it, std::ldexp(1.0, -sexp),
                                  centroids, reinterpret_cast<float*>(ws + L.off_cf), errors, st);
  count_launch();
  k_mark_empty<<<1, 1, 0, s>>>(st);
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

int nys_gather_point(const float* points, int64_t plane_stride, int rho, int64_t index, double* dst, void* stream) {
  if (!points || !dst || rho < 1 || index < 0) return NYS_EINVAL;
  count_launch(); k_gather<<<1, 64, 0, (cudaStream_t)stream>>>(points, plane_stride, rho, nullptr, index, dst);
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

}  // extern "C"
