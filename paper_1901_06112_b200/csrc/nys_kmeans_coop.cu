// Single-GPU k-means as two persistent cooperative kernels (one launch each):
//
//   k_seed_coop   k-means++ seeding (landmarks.py:60-73): m0-1 sequential D^2
//                 draws, each = one FP64 pass over the points + a grid-wide
//                 deterministic prefix search for the first index whose running
//                 D^2 sum exceeds u * total.  Two grid barriers per draw.
//   k_lloyd_coop  Lloyd iterations (landmarks.py:101-119): FP32 differenced
//                 assignment with first-index ties, warp-deterministic FP64
//                 cluster sums, slot-parallel cross-block reduction, the
//                 reference's break rule and empty-cluster repair.  Every block
//                 applies the (identical) centroid update itself, so the next
//                 assignment needs no extra launch.  Two barriers per iteration.
//
// Launch/latency cost replaced: ~2*m0 + 4*max_iter dependent tiny launches.
// Cross-block data (C, ppart, part, tot) is read with ld.global.cg so no SM
// sees a stale L1 line written by another SM before a grid barrier.
#include <cooperative_groups.h>

#include "nys_kmeans_dev.cuh"

namespace cg = cooperative_groups;

namespace nys {

struct SeedArgs {
  const float* pts;
  long long ps, m;
  int rho, m0;
  const double* uniforms;  // device, m0-1
  double* C;               // m0*rho FP64 (row 0 pre-filled)
  long long* seeds;        // m0 (nullable)
  double* d2;
  double* ppart;
  KState* st;
  int d2_in_smem;
};

// owner search over vals[0..n) for the first index whose running sum exceeds
// `target`: each thread sums a contiguous run, the run sums are scanned, the
// owning thread walks its run.  If rounding pushed target past the end, the
// last positive index is returned.  *before_out (nullable) receives the
// running sum of all values before the returned index.  CG: vals were
// written by other blocks (read with ld.global.cg); otherwise plain loads
// (shared memory or this block's own global writes).
template <bool CG>
__device__ long long scan_find(const double* vals, long long n, double target, double* sh, int* shi,
                               double* before_out) {
  auto ld = [&](long long i) { return CG ? __ldcg(vals + i) : vals[i]; };
  const long long per = ceil_div(n, (long long)blockDim.x);
  const long long a0 = min(n, (long long)threadIdx.x * per), a1 = min(n, a0 + per);
  double mine = 0.0;
  long long lastpos = -1;
  for (long long i = a0; i < a1; ++i) {
    const double v = ld(i);
    mine += v;
    if (v > 0.0) lastpos = i;
  }
  const double incl = block_incl_scan(mine, sh);
  __shared__ long long res_sh;
  __shared__ double pre_sh;
  const int owner = block_first_true(incl > target, shi);
  if (threadIdx.x == 0) res_sh = -1;
  __syncthreads();
  if ((int)threadIdx.x == owner) {
    double acc = incl - mine;
    long long idx = -1;
    for (long long i = a0; i < a1; ++i) {
      const double v = ld(i);
      if (acc + v > target) {
        idx = i;
        break;
      }
      acc += v;
    }
    if (idx < 0) {  // rounding inside the run: fall back to its last positive value
      idx = lastpos;
      acc = incl - mine;
      for (long long i = a0; i < idx; ++i) acc += ld(i);
    }
    res_sh = idx;
    pre_sh = acc;
  }
  __syncthreads();
  if (owner == (int)blockDim.x) {
    // no prefix exceeded target (rounding): last positive value overall
    long long lp = lastpos;
    for (int o = 16; o > 0; o >>= 1) lp = max(lp, __shfl_xor_sync(0xffffffffu, lp, o));
    __shared__ long long lps[32];
    if ((threadIdx.x & 31) == 0) lps[threadIdx.x >> 5] = lp;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long r = -1;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = max(r, lps[w]);
      res_sh = r;
      double acc = 0.0;
      for (long long i = 0; i < r; ++i) acc += ld(i);
      pre_sh = acc;
    }
    __syncthreads();
  }
  const long long r = res_sh;
  if (before_out) *before_out = pre_sh;
  __syncthreads();
  return r;
}

template <int GR>
__device__ __forceinline__ double d2_exact_r(const float (&x)[GR], int rho, const double* __restrict__ c) {
  if (GR <= 8 || rho < 8) {
    double r = 0.0;
#pragma unroll
    for (int d = 0; d < (GR < 8 ? GR : 8); ++d)
      if (d < rho) r = __dadd_rn(r, sqdiff((double)x[d], c[d]));
    return r;
  }
  double r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = sqdiff((double)x[k], c[k]);
  const int full = rho - (rho % 8);
#pragma unroll
  for (int d = 8; d < GR; d += 8)
    if (d < full) {
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], sqdiff((double)x[d + k], c[d + k]));
    }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
#pragma unroll
  for (int d = 0; d < GR; ++d)
    if (d >= full && d < rho) res = __dadd_rn(res, sqdiff((double)x[d], c[d]));
  return res;
}

template <int GR>
__global__ void __launch_bounds__(512) k_seed_coop(const SeedArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double d2s[];  // this block's chunk of D^2 when it fits
  __shared__ double cs[NYS_MAX_RHO];
  __shared__ double sh[64];
  __shared__ int shi[2];
  __shared__ long long sel[1];
  __shared__ double tot_sh;
  const int nb = gridDim.x, b = blockIdx.x, rho = a.rho;
  const long long chunk = ceil_div(a.m, (long long)nb);
  const long long lo = min(a.m, b * chunk), hi = min(a.m, lo + chunk);
  const int len = (int)(hi - lo);
  double* d2 = a.d2_in_smem ? d2s : a.d2 + lo;
  const int B = blockDim.x;
  for (int j = 1; j < a.m0; ++j) {
    if ((int)threadIdx.x < rho) cs[threadIdx.x] = __ldcg(a.C + (size_t)(j - 1) * rho + threadIdx.x);
    __syncthreads();
    double s = 0.0;
    int i = threadIdx.x;
    for (; i + 3 * B < len; i += 4 * B) {  // 4 independent points in flight
      float x[4][GR];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int d = 0; d < GR; ++d) x[u][d] = d < rho ? __ldg(a.pts + d * a.ps + lo + i + u * B) : 0.f;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double v = d2_exact_r<GR>(x[u], rho, cs);
        const double nv = j == 1 ? v : fmin(d2[i + u * B], v);
        d2[i + u * B] = nv;
        s += nv;
      }
    }
    for (; i < len; i += B) {
      float x[GR];
#pragma unroll
      for (int d = 0; d < GR; ++d) x[d] = d < rho ? __ldg(a.pts + d * a.ps + lo + i) : 0.f;
      const double v = d2_exact_r<GR>(x, rho, cs);
      const double nv = j == 1 ? v : fmin(d2[i], v);
      d2[i] = nv;
      s += nv;
    }
    const double bs = block_sum(s, sh);
    if (threadIdx.x == 0) a.ppart[b] = bs;
    grid.sync();
    // every block resolves the owning block redundantly (identical arithmetic)
    double total;
    {
      const long long per = ceil_div((long long)nb, (long long)B);
      const long long a0 = min((long long)nb, (long long)threadIdx.x * per), a1 = min((long long)nb, a0 + per);
      double mine = 0.0;
      for (long long q = a0; q < a1; ++q) mine += __ldcg(a.ppart + q);
      const double incl = block_incl_scan(mine, sh);
      if (threadIdx.x == B - 1) tot_sh = incl;
      __syncthreads();
      total = tot_sh;
    }
    if (!(total > 0.0)) {  // sum(D^2) == 0: the reference switches to rng.integers (host redo)
      if (b == 0 && threadIdx.x == 0) a.st->zero_draw = j;
      return;  // uniform across the grid
    }
    const double target = a.uniforms[j - 1] * total;
    double before = 0.0;
    const long long bstar = scan_find<true>(a.ppart, nb, target, sh, shi, &before);
    if (b == (int)bstar) {
      const long long k = scan_find<false>(d2, len, target - before, sh, shi, nullptr);
      if (threadIdx.x == 0) sel[0] = lo + max(0ll, k);
      __syncthreads();
      const long long idx = sel[0];
      if ((int)threadIdx.x < rho) a.C[(size_t)j * rho + threadIdx.x] = (double)__ldg(a.pts + threadIdx.x * a.ps + idx);
      if (threadIdx.x == 0 && a.seeds) a.seeds[j] = idx;
    }
    grid.sync();
  }
}

struct LloydArgs {
  const float* pts;
  long long ps, m;
  int rho, m0, max_iter, S;
  double* C;        // in: seeds; out: final centroids
  int* labels;
  double* part;     // nb x S
  double* tot;      // S
  double* arg;      // 2 x nb x 2 (double-buffered argmax pairs)
  double* errors;
  KState* st;
  int nw;           // warps per block
};

template <int GR>
__global__ void __launch_bounds__(256) k_lloyd_coop(const LloydArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double dsm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int rho = a.rho, m0 = a.m0, slots = m0 * (rho + 1), S = a.S;
  double* wacc = dsm;                                   // nw x slots
  double* Cd = wacc + (size_t)max(nw * slots, S);       // m0*rho current centroids (FP64)
  double* Cp = Cd + (size_t)m0 * rho;                   // m0*rho previous centroids
  long long* excl = reinterpret_cast<long long*>(Cp + (size_t)m0 * rho);  // m0
  float* Cf = reinterpret_cast<float*>(excl + m0);      // m0*rho FP32 copy for the assignment
  __shared__ double sh[64];
  __shared__ double extra[2][32];
  const int nb = gridDim.x, b = blockIdx.x;
  const long long chunk = ceil_div(a.m, (long long)nb);
  const long long lo = min(a.m, b * chunk), hi = min(a.m, lo + chunk);

  for (int k = threadIdx.x; k < m0 * rho; k += blockDim.x) Cd[k] = __ldcg(a.C + k);
  __syncthreads();
  for (int it = 0; it < a.max_iter; ++it) {
    for (int k = threadIdx.x; k < m0 * rho; k += blockDim.x) Cf[k] = (float)Cd[k];
    for (int k = threadIdx.x; k < nw * slots; k += blockDim.x) wacc[k] = 0.0;
    __syncthreads();
    double* my = wacc + (size_t)w * slots;
    double near_sum = 0.0, changed = 0.0;
    for (long long base = lo + (long long)w * 32; base < hi; base += (long long)nw * 32) {
      const long long i = base + lane;
      const bool valid = i < hi;
      float x[GR];
#pragma unroll
      for (int d = 0; d < GR; ++d) x[d] = (valid && d < rho) ? __ldg(a.pts + d * a.ps + i) : 0.f;
      float best = INFINITY;
      int arg = 0;
      for (int j = 0; j < m0; ++j) {
        float d2 = 0.f;
#pragma unroll
        for (int d = 0; d < GR; ++d)
          if (d < rho) {
            const float t = x[d] - Cf[j * rho + d];
            d2 = fmaf(t, t, d2);
          }
        if (d2 < best) {  // strict: first index wins ties (np.argmin)
          best = d2;
          arg = j;
        }
      }
      if (valid) {
        near_sum += (double)best;
        const int old = a.labels[i];
        if (it == 0 || old != arg) changed += 1.0;
        a.labels[i] = arg;
      }
      warp_accumulate<GR>(x, rho, arg, valid, my);
    }
    near_sum = warp_sum(near_sum);
    changed = warp_sum(changed);
    if (lane == 0) {
      extra[0][w] = near_sum;
      extra[1][w] = changed;
    }
    __syncthreads();
    double* out = a.part + (size_t)b * S;
    for (int k = threadIdx.x; k < slots; k += blockDim.x) {
      double s = 0.0;
      for (int q = 0; q < nw; ++q) s += wacc[(size_t)q * slots + k];
      out[k] = s;
    }
    if (threadIdx.x == 0) {
      double e = 0.0, c = 0.0;
      for (int q = 0; q < nw; ++q) {
        e += extra[0][q];
        c += extra[1][q];
      }
      out[slots] = e;
      out[slots + 1] = c;
    }
    grid.sync();
    // cross-block reduction: one warp per slot, lanes stride over the blocks,
    // fixed butterfly -> deterministic; latency ~ nb/32 loads instead of nb
    {
      const int gw = (b * (int)blockDim.x + (int)threadIdx.x) >> 5;
      const int nwarps = (nb * (int)blockDim.x) >> 5;
      for (int k = gw; k < S; k += nwarps) {
        double s0 = 0.0, s1 = 0.0;
        int q = lane;
        for (; q + 32 < nb; q += 64) {
          s0 += __ldcg(a.part + (size_t)q * S + k);
          s1 += __ldcg(a.part + (size_t)(q + 32) * S + k);
        }
        if (q < nb) s0 += __ldcg(a.part + (size_t)q * S + k);
        const double t = warp_sum(s0 + s1);
        if (lane == 0) a.tot[k] = t;
      }
    }
    grid.sync();
    // every block pulls the totals into shared memory once
    double* tsh = wacc;  // reuse: the per-warp accumulators are rebuilt next iteration
    for (int k = threadIdx.x; k < S; k += blockDim.x) tsh[k] = __ldcg(a.tot + k);
    __syncthreads();
    const double chg = tsh[slots + 1];
    if (b == 0 && threadIdx.x == 0) {
      a.errors[it] = tsh[slots];
      a.st->iters = it + 1;
      a.st->changed = (long long)chg;
    }
    if (it > 0 && chg == 0.0) {
      if (b == 0 && threadIdx.x == 0) a.st->converged = 1;
      break;  // uniform: every block read the same total
    }
    for (int k = threadIdx.x; k < m0 * rho; k += blockDim.x) {
      Cp[k] = Cd[k];
      const int j = k / rho, d = k - j * rho;
      const double cnt = tsh[j * (rho + 1) + rho];
      if (cnt > 0.0) Cd[k] = tsh[j * (rho + 1) + d] / cnt;
    }
    __syncthreads();
    // empty clusters, ascending j: farthest remaining point from its old centroid
    int nex = 0;
    for (int j = 0; j < m0; ++j) {
      if (tsh[j * (rho + 1) + rho] > 0.0) continue;
      double bv = -INFINITY;
      long long bi = a.m;
      for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        bool ex = false;
        for (int q = 0; q < nex; ++q) ex |= (excl[q] == i);
        const double v = ex ? -1.0 : d2_exact(a.pts, a.ps, i, rho, Cp + (size_t)a.labels[i] * rho);
        if (v > bv) {
          bv = v;
          bi = i;
        }
      }
      // block argmax (value desc, index asc)
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      __shared__ double wv[32];
      __shared__ long long wi[32];
      if (lane == 0) {
        wv[w] = bv;
        wi[w] = bi;
      }
      __syncthreads();
      double* pairs = a.arg + (size_t)(nex & 1) * nb * 2;
      if (threadIdx.x == 0) {
        double v = -INFINITY;
        long long ix = a.m;
        for (int q = 0; q < nw; ++q)
          if (wv[q] > v || (wv[q] == v && wi[q] < ix)) {
            v = wv[q];
            ix = wi[q];
          }
        pairs[2 * b] = v;
        pairs[2 * b + 1] = (double)ix;
      }
      grid.sync();
      if (threadIdx.x == 0) {
        double v = -INFINITY;
        long long ix = a.m;
        for (int q = 0; q < nb; ++q) {
          const double qv = __ldcg(pairs + 2 * q);
          const long long qi = (long long)__ldcg(pairs + 2 * q + 1);
          if (qv > v || (qv == v && qi < ix)) {
            v = qv;
            ix = qi;
          }
        }
        excl[nex] = ix;
        if (b == 0) a.st->repairs += 1;
      }
      __syncthreads();
      const long long idx = excl[nex];
      for (int d = threadIdx.x; d < rho; d += blockDim.x) Cd[j * rho + d] = (double)__ldg(a.pts + d * a.ps + idx);
      ++nex;
      __syncthreads();
    }
    __syncthreads();  // tsh aliases wacc: nobody may still read the totals when it is re-zeroed
  }
  if (b == 0)
    for (int k = threadIdx.x; k < m0 * rho; k += blockDim.x) a.C[k] = Cd[k];
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
int launch_seed_coop(const float* pts, long long ps, long long m, int rho, int m0, const double* uniforms_dev,
                     double* C, long long* seeds, char* ws, const KLayout& L, cudaStream_t s) {
  if (m0 < 2) return NYS_OK;
  int dev = 0, coop = 0;
  NYS_CUDA_TRY(cudaGetDevice(&dev));
  NYS_CUDA_TRY(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  if (!coop) return NYS_EUNSUPPORTED;
  SeedArgs a;
  a.pts = pts;
  a.ps = ps;
  a.m = m;
  a.rho = rho;
  a.m0 = m0;
  a.uniforms = uniforms_dev;
  a.C = C;
  a.seeds = seeds;
  a.d2 = reinterpret_cast<double*>(ws + L.off_d2);
  a.ppart = reinterpret_cast<double*>(ws + L.off_ppart);
  a.st = reinterpret_cast<KState*>(ws + L.off_state);
  void* args[] = {&a};
  auto go = [&](auto kern) -> int {
    // one block per SM; the block's D^2 chunk lives in shared memory when it fits
    const int nb = (int)std::max<long long>(1, std::min<long long>((long long)sms(), ceil_div(m, 512)));
    const long long chunk = ceil_div(m, (long long)nb);
    size_t smem = (size_t)chunk * 8;
    a.d2_in_smem = smem <= 200 * 1024;
    if (!a.d2_in_smem) smem = 0;
    NYS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smem, 1)));
    int per_sm = 0;
    NYS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 512, smem));
    if (per_sm < 1) return NYS_EUNSUPPORTED;
    count_launch();
    NYS_CUDA_TRY(cudaLaunchCooperativeKernel((void*)kern, dim3(nb), dim3(512), args, smem, s));
    return NYS_OK;
  };
  if (rho <= 4) return go(k_seed_coop<4>);
  if (rho <= 16) return go(k_seed_coop<16>);
  if (rho <= 32) return go(k_seed_coop<32>);
  return go(k_seed_coop<64>);
}

int launch_lloyd_coop(const float* pts, long long ps, long long m, int rho, int m0, int max_iter, double* C,
                      double* errors, char* ws, const KLayout& L, cudaStream_t s) {
  int dev = 0, coop = 0;
  NYS_CUDA_TRY(cudaGetDevice(&dev));
  NYS_CUDA_TRY(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  if (!coop) return NYS_EUNSUPPORTED;
  const int slots = m0 * (rho + 1);
  const size_t fixed = (size_t)m0 * rho * 8 * 2 + (size_t)m0 * 8 + (size_t)m0 * rho * 4 + 64;
  int nw = 8;
  while (nw > 1 && (size_t)std::max(nw * slots, L.S) * 8 + fixed > 200 * 1024) --nw;
  const size_t smem = (size_t)std::max(nw * slots, L.S) * 8 + fixed;
  if (smem > 220 * 1024) return NYS_EUNSUPPORTED;
  LloydArgs a;
  a.pts = pts;
  a.ps = ps;
  a.m = m;
  a.rho = rho;
  a.m0 = m0;
  a.max_iter = max_iter;
  a.S = L.S;
  a.C = C;
  a.labels = reinterpret_cast<int*>(ws + L.off_labels);
  a.part = reinterpret_cast<double*>(ws + L.off_part);
  a.tot = reinterpret_cast<double*>(ws + L.off_tot);
  a.arg = reinterpret_cast<double*>(ws + L.off_arg);
  a.errors = errors;
  a.st = reinterpret_cast<KState*>(ws + L.off_state);
  a.nw = nw;
  void* args[] = {&a};
  auto go = [&](auto kern) -> int {
    int per_sm = 0;
    NYS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    NYS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nw * 32, smem));
    if (per_sm < 1) return NYS_EUNSUPPORTED;
    const int nb = (int)std::max<long long>(
        1, std::min<long long>({(long long)per_sm * sms(), (long long)L.nb_coop, ceil_div(m, (long long)nw * 32)}));
    count_launch();
    NYS_CUDA_TRY(cudaLaunchCooperativeKernel((void*)kern, dim3(nb), dim3(nw * 32), args, smem, s));
    return NYS_OK;
  };
  if (rho <= 4) return go(k_lloyd_coop<4>);
  if (rho <= 16) return go(k_lloyd_coop<16>);
  if (rho <= 32) return go(k_lloyd_coop<32>);
  return go(k_lloyd_coop<64>);
}

}  // namespace nys
