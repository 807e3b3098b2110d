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
};

// owner search over `vals[0..n)` (global, read with ld.cg) for the first index
// whose running sum exceeds `target`; each thread sums a contiguous run, the
// runs are scanned, the owning thread walks its run.  Returns index (or the
// last positive index if rounding pushed target past the end) and the sum of
// all values before that index through *pre_out (thread 0 result).
__device__ long long scan_find(const double* vals, long long n, double target, double* sh, int* shi,
                               double* total_out) {
  const long long per = ceil_div(n, (long long)blockDim.x);
  const long long a0 = min(n, (long long)threadIdx.x * per), a1 = min(n, a0 + per);
  double mine = 0.0;
  long long lastpos = -1;
  for (long long i = a0; i < a1; ++i) {
    const double v = __ldcg(vals + i);
    mine += v;
    if (v > 0.0) lastpos = i;
  }
  const double incl = block_incl_scan(mine, sh);
  __shared__ double tot_sh;
  __shared__ long long res_sh;
  if (threadIdx.x == blockDim.x - 1) tot_sh = incl;
  __syncthreads();
  if (total_out) *total_out = tot_sh;
  const int owner = block_first_true(incl > target, shi);
  if (threadIdx.x == 0) res_sh = -1;
  __syncthreads();
  if ((int)threadIdx.x == owner) {
    double acc = incl - mine;
    long long idx = -1;
    for (long long i = a0; i < a1; ++i) {
      acc += __ldcg(vals + i);
      if (acc > target) {
        idx = i;
        break;
      }
    }
    res_sh = idx >= 0 ? idx : lastpos;
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
    }
    __syncthreads();
  }
  const long long r = res_sh;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(512) k_seed_coop(const SeedArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double cs[NYS_MAX_RHO];
  __shared__ double sh[64];
  __shared__ int shi[2];
  __shared__ long long sel[1];
  const int nb = gridDim.x, b = blockIdx.x, rho = a.rho;
  const long long chunk = ceil_div(a.m, (long long)nb);
  const long long lo = min(a.m, b * chunk), hi = min(a.m, lo + chunk);
  for (int j = 1; j < a.m0; ++j) {
    if ((int)threadIdx.x < rho) cs[threadIdx.x] = __ldcg(a.C + (size_t)(j - 1) * rho + threadIdx.x);
    __syncthreads();
    double s = 0.0;
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      const double v = d2_exact(a.pts, a.ps, i, rho, cs);
      const double nv = j == 1 ? v : fmin(a.d2[i], v);
      a.d2[i] = nv;
      s += nv;
    }
    const double bs = block_sum(s, sh);
    if (threadIdx.x == 0) a.ppart[b] = bs;
    grid.sync();
    // every block resolves the owning block redundantly (identical arithmetic)
    double total = 0.0;
    const double u = a.uniforms[j - 1];
    __shared__ double tot_sh;
    {
      // total first, then the target
      const long long per = ceil_div((long long)nb, (long long)blockDim.x);
      const long long a0 = min((long long)nb, (long long)threadIdx.x * per), a1 = min((long long)nb, a0 + per);
      double mine = 0.0;
      for (long long i = a0; i < a1; ++i) mine += __ldcg(a.ppart + i);
      const double incl = block_incl_scan(mine, sh);
      if (threadIdx.x == blockDim.x - 1) tot_sh = incl;
      __syncthreads();
      total = tot_sh;
    }
    if (!(total > 0.0)) {  // sum(D^2) == 0: the reference switches to rng.integers (host redo)
      if (b == 0 && threadIdx.x == 0) a.st->zero_draw = j;
      return;  // uniform across the grid
    }
    const double target = u * total;
    const long long bstar = scan_find(a.ppart, nb, target, sh, shi, nullptr);
    if (b == (int)bstar) {
      // prefix before this block, recomputed with the same run/scan shape
      double before = 0.0;
      {
        const long long per = ceil_div((long long)nb, (long long)blockDim.x);
        const long long a0 = min((long long)nb, (long long)threadIdx.x * per), a1 = min((long long)nb, a0 + per);
        double mine = 0.0;
        for (long long i = a0; i < a1 && i < bstar; ++i) mine += __ldcg(a.ppart + i);
        const double incl = block_incl_scan(mine, sh);
        if (threadIdx.x == blockDim.x - 1) tot_sh = incl;
        __syncthreads();
        before = tot_sh;
      }
      const long long k = scan_find(a.d2 + lo, hi - lo, target - before, sh, shi, nullptr);
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
  double* Cd = wacc + (size_t)nw * slots;               // m0*rho current centroids (FP64)
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
    // slot-parallel cross-block reduction (fixed block order)
    for (long long k = (long long)b * blockDim.x + threadIdx.x; k < S; k += (long long)nb * blockDim.x) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int q = 0;
      for (; q + 4 <= nb; q += 4) {
        s0 += __ldcg(a.part + (size_t)q * S + k);
        s1 += __ldcg(a.part + (size_t)(q + 1) * S + k);
        s2 += __ldcg(a.part + (size_t)(q + 2) * S + k);
        s3 += __ldcg(a.part + (size_t)(q + 3) * S + k);
      }
      for (; q < nb; ++q) s0 += __ldcg(a.part + (size_t)q * S + k);
      a.tot[k] = (s0 + s1) + (s2 + s3);
    }
    grid.sync();
    const double chg = __ldcg(a.tot + slots + 1);
    if (b == 0 && threadIdx.x == 0) {
      a.errors[it] = __ldcg(a.tot + slots);
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
      const double cnt = __ldcg(a.tot + j * (rho + 1) + rho);
      if (cnt > 0.0) Cd[k] = __ldcg(a.tot + j * (rho + 1) + d) / cnt;
    }
    __syncthreads();
    // empty clusters, ascending j: farthest remaining point from its old centroid
    int nex = 0;
    for (int j = 0; j < m0; ++j) {
      if (__ldcg(a.tot + j * (rho + 1) + rho) > 0.0) continue;
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
  int dev = 0, coop = 0, per_sm = 0;
  NYS_CUDA_TRY(cudaGetDevice(&dev));
  NYS_CUDA_TRY(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  if (!coop) return NYS_EUNSUPPORTED;
  NYS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_seed_coop, 512, 0));
  const int nb = (int)std::max<long long>(1, std::min<long long>({(long long)per_sm * sms(), (long long)L.nb_coop,
                                                                   ceil_div(m, 512)}));
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
  count_launch();
  NYS_CUDA_TRY(cudaLaunchCooperativeKernel((void*)k_seed_coop, dim3(nb), dim3(512), args, 0, s));
  return NYS_OK;
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
  while (nw > 1 && (size_t)nw * slots * 8 + fixed > 200 * 1024) --nw;
  const size_t smem = (size_t)nw * slots * 8 + fixed;
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
