// Device helpers shared by the k-means kernels (step-wise and cooperative).
#pragma once

#include <algorithm>
#include <mutex>
#include <vector>

#include "nys_common.cuh"

namespace nys {

struct KState {
  int converged;
  int iters;
  int n_empty;
  int zero_draw;
  long long changed;
  long long repairs;
};

struct KLayout {
  int64_t m;
  int rho, m0, S;  // S: Lloyd slots per block = m0*(rho+1) + 2
  int nb_assign, nb_seed, nb_coop, nb_exact;
  int64_t seed_chunk;
  size_t off_d2, off_labels, off_part, off_ppart, off_tot, off_cf, off_cprev, off_excl, off_state, off_arg,
      off_idx, off_unif, off_pp, off_tsum, total;
  int64_t m_pad;  // m + 512 * nb_coop: slots of the thread-run-permuted seeding copy
};

inline int sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline KLayout klayout(int64_t m, int rho, int m0) {
  KLayout L;
  L.m = m;
  L.rho = rho;
  L.m0 = m0;
  L.S = m0 * (rho + 1) + 2;
  L.nb_assign = (int)std::max<int64_t>(1, std::min<int64_t>(2 * 148, ceil_div(m, 256)));
  L.nb_exact = (int)std::max<int64_t>(1, std::min<int64_t>(8 * 148, ceil_div(m, 256)));  // cap; the launch sizes by occupancy
  L.nb_seed = (int)std::max<int64_t>(1, std::min<int64_t>(4 * 148, ceil_div(m, 1024)));
  L.seed_chunk = ceil_div(m, L.nb_seed);
  L.nb_coop = 4 * sms();  // upper bound on co-resident blocks of the cooperative kernels
  size_t o = 0;
  L.m_pad = m + (int64_t)512 * L.nb_coop;
  L.off_d2 = o;      o = align256(o + (size_t)L.m_pad * 8);
  L.off_labels = o;  o = align256(o + (size_t)m * 4);
  // ppart before anything that depends on (rho, m0): the step-wise
  // nys_kmeanspp_update / _pick pair must agree on it for any (rho, m0)
  L.off_ppart = o;   o = align256(o + (size_t)std::max(L.nb_seed, L.nb_coop) * 8);
  L.off_part = o;    o = align256(o + (size_t)std::max(L.nb_assign, L.nb_coop) * L.S * 8);
  L.off_tot = o;     o = align256(o + (size_t)std::max(L.S, 3 * (m0 * rho + m0)) * 8);
  L.off_cf = o;      o = align256(o + (size_t)m0 * rho * 4);
  L.off_cprev = o;   o = align256(o + (size_t)m0 * rho * 8);
  L.off_excl = o;    o = align256(o + (size_t)m0 * 8);
  L.off_state = o;   o = align256(o + sizeof(KState));
  L.off_arg = o;     o = align256(o + (size_t)std::max({L.nb_assign, L.nb_seed, L.nb_coop, L.nb_exact}) * 32);
  L.off_idx = o;     o = align256(o + 64);
  L.off_unif = o;    o = align256(o + (size_t)m0 * 8);
  L.off_tsum = o;    o = align256(o + (size_t)L.nb_coop * 512 * 8);
  L.off_pp = o;      o = align256(o + (rho <= NYS_MAX_RHO ? (size_t)L.m_pad * rho * 4 : 0));  // coop seeding only
  L.total = o;
  return L;
}

// owner flag of the cooperative seeding (zeroed by k_seed_prologue)
inline int* seed_flag(char* ws, const KLayout& L) { return reinterpret_cast<int*>(ws + L.off_idx + 32); }

// cached per process: these queries sat on the host path before the first seeding draw
inline bool coop_supported() {
  static int cached = -1;
  if (cached < 0) {
    int dev = 0, coop = 0;
    cached = (cudaGetDevice(&dev) == cudaSuccess &&
              cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev) == cudaSuccess && coop)
                 ? 1
                 : 0;
  }
  return cached == 1;
}

// raises the kernel's dynamic shared-memory limit and returns its resident blocks per SM,
// once per (kernel, threads, smem)
inline cudaError_t coop_blocks_per_sm(const void* kern, int threads, size_t smem, int* per_sm) {
  struct Entry {
    const void* k;
    int dev;
    int threads;
    size_t smem;
    int per_sm;
  };
  static std::mutex mu;
  static std::vector<Entry> cache;
  struct Limit {
    const void* k;
    int dev;
    size_t bytes;  // the kernel's raised limit only ever grows
  };
  static std::vector<Limit> limit;
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  std::lock_guard<std::mutex> g(mu);
  for (const Entry& e : cache)
    if (e.k == kern && e.dev == dev && e.threads == threads && e.smem == smem) {
      *per_sm = e.per_sm;
      return cudaSuccess;
    }
  size_t* cur = nullptr;
  for (auto& l : limit)
    if (l.k == kern && l.dev == dev) cur = &l.bytes;
  if (!cur) {
    limit.push_back(Limit{kern, dev, 0});
    cur = &limit.back().bytes;
  }
  if (std::max<size_t>(smem, 1) > *cur) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smem, 1));
    if (err != cudaSuccess) return err;
    *cur = std::max<size_t>(smem, 1);
  }
  err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kern, threads, smem);
  if (err != cudaSuccess) return err;
  cache.push_back(Entry{kern, dev, threads, smem, *per_sm});
  return cudaSuccess;
}

// numpy's row reduction order for ((x - c)**2).sum(axis=1) over rho entries
// (pairwise_sum: sequential from 0 below 8 terms, else 8 strided partials
// combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a sequential tail).
// __dmul_rn/__dadd_rn forbid FMA contraction, so every D^2 value is
// bit-identical to the reference's (landmarks.py:64,72).
__device__ __forceinline__ double sqdiff(double x, double c) {
  const double t = __dsub_rn(x, c);
  return __dmul_rn(t, t);
}

// numpy's pairwise summation above its 128-element block (rho > 128): the two halves (the
// first rounded down to a multiple of 8) summed recursively, then added
static __device__ double d2_exact_pw(const float* __restrict__ pts, long long ps, long long i, int rho,
                              const double* __restrict__ c);

__device__ __forceinline__ double d2_exact(const float* __restrict__ pts, long long ps, long long i, int rho,
                           const double* __restrict__ c) {
  if (rho > 128) return d2_exact_pw(pts, ps, i, rho, c);
  if (rho < 8) {
    double r = 0.0;
    for (int d = 0; d < rho; ++d) r = __dadd_rn(r, sqdiff((double)__ldg(pts + d * ps + i), c[d]));
    return r;
  }
  double r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = sqdiff((double)__ldg(pts + k * ps + i), c[k]);
  int d = 8;
  const int full = rho - (rho % 8);
  for (; d < full; d += 8) {
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], sqdiff((double)__ldg(pts + (d + k) * ps + i), c[d + k]));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; d < rho; ++d) res = __dadd_rn(res, sqdiff((double)__ldg(pts + d * ps + i), c[d]));
  return res;
}

static __device__ __noinline__ double d2_exact_pw(const float* __restrict__ pts, long long ps, long long i, int rho,
                                           const double* __restrict__ c) {
  int n2 = rho / 2;
  n2 -= n2 % 8;
  const double a = d2_exact(pts, ps, i, n2, c);
  const double b = d2_exact(pts + (long long)n2 * ps, ps, i, rho - n2, c + n2);
  return __dadd_rn(a, b);
}

// exact FP64 |x - c|^2 in numpy's pairwise order for a compile-time bound GR >= rho
template <int GR>
__device__ __forceinline__ double d2_exact_regs(const float (&x)[GR], int rho, const double* __restrict__ c) {
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

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// fixed-shape block sum (blockDim multiple of 32, <= 1024)
__device__ __forceinline__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < nw; ++k) r += sh[k];
  return r;  // valid in thread 0
}


// fixed-shape block inclusive scan (blockDim multiple of 32, <= 1024); sh >= 32 doubles
__device__ __forceinline__ double block_incl_scan(double v, double* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  __syncthreads();
  if (lane == 31) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    double s = lane < nw ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double t = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += t;
    }
    sh[lane] = s;
  }
  __syncthreads();
  if (w > 0) v += sh[w - 1];
  return v;
}

// first thread (lowest index) whose predicate holds, or blockDim.x; shi >= 1 int
__device__ __forceinline__ int block_first_true(bool p, int* shi) {
  if (threadIdx.x == 0) *shi = (int)blockDim.x;
  __syncthreads();
  const unsigned b = __ballot_sync(0xffffffffu, p);
  if ((threadIdx.x & 31) == 0 && b) atomicMin(shi, (int)((threadIdx.x & ~31) + __ffs(b) - 1));
  __syncthreads();
  const int r = *shi;
  __syncthreads();
  return r;
}

// Warp-level deterministic accumulation of per-cluster coordinate sums and
// counts: each distinct label among the valid lanes is reduced with a fixed
// butterfly over zero-masked values; lane 0 adds the group sum into `acc`
// (this warp's private [m0][rho+1] FP64 accumulators).
template <int GR>
__device__ __forceinline__ void warp_accumulate(const float (&x)[GR], int rho, int label, bool valid, double* acc) {
  const int lane = threadIdx.x & 31;
  unsigned rem = __ballot_sync(0xffffffffu, valid);
  while (rem) {
    const int leader = __ffs(rem) - 1;
    const int L = __shfl_sync(0xffffffffu, label, leader);
    const unsigned grp = __ballot_sync(0xffffffffu, valid && label == L);
    const bool in = (grp >> lane) & 1u;
#pragma unroll
    for (int d = 0; d < GR; ++d)
      if (d < rho) {
        const double s = warp_sum(in ? (double)x[d] : 0.0);
        if (lane == 0) acc[L * (rho + 1) + d] += s;
      }
    if (lane == 0) acc[L * (rho + 1) + rho] += (double)__popc(grp);
    rem &= ~grp;
  }
}

int launch_seed_coop(const float* pts, long long ps, long long m, int rho, int m0, const double* uniforms_dev,
                     double* C, long long* seeds, char* ws, const KLayout& L, cudaStream_t s);
int launch_lloyd_coop(const float* pts, long long ps, long long m, int rho, int m0, int max_iter, double* C,
                      double* errors, char* ws, const KLayout& L, cudaStream_t s, bool prezeroed = false);

// Warp-level accumulation of per-cluster coordinate sums as EXACT fixed-point
// integers (x * 2^s rounded once per point, two's complement): each distinct
// label among the lanes is reduced with REDUX on 21-bit limbs, so sums are
// independent of order and hence deterministic across blocks, warps and runs.
// `sign` = -1 removes the lanes' points from their clusters.
template <int GR>
__device__ __forceinline__ void warp_accumulate_fx(const float (&x)[GR], int rho, int label, bool valid, double scale,
                                                   int sign, unsigned long long* acc, int* cnt) {
  const int lane = threadIdx.x & 31;
  unsigned rem = __ballot_sync(0xffffffffu, valid);
  while (rem) {
    const int leader = __ffs(rem) - 1;
    const int L = __shfl_sync(0xffffffffu, label, leader);
    const unsigned grp = __ballot_sync(0xffffffffu, valid && label == L);
    if ((grp >> lane) & 1u) {
#pragma unroll
      for (int d = 0; d < GR; ++d)
        if (d < rho) {
          const unsigned long long v = (unsigned long long)__double2ll_rn((double)(sign * x[d]) * scale);
          const unsigned long long s0 = __reduce_add_sync(grp, (unsigned)(v & 0x1FFFFFull));
          const unsigned long long s1 = __reduce_add_sync(grp, (unsigned)((v >> 21) & 0x1FFFFFull));
          const unsigned long long s2 = __reduce_add_sync(grp, (unsigned)(v >> 42));
          if (lane == leader) acc[L * rho + d] += s0 + (s1 << 21) + (s2 << 42);
        }
      if (lane == leader) cnt[L] += sign * __popc(grp);
    }
    rem &= ~grp;
  }
}

}  // namespace nys
