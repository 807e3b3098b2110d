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

#include <type_traits>
#include <cstdlib>

#include "nys_kmeans_dev.cuh"
#include "nys_umma.cuh"

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
  int* flag;  // last published draw (owner block -> everyone)
  // thread-run seeding (k_seed_runs)
  float* pp;        // permuted copy: plane d, slot (block, r, t) at pp[d * pps + (block * per + r) * B + t]
  long long pps;    // plane stride of pp
  double* tsum;     // per-thread run sums [block][B]
  int per;          // points per thread run
  int mode;         // 0: every block resolves the draw (remote run sums, recomputed run; NYS_SEED_MODE=0, A/B);
                    // 1: the owning block resolves it from its own run sums and D^2 and publishes the point
};

// Cross-block words exchanged by polling (k_seed_runs mode 1): a slot holds this bit pattern (a NaN
// no arithmetic produces) until its value is published; published NaNs are canonicalised.
// (Exchanging the block totals the same way instead of a grid barrier -- three rounds of polled
// slots -- measured slower: 1.35 -> 1.52 ms k-means on cfg 2; grid.sync is the cheaper all-to-all.)
constexpr unsigned long long SEED_EMPTY = 0xFFFFFFFFFFFFFFFFull;
__device__ __forceinline__ void seed_publish(double* slot, double v) {
  unsigned long long bits = (unsigned long long)__double_as_longlong(v);
  if (v != v) bits = 0x7FF8000000000000ull;
  __stcg(reinterpret_cast<unsigned long long*>(slot), bits);
}
__device__ __forceinline__ double seed_poll(const double* slot) {
  unsigned long long bits = __ldcg(reinterpret_cast<const unsigned long long*>(slot));
  long long spins = 0;
  while (bits == SEED_EMPTY) {
    if (++spins > (1ll << 22)) __trap();  // seconds: a protocol error must fail loudly, not hang the GPU
    bits = __ldcg(reinterpret_cast<const unsigned long long*>(slot));
  }
  return __longlong_as_double((long long)bits);
}

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

template <int GR, int RX>
__global__ void __launch_bounds__(512) k_seed_coop(const SeedArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double d2s[];  // this block's chunk of D^2 when it fits
  __shared__ double cs[NYS_MAX_RHO];
  __shared__ double sh[64];
  __shared__ int shi[2];
  __shared__ long long sel[1];
  __shared__ double tot_sh;
  const int nb = gridDim.x, b = blockIdx.x, rho = RX > 0 ? RX : a.rho;  // RX: compile-time rho
  const long long chunk = ceil_div(a.m, (long long)nb);
  const long long lo = min(a.m, b * chunk), hi = min(a.m, lo + chunk);
  const int len = (int)(hi - lo);
  double* d2 = a.d2_in_smem ? d2s : a.d2 + lo;
  const int B = blockDim.x;
  for (int j = 1; j < a.m0; ++j) {
    if ((int)threadIdx.x < rho) cs[threadIdx.x] = __ldcg(a.C + (size_t)(j - 1) * rho + threadIdx.x);
    __syncthreads();
    double s = 0.0;
    constexpr int U = GR <= 4 ? 7 : 2;  // independent points in flight (register budget; 28 = 4 x 7 on cfg 2; 14 measured no faster)
    int i = threadIdx.x;
    for (; i + (U - 1) * B < len; i += U * B) {
      float x[U][GR];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int d = 0; d < GR; ++d) x[u][d] = d < rho ? __ldg(a.pts + d * a.ps + lo + i + u * B) : 0.f;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double v = d2_exact_regs<GR>(x[u], rho, cs);
        const double nv = j == 1 ? v : fmin(d2[i + u * B], v);
        d2[i + u * B] = nv;
        s += nv;
      }
    }
    for (; i < len; i += B) {
      float x[GR];
#pragma unroll
      for (int d = 0; d < GR; ++d) x[d] = d < rho ? __ldg(a.pts + d * a.ps + lo + i) : 0.f;
      const double v = d2_exact_regs<GR>(x, rho, cs);
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
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicExch(a.flag, j);  // publish centroid j (cheaper than a second grid barrier)
      }
    }
    if (threadIdx.x == 0) {
      while (atomicAdd(a.flag, 0) < j) __nanosleep(32);
      __threadfence();
    }
    __syncthreads();
  }
}

// One value per thread (the first n threads; the rest pass 0): inclusive
// block scan, target = tfn(total), then the first thread whose inclusive
// prefix exceeds target -- or, when rounding left none, the last thread with a
// positive value.  Returns that thread; *before = the sum of the values before
// it, *total_out = the total.  Six block barriers.
template <class TF>
__device__ __forceinline__ int scan_pick(double v, TF tfn, double* sh, int* shi, double* before, double* total_out) {
  __shared__ double tot_s, bef_s;
  const double incl = block_incl_scan(v, sh);
  if (threadIdx.x == blockDim.x - 1) tot_s = incl;
  if (threadIdx.x == 0) {
    shi[0] = (int)blockDim.x;
    shi[1] = -1;
  }
  __syncthreads();
  const double total = tot_s, target = tfn(total);
  const unsigned bp = __ballot_sync(0xffffffffu, incl > target), bv = __ballot_sync(0xffffffffu, v > 0.0);
  if ((threadIdx.x & 31) == 0) {
    if (bp) atomicMin(&shi[0], (int)(threadIdx.x + __ffs(bp) - 1));
    if (bv) atomicMax(&shi[1], (int)(threadIdx.x + 31 - __clz(bv)));
  }
  __syncthreads();
  const int owner = shi[0] < (int)blockDim.x ? shi[0] : max(shi[1], 0);
  if ((int)threadIdx.x == owner) bef_s = incl - v;
  __syncthreads();
  *before = bef_s;
  if (total_out) *total_out = total;
  return owner;
}

// k-means++ seeding with ONE grid barrier per draw (landmarks.py:60-73).
// Thread t of block b owns the contiguous run of points lo_b + t*per + r,
// r < per (a permuted copy of the guide keeps the per-r loads coalesced), so
// the global linear order is (block, thread, r).  After the D^2 update every
// block publishes its per-thread run sums and their block total; after the
// barrier every block resolves the draw redundantly with identical
// arithmetic: the owning block (scan over block totals), the owning thread
// (scan over that block's run sums), then the point inside the run, whose
// D^2 values it recomputes exactly (min over the centroids so far, the same
// FP64 formula, so bit-identical to the stored ones).  No owner handoff.
template <int GR, int RX>
__global__ void __launch_bounds__(512) k_seed_runs(const SeedArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double d2s[];  // this block's D^2 (slot order r*B + t) when it fits
  __shared__ double sh[64];
  __shared__ int shi[2];
  const int nb = gridDim.x, b = blockIdx.x, rho = RX > 0 ? RX : a.rho;  // RX: compile-time rho
  const int B = blockDim.x, t = threadIdx.x, lane = t & 31, wid = t >> 5, nwarp = B >> 5;
  const long long chunk = ceil_div(a.m, (long long)nb);
  const long long lo = min(a.m, b * chunk), hi = min(a.m, lo + chunk);
  const int len = (int)(hi - lo), per = a.per;
  const long long slot0 = (long long)b * per * B;
  double* d2 = a.d2_in_smem ? d2s : a.d2 + slot0;
  double* Cs = a.d2_in_smem ? d2s + (size_t)per * B : d2s;  // [m0][rho] centroid history
  double* rd2 = Cs + (size_t)a.m0 * rho;                      // [per] D^2 of the owning run
  // permuted copy of this block's points (read back only by the thread that wrote each slot)
  for (int r = 0; r < per; ++r) {
    const int li = t * per + r;
#pragma unroll 4
    for (int d = 0; d < rho; ++d)
      a.pp[d * a.pps + slot0 + (long long)r * B + t] = li < len ? __ldg(a.pts + d * a.ps + lo + li) : 0.f;
  }
  for (int k = t; k < rho; k += B) Cs[k] = __ldcg(a.C + k);
  if (a.mode) {  // polled slots start empty: the centroid rows 1..
    if (b == 0)
      for (int k = rho + t; k < a.m0 * rho; k += B)
        __stcg(reinterpret_cast<unsigned long long*>(a.C + k), SEED_EMPTY);
    grid.sync();
  }
  __syncthreads();
  for (int j = 1; j < a.m0; ++j) {
    const double* cs = Cs + (size_t)(j - 1) * rho;
    double s = 0.0;
    constexpr int U = GR <= 4 ? 7 : 2;  // independent points in flight (register budget; 28 = 4 x 7 on cfg 2; 14 measured no faster)
    // Wide guides: every draw streams the whole permuted guide (113 MB on cfg 3, just above what the
    // 126 MB L2 keeps), so with a fixed sweep direction every line has been evicted by the time it
    // is needed again.  Odd draws sweep the runs backwards: the lines touched last are touched
    // first, and most of the guide is served from the L2.  The run sum is still accumulated in
    // ascending order (a second pass over the stored D^2), so it has the bits of the forward sweep.
    const bool rev = GR >= 16 && (j & 1) && a.d2_in_smem;
    auto RR = [&](int q) { return rev ? per - 1 - q : q; };
    int r = 0;
    for (; r + U <= per; r += U) {
      float x[U][GR];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int d = 0; d < GR; ++d) x[u][d] = d < rho ? a.pp[d * a.pps + slot0 + (long long)RR(r + u) * B + t] : 0.f;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double v = d2_exact_regs<GR>(x[u], rho, cs);
        const int sl = RR(r + u) * B + t;
        double nv = j == 1 ? v : fmin(d2[sl], v);
        if (t * per + RR(r + u) >= len) nv = 0.0;
        d2[sl] = nv;
        s += nv;  // run sum in linear order (forward sweeps)
      }
    }
    for (; r < per; ++r) {
      float x[GR];
#pragma unroll
      for (int d = 0; d < GR; ++d) x[d] = d < rho ? a.pp[d * a.pps + slot0 + (long long)RR(r) * B + t] : 0.f;
      const double v = d2_exact_regs<GR>(x, rho, cs);
      const int sl = RR(r) * B + t;
      double nv = j == 1 ? v : fmin(d2[sl], v);
      if (t * per + RR(r) >= len) nv = 0.0;
      d2[sl] = nv;
      s += nv;
    }
    if (rev) {
      s = 0.0;
      for (int q = 0; q < per; ++q) s += d2[q * B + t];
    }
    if (a.mode == 0) a.tsum[(long long)b * B + t] = s;
    {
      const double incl = block_incl_scan(s, sh);  // the scan scan_pick runs over the run sums
      if (t == B - 1) a.ppart[b] = incl;
    }
    grid.sync();
    // --- the owning block (nb <= blockDim: one block total per thread), identical in every block ---
    double total = 0.0, before_b = 0.0, before_t = 0.0, before_r = 0.0;
    const double u = a.uniforms[j - 1];
    const int bstar = scan_pick(t < nb ? __ldcg(a.ppart + t) : 0.0, [&](double tot) { return u * tot; }, sh, shi,
                                &before_b, &total);
    if (!(total > 0.0)) {  // sum(D^2) == 0: the reference switches to rng.integers (host redo)
      if (b == 0 && t == 0) a.st->zero_draw = j;
      return;  // uniform across the grid
    }
    const double target = u * total, tgt_b = target - before_b;
    if (a.mode) {
      // The owning block resolves the thread run and the point from its own run sums (registers) and
      // stored D^2 (the values the other path recomputes), and publishes the point's coordinates;
      // everyone else polls them: one L2 round trip instead of two plus the recomputation.
      double* cn = Cs + (size_t)j * rho;
      if (b == bstar) {
        const int tstar = scan_pick(s, [&](double) { return tgt_b; }, sh, shi, &before_t, nullptr);
        const double tgt = tgt_b - before_t;
        long long idx = -1;
        for (int r0 = 0; r0 < per && idx < 0; r0 += B) {
          const int cnt = min(B, per - r0);
          double run_tot = 0.0, before_in = 0.0;
          const int rstar = scan_pick(t < cnt ? d2[(size_t)(r0 + t) * B + tstar] : 0.0,
                                      [&](double) { return tgt - before_r; }, sh, shi, &before_in, &run_tot);
          if (r0 + cnt >= per || run_tot > tgt - before_r)
            idx = lo + (long long)tstar * per + r0 + rstar;
          else
            before_r += run_tot;  // the target lies in a later round of this run
        }
        for (int k = t; k < rho; k += B) {
          const double v = (double)__ldg(a.pts + k * a.ps + idx);
          cn[k] = v;
          seed_publish(a.C + (size_t)j * rho + k, v);
        }
        if (t == 0 && a.seeds) a.seeds[j] = idx;
      } else {
        for (int k = t; k < rho; k += B) cn[k] = seed_poll(a.C + (size_t)j * rho + k);
      }
      __syncthreads();
      continue;
    }
    // the owning thread run inside block bstar
    const int tstar = scan_pick(__ldcg(a.tsum + (long long)bstar * B + t), [&](double) { return tgt_b; }, sh, shi,
                                &before_t, nullptr);
    // the point inside the run: its D^2 recomputed exactly (warp per point, lanes over the centroids so far)
    const long long lo_s = min(a.m, (long long)bstar * chunk), len_s = min(a.m, lo_s + chunk) - lo_s;
    const double tgt = tgt_b - before_t;
    long long idx = -1;
    for (int r0 = 0; r0 < per && idx < 0; r0 += 512) {
      const int cnt = min(512, per - r0);
      for (int rr = wid; rr < cnt; rr += nwarp) {
        const long long li = (long long)tstar * per + r0 + rr;
        double mn = 0.0;
        if (li < len_s) {
          float x[GR];
#pragma unroll
          for (int d = 0; d < GR; ++d) x[d] = d < rho ? __ldg(a.pts + d * a.ps + lo_s + li) : 0.f;
          mn = INFINITY;
          for (int k = lane; k < j; k += 32) mn = fmin(mn, d2_exact_regs<GR>(x, rho, Cs + (size_t)k * rho));
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        }
        if (lane == 0) rd2[r0 + rr] = mn;
      }
      __syncthreads();
      double run_tot = 0.0, before_in = 0.0;
      const int rstar = scan_pick(t < cnt ? rd2[r0 + t] : 0.0, [&](double) { return tgt - before_r; }, sh, shi,
                                  &before_in, &run_tot);
      if (r0 + cnt >= per || run_tot > tgt - before_r)
        idx = lo_s + (long long)tstar * per + r0 + rstar;
      else
        before_r += run_tot;  // the target lies in a later round of this run
    }
    double* cn = Cs + (size_t)j * rho;
    for (int k = t; k < rho; k += B) cn[k] = (double)__ldg(a.pts + k * a.ps + idx);
    if (b == 0) {
      for (int k = t; k < rho; k += B) a.C[(size_t)j * rho + k] = (double)__ldg(a.pts + k * a.ps + idx);
      if (t == 0 && a.seeds) a.seeds[j] = idx;
    }
    __syncthreads();
  }
}

struct LloydArgs {
  const float* pts;
  long long ps, m;
  int rho, m0, max_iter, S;
  double* C;                 // in: seeds; out: final centroids
  int* labels;
  unsigned long long* gacc;  // 3 x (m0*rho sums + m0 counts): per-iteration exact fixed-point deltas
  double* part;              // 2 x nb x 2 (objective, changed) per block, parity-buffered
  double* arg;               // 2 x nb x 2 (double-buffered argmax pairs)
  double* errors;
  KState* st;
  unsigned* maxabs_bits;     // global max |x| (float bits), zeroed by k_init_state
  float* lb;                 // m: lower bound on the distance to the second-closest centroid (+ drift)
  int* list;                 // m: per-warp lists of points that need the full search
  int nw;                    // warps per block
  int bounds;                // 0: full search every iteration (debug / A-B check)
  // (the cell-pruned kernel keeps its KM_NG^rho candidate masks where the bounds would be, at
  // `lb`; the struct's size is left alone: two more members changed the register allocation of
  // the wide-guide instantiations from 255 to 167-207 and cost cfg 4 1.5 ms)
};

// Cell-pruned exact assignment for guides of up to three dimensions (colour images).
// The bounding box of the points is cut into KM_NG^rho cells.  After every centroid update
// the blocks rebuild, one warp per cell, the set of centroids that can be nearest to *some*
// point of the cell: with U = min_c maxdist^2(c, cell), centroid c is a candidate iff
// mindist^2(c, cell) <= U (1 + 1e-4).  A non-candidate is farther from every point of the
// cell than the best candidate by a relative 1e-4, far above the 3e-7 rounding of the FP32
// differenced distance, so searching only the candidates (ascending index, strict <) returns
// the label, distance and tie-break of the full m0-way search; cells are grown by 1e-3 of
// their width against the rounding of the point-to-cell map.  A point then evaluates a
// handful of centroids instead of m0, every iteration, with no per-point bound state.
constexpr int KM_NG = 16;
__device__ __forceinline__ unsigned f32_ordered(float v) {  // order-preserving, > 0 for finite v
  const unsigned u = __float_as_uint(v);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float f32_unordered(unsigned e) {
  return __uint_as_float((e & 0x80000000u) ? (e & 0x7fffffffu) : ~e);
}

// squared FP32 distance, difference form, dimensions in ascending order -- the
// one formula every assignment uses, so a bound-skipped point gets the same
// value the full search would have produced
template <int GR>
__device__ __forceinline__ float d2_f32(const float (&x)[GR], int rho, const float* __restrict__ c) {
  float d2 = 0.f;
#pragma unroll
  for (int d4 = 0; d4 < (GR + 3) / 4; ++d4) {
    if (4 * d4 < rho) {
      const float4 c4 = reinterpret_cast<const float4*>(c)[d4];
      const float cc[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (4 * d4 + e < GR && 4 * d4 + e < rho) {
          const float t = x[4 * d4 + e] - cc[e];
          d2 = fmaf(t, t, d2);
        }
    }
  }
  return d2;
}

// Lloyd iterations with Hamerly-style bounds.  A point keeps its label without
// the m0-way search when its FP32 distance to the assigned centroid is below a
// lower bound on its distance to every other centroid, with a relative margin
// (LB_EPS) that covers the FP32 rounding of both sides: then the full search
// would return the same label with the same distance, so labels, exact sums,
// centroids and iteration counts are identical to searching every point.
// The bound is stored drift-adjusted (lb + cumulative max centroid movement at
// the time it was set), so skipped points cost no writes.  Per-iteration sums
// are exact fixed-point deltas of the points whose label changed.
constexpr double LB_EPS = 1.0 / 32768.0;

// GRID: the cell-pruned search (a separate instantiation, so the bounds kernels compile as before)
//
// TC (wide guides, north_star (1)): the m0-way search of every point runs on the 5th-generation
// tensor cores, every iteration, with no per-point bound state.  A group of four warps takes
// 128 points (TMEM lanes); each thread splits its point x = x_hi + x_lo into TF32 pairs and
// stores (x, 1) as the A operand in TMEM; one thread issues 3 x K/8 tcgen05.mma kind::tf32
// against B = (-2 c_j, |c_j|^2) (centroids in shared memory, K-major, hi/lo split, rebuilt after
// every update), so D_j = |c_j|^2 - 2 x.c_j = approx_j - |x|^2 accumulates in TMEM.  The thread
// drains its row, takes the minimum, and re-checks every centroid within 2 delta of it with the
// exact FP32 difference form (ascending j, strict <): delta = 1e-4 (|x|^2 + max|c|^2) bounds the
// 3xTF32 / FP32-norm error with a wide margin, so labels, distances and tie-breaks equal the FP32
// search's (test_lloyd_bounds_are_exact, NYS_KM_NOBOUNDS A/B).  Two groups per CTA, each with its
// own TMEM columns and mbarrier, overlap one group's MMAs with the other's re-check.  Label
// changes feed the same exact fixed-point delta sums as the bounds kernel.
template <int GR, int RX, bool GRID = false, bool TC = false>
__global__ void __launch_bounds__(256) k_lloyd_coop(const LloydArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double dsm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int rho = RX > 0 ? RX : a.rho, m0 = a.m0, msl = m0 * rho, gstride = msl + m0;  // RX: compile-time rho
  unsigned long long* wacc = reinterpret_cast<unsigned long long*>(dsm);      // nw x msl (per-warp sums)
  int* wcnt = reinterpret_cast<int*>(wacc + (size_t)nw * msl);                 // nw x m0 (per-warp counts)
  double* Cd = reinterpret_cast<double*>(wcnt + (((size_t)nw * m0 + 1) & ~size_t(1)));  // m0*rho current (FP64)
  double* Cp = Cd + (size_t)msl;                                               // m0*rho previous
  long long* T = reinterpret_cast<long long*>(Cp + (size_t)msl);              // msl sums + m0 counts (exact)
  long long* excl = T + gstride;                                               // m0
  float* Cf = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(excl + m0) + 15) & ~uintptr_t(15));
  const int rhop = (rho + 3) & ~3;                                             // Cf rows: 16-byte aligned
  const int m0p = (m0 + 3) & ~3;                                               // Cf rows padded to 4
  float* Cfo = Cf + (size_t)m0p * rhop;                                        // previous iteration's Cf
  constexpr bool GRIDOK = GRID;
  constexpr bool gridmode = GRID;
  static_assert(!GRID || (RX >= 1 && RX <= 3), "cell-pruned search: rho <= 3");
  constexpr int NCELL_ALL = RX == 1 ? KM_NG : (RX == 2 ? KM_NG * KM_NG : KM_NG * KM_NG * KM_NG);
  unsigned long long* gts = reinterpret_cast<unsigned long long*>(                // candidate masks (grid mode)
      (reinterpret_cast<uintptr_t>(Cfo + (size_t)m0p * rhop) + 15) & ~uintptr_t(15));
  double* gh = reinterpret_cast<double*>(gts + (GRID ? NCELL_ALL : 0));            // 3 cell widths
  float* glo = reinterpret_cast<float*>(gh + 3);                                   // 3 box origins
  float* ginv = glo + 3;                                                           // 3 inverse cell widths
  int* wlim = reinterpret_cast<int*>(ginv + 3 + 1);                                // nw x msl x 3 signed 21-bit limbs (grid mode)
  // TC: B operand (NU x KU, K-major core matrices, hi / lo) and this CTA's TMEM / mbarriers
  const int KU = TC ? ((rho + 1 + 7) / 8) * 8 : 0, NU = TC ? ((m0 + 15) / 16) * 16 : 0;
  float* Bh = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(Cfo + (size_t)m0p * rhop) + 127) & ~uintptr_t(127));
  float* Bl = Bh + (size_t)NU * KU;
  __shared__ uint64_t tc_bar[2];
  __shared__ uint32_t tc_tmem;
  __shared__ float tc_ccmax;
  const int tcols = ((NU + 31) & ~31) + 2 * ((KU + 31) & ~31);  // per group: D, A_hi, A_lo
  int tc_alloc = 32;
  if constexpr (TC) {
    // the whole tensor memory of the SM (one CTA per SM: 255 registers): the base is then column 0 by
    // construction, so the MMA operands below are kernel-parameter arithmetic in uniform registers
    // (addresses derived from the allocation word in shared memory cost a register-to-uniform move per
    // operand per MMA: ~125 cycles per instruction, measured)
    tc_alloc = 512;
    if (w == 0) umma::tmem_alloc(&tc_tmem, (uint32_t)tc_alloc);
    if (threadIdx.x < 2) {
      umma::mbar_init(&tc_bar[threadIdx.x], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
  }
  uint32_t tc_phase = 0;
  __shared__ double sh[64];
  __shared__ double extra[2][32];
  __shared__ double misc[2];
  __shared__ int wlen[32], wpre[33];
  __shared__ double dcum_sh;
  const int nb = gridDim.x, b = blockIdx.x;
  const long long chunk = ceil_div(a.m, (long long)nb);
  const long long clo = min(a.m, b * chunk), chi = min(a.m, clo + chunk);  // contiguous chunk: sweeps, repair
  // Assignment partition of the bounds kernel: block b owns the KM_SEG-point segments b, b + nb,
  // b + 2 nb, ... of the image (a uniform sample of it: bound failures and label changes cluster
  // in busy regions, and contiguous chunks left the grid barrier waiting for the blocks that own
  // them).  A block walks its segments as one contiguous *virtual* range [lo, hi); gmap turns a
  // virtual index into the point index (>= m: padding).  Lists, bounds and labels are indexed by
  // point, the list segments by virtual position.
  constexpr long long KM_SEG = 256;
  const long long chunk_v = ceil_div(chunk, KM_SEG) * KM_SEG;
  const long long lo = (long long)b * chunk_v, hi = lo + chunk_v;
  auto gmap = [&](long long v) { return (((v - lo) / KM_SEG) * nb + b) * KM_SEG + ((v - lo) % KM_SEG); };
  const long long cw = ceil_div(ceil_div(hi - lo, (long long)nw), 128ll) * 128;  // phase-A sub-range per warp
  const long long wlo = min(hi, lo + w * cw), whi = min(hi, wlo + cw);

  // fixed-point scale 2^s with |sum| < 2^61 for any cluster: s = 61 - log2(max|x| * m)
  {
    float mx = 0.f;
    if (a.ps == a.m && (reinterpret_cast<uintptr_t>(a.pts) & 15) == 0 && (a.m & 3) == 0) {
      // contiguous planes: one flat float4 sweep over rho*m values
      const long long n4 = (long long)rho * a.m / 4;
      const float4* p4 = reinterpret_cast<const float4*>(a.pts);
      for (long long q = (long long)b * blockDim.x + threadIdx.x; q < n4; q += (long long)nb * blockDim.x) {
        const float4 v = __ldg(p4 + q);
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
      }
    } else {
      for (long long i = clo + threadIdx.x; i < chi; i += blockDim.x)
        for (int d = 0; d < rho; ++d) mx = fmaxf(mx, fabsf(__ldg(a.pts + d * a.ps + i)));
    }
    mx = warp_max(mx);
    if (lane == 0 && mx > 0.f) atomicMax(a.maxabs_bits, __float_as_uint(mx));
    if constexpr (gridmode) {  // per-dimension bounding box: words 1..3 max, 4..6 -min (order-preserving, zero = identity)
      for (int d = 0; d < rho; ++d) {
        float hi_v = -INFINITY, lo_v = INFINITY;
        for (long long i = clo + threadIdx.x; i < chi; i += blockDim.x) {
          const float v = __ldg(a.pts + d * a.ps + i);
          hi_v = fmaxf(hi_v, v);
          lo_v = fminf(lo_v, v);
        }
        hi_v = warp_max(hi_v);
        lo_v = -warp_max(-lo_v);
        if (lane == 0 && hi_v >= lo_v) {
          atomicMax(a.maxabs_bits + 1 + d, f32_ordered(hi_v));
          atomicMax(a.maxabs_bits + 4 + d, f32_ordered(-lo_v));
        }
      }
    }
  }
  for (int k = threadIdx.x; k < msl; k += blockDim.x) Cd[k] = __ldcg(a.C + k);
  for (int k = threadIdx.x; k < gstride; k += blockDim.x) T[k] = 0;
  if (threadIdx.x == 0) dcum_sh = 0.0;
  __syncthreads();
  for (int k = threadIdx.x; k < m0p * rhop; k += blockDim.x) {
    const int j = k / rhop, d = k - j * rhop;
    Cf[k] = j >= m0 ? 3.0e38f : (d < rho ? (float)Cd[j * rho + d] : 0.f);  // padded rows never win
  }
  grid.sync();
  const float maxabs = __uint_as_float(__ldcg(a.maxabs_bits));
  int sexp = 0;
  if (maxabs > 0.f) sexp = 61 - ilogb((double)maxabs * (double)a.m) - 1;
  const double scale = ldexp(1.0, sexp), inv_scale = ldexp(1.0, -sexp);
  const float scalef = (float)scale;  // a power of two: x * scalef is exact (|x| 2^s < 2^61)
  constexpr int HH = GR <= 4 ? 3 : 1;  // points per lane in the full search: every centroid LDS serves HH
  constexpr int JJ = GR >= 16 ? 4 : 1; // centroids per step: independent FMA chains for long guides
  // candidate masks of every cell from the current FP32 centroids (one warp per cell, lanes over centroids)
  auto build_grid = [&]() {
    int ncell = 1;
    for (int d = 0; d < rho; ++d) ncell *= KM_NG;
    for (int cell = b * nw + w; cell < ncell; cell += nb * nw) {
      int kk[3] = {cell % KM_NG, (cell / KM_NG) % KM_NG, cell / (KM_NG * KM_NG)};
      double mind[2] = {INFINITY, INFINITY}, maxd = INFINITY;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int j = lane + 32 * u;
        if (j < m0) {
          double mn = 0.0, mx = 0.0;
          for (int d = 0; d < rho; ++d) {
            const double blo = (double)glo[d] + ((double)kk[d] - 1e-3) * gh[d];
            const double bhi = (double)glo[d] + ((double)kk[d] + 1.0 + 1e-3) * gh[d];
            const double c = (double)Cf[j * rhop + d];
            const double below = blo - c, above = c - bhi;
            const double t = fmax(fmax(below, above), 0.0);
            mn += t * t;
            const double f = fmax(c - blo, bhi - c);
            mx += f * f;
          }
          mind[u] = mn;
          maxd = fmin(maxd, mx);
        }
      }
      for (int o = 16; o > 0; o >>= 1) maxd = fmin(maxd, __shfl_xor_sync(0xffffffffu, maxd, o));
      const double thr = maxd * (1.0 + 1e-4) + 1e-300;
      const unsigned m_lo = __ballot_sync(0xffffffffu, mind[0] <= thr);
      const unsigned m_hi = __ballot_sync(0xffffffffu, mind[1] <= thr);
      if (lane == 0) reinterpret_cast<unsigned long long*>(a.lb)[cell] = ((unsigned long long)m_hi << 32) | m_lo;
    }
  };
  if constexpr (gridmode) {
    if (threadIdx.x < 3) {
      const int d = threadIdx.x;
      float lo_v = 0.f, hi_v = 0.f;
      if (d < rho) {
        const unsigned eh = __ldcg(a.maxabs_bits + 1 + d), el = __ldcg(a.maxabs_bits + 4 + d);
        if (eh && el) {
          hi_v = f32_unordered(eh);
          lo_v = -f32_unordered(el);
        }
      }
      const float range = hi_v - lo_v;
      const bool ok = range > 1e-30f && range < 3.0e38f;
      glo[d] = lo_v;
      ginv[d] = ok ? (float)KM_NG / range : 0.f;
      gh[d] = ok ? ((double)hi_v - (double)lo_v) / (double)KM_NG : 0.0;
    }
    __syncthreads();
    build_grid();
    grid.sync();
  }

  for (int it = 0; it < a.max_iter; ++it) {
    const int par = it & 1;
    unsigned long long* D = a.gacc + (size_t)(it % 3) * gstride;
    // next iteration's delta buffer: last read after the barrier of it-2, next written after this one's
    if (b == 0)
      for (int k = threadIdx.x; k < gstride; k += blockDim.x) a.gacc[(size_t)((it + 1) % 3) * gstride + k] = 0ull;
    for (int k = threadIdx.x; k < nw * msl; k += blockDim.x) wacc[k] = 0ull;
    for (int k = threadIdx.x; k < nw * m0; k += blockDim.x) wcnt[k] = 0;
    if constexpr (GRID)
      for (int k = threadIdx.x; k < nw * msl * 3; k += blockDim.x) wlim[k] = 0;
    const double dcum = dcum_sh;
    if constexpr (TC) {  // B = (-2 c_j, |c_j|^2) from the current FP32 centroids, split hi / lo
      for (int k = threadIdx.x; k < NU * KU; k += blockDim.x) {
        const int j = k / KU, d = k - j * KU;
        float v = 0.f;
        if (j < m0) {
          if (d < rho) {
            v = -2.f * Cf[j * rhop + d];
          } else if (d == rho) {
            for (int q = 0; q < rho; ++q) v = fmaf(Cf[j * rhop + q], Cf[j * rhop + q], v);
          }
        }
        const float h = umma::to_tf32(v);
        const int o = umma::kmajor_offset(j, d, NU);
        Bh[o] = h;
        Bl[o] = umma::to_tf32(v - h);
      }
      if (w == 0) {
        float mx = 0.f;
        for (int j = lane; j < m0; j += 32) {
          float v = 0.f;
          for (int q = 0; q < rho; ++q) v = fmaf(Cf[j * rhop + q], Cf[j * rhop + q], v);
          mx = fmaxf(mx, v);
        }
        mx = warp_max(mx);
        if (lane == 0) tc_ccmax = mx;
      }
      umma::fence_proxy_async();  // generic-proxy writes of B -> tensor core
    }
    __syncthreads();
    unsigned long long* myacc = wacc + (size_t)w * msl;
    int* mycnt = wcnt + (size_t)w * m0;
    double near_sum = 0.0, changed = 0.0;
    const bool full_pass = it == 0 || !a.bounds;
    long long nlist = hi - lo;
    if constexpr (gridmode) {
      if constexpr (GRIDOK) {
        constexpr int NCELL = RX == 1 ? KM_NG : (RX == 2 ? KM_NG * KM_NG : KM_NG * KM_NG * KM_NG);
        for (int k0 = threadIdx.x; k0 < NCELL; k0 += 8 * blockDim.x) {  // 8 loads in flight per thread
          unsigned long long tmp[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) tmp[u] = k0 + u * blockDim.x < NCELL ? __ldcg(reinterpret_cast<unsigned long long*>(a.lb) + k0 + u * blockDim.x) : 0ull;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (k0 + u * blockDim.x < NCELL) gts[k0 + u * blockDim.x] = tmp[u];
        }
        __syncthreads();
        // A warp takes HG x 32 consecutive points per trip and searches the *union* of their
        // cells' candidate sets, in ascending index, for all of them: a superset search returns
        // the same label and distance, the loop and the centroid loads are warp-uniform
        // (broadcast LDS, no per-lane mask arithmetic or divergence), and consecutive pixels
        // share most of their candidates.
        constexpr int HG = 2;
        const float4* Cf4 = reinterpret_cast<const float4*>(Cf);  // rhop == 4
        // trips are dealt round-robin over every warp of the grid (not a contiguous chunk per
        // block): busy image regions, whose pixels touch more cells, spread over all blocks
        const long long gw = (long long)b * nw + w, gnw = (long long)nb * nw;
        for (long long q0 = gw * 32 * HG; q0 < a.m; q0 += gnw * 32 * HG) {
          float x[HG][GR], best[HG];
          int arg[HG], oldl[HG];
          bool valid[HG];
#pragma unroll
          for (int h = 0; h < HG; ++h) {
            const long long q = q0 + 32 * h + lane;
            valid[h] = q < a.m;
            const long long i = valid[h] ? q : 0;
#pragma unroll
            for (int d = 0; d < GR; ++d) x[h][d] = (valid[h] && d < rho) ? __ldg(a.pts + d * a.ps + i) : 0.f;
            oldl[h] = (valid[h] && it > 0) ? a.labels[i] : -1;
          }
          unsigned ulo = 0u, uhi = 0u;
#pragma unroll
          for (int h = 0; h < HG; ++h) {
            int cell = 0, mul = 1;
#pragma unroll
            for (int d = 0; d < RX; ++d) {
              const int kd = min(KM_NG - 1, max(0, (int)((x[h][d] - glo[d]) * ginv[d])));
              cell += kd * mul;
              mul *= KM_NG;
            }
            const unsigned long long mk = valid[h] ? gts[cell] : 0ull;
            ulo |= (unsigned)mk;
            uhi |= (unsigned)(mk >> 32);
            best[h] = INFINITY;
            arg[h] = 0;
          }
          ulo = __reduce_or_sync(0xffffffffu, ulo);
          uhi = __reduce_or_sync(0xffffffffu, uhi);
          auto eval = [&](int j) {
            const float4 c4 = Cf4[j];
            const float cc[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
            for (int h = 0; h < HG; ++h) {
              float d2 = 0.f;
#pragma unroll
              for (int d = 0; d < RX; ++d) {
                const float t = x[h][d] - cc[d];
                d2 = fmaf(t, t, d2);
              }
              if (d2 < best[h]) {  // ascending j, strict: first index wins ties
                best[h] = d2;
                arg[h] = j;
              }
            }
          };
          for (unsigned u = ulo; u; u &= u - 1u) eval(__ffs(u) - 1);
          for (unsigned u = uhi; u; u &= u - 1u) eval(31 + __ffs(u));
#pragma unroll
          for (int h = 0; h < HG; ++h) {
            const long long i = q0 + 32 * h + lane;
            int old = -1;
            bool chg = false;
            if (valid[h]) {
              near_sum += (double)best[h];
              old = oldl[h];
              chg = old != arg[h];
              if (chg) {
                changed += 1.0;
                a.labels[i] = arg[h];
              }
            }
            if (it == 0) {  // every point enters its cluster: label groups reduced with REDUX
              warp_accumulate_fx<GR>(x[h], rho, arg[h], valid[h] && chg, scale, 1, myacc, mycnt);
            } else if (chg) {
              // few lanes change label after the first iteration: they add their fixed-point
              // coordinates to this warp's table with shared-memory atomics (integer adds commute,
              // so the sums stay exact and order-independent); x * 2^s is exact in FP32.  64-bit
              // shared atomics are compare-and-swap loops on sm_100a, so the value goes in as three
              // signed 21-bit limbs with native 32-bit adds (a warp adds < 2^9 points per iteration)
              int* mylim = wlim + (size_t)w * msl * 3;
#pragma unroll
              for (int d = 0; d < RX; ++d) {
                const long long v = __float2ll_rn(x[h][d] * scalef);
                const unsigned long long mag = (unsigned long long)(v < 0 ? -v : v);
                const int sg = v < 0 ? -1 : 1;
                const int l0 = sg * (int)(mag & 0x1FFFFFull), l1 = sg * (int)((mag >> 21) & 0x1FFFFFull),
                          l2 = sg * (int)(mag >> 42);
                int* pn = mylim + (arg[h] * rho + d) * 3;
                int* po = mylim + (old * rho + d) * 3;
                atomicAdd(pn, l0);
                atomicAdd(po, -l0);
                if (l1) {
                  atomicAdd(pn + 1, l1);
                  atomicAdd(po + 1, -l1);
                }
                if (l2) {
                  atomicAdd(pn + 2, l2);
                  atomicAdd(po + 2, -l2);
                }
              }
              atomicAdd(mycnt + arg[h], 1);
              atomicSub(mycnt + old, 1);
            }
          }
        }
        nlist = 0;  // phase B has nothing left
      }
    } else if constexpr (TC) {
      const int g = w >> 2, gw = w & 3, gtid = threadIdx.x & 127;  // two groups of four warps (nw == 8)
      const int wu = __shfl_sync(0xffffffffu, w, 0);
      const uint32_t tbase = (uint32_t)(g * tcols);  // tc_tmem == 0
      const uint32_t dcol = tbase, a_hi = tbase + (uint32_t)((NU + 31) & ~31), a_lo = a_hi + (uint32_t)((KU + 31) & ~31);
      const uint32_t lane_base = (uint32_t)(32 * gw) << 16;
      const uint32_t idesc = umma::idesc_tf32(128, NU);
      const uint32_t lbo_b = (uint32_t)NU * 16;
      const uint64_t desc_h = umma::desc_kmajor(Bh, lbo_b, 128), desc_l = umma::desc_kmajor(Bl, lbo_b, 128);
      const uint64_t desc_step = (uint64_t)((8 * NU * 4) >> 4);  // one K step (8 columns) in the address field
      const float ccmax = tc_ccmax;
      constexpr int KC = (GR + 1 + 15) / 16;  // 16-column chunks of the A operand (x, 1, 0 ...)
      auto load_pt = [&](long long i, bool valid, float (&x)[GR], int& oldl) {
#pragma unroll
        for (int d = 0; d < GR; ++d) x[d] = (valid && d < rho) ? __ldg(a.pts + d * a.ps + i) : 0.f;
        oldl = (valid && it > 0) ? a.labels[i] : -1;
      };
      float x[GR];
      int oldl;
      // 128-point tiles dealt round-robin over every group of the grid (content-dependent work --
      // label changes, multi-candidate points -- spreads over all blocks)
      const long long tstep = 128ll * 2 * nb;
      long long base = 128ll * (2 * b + g);
      load_pt(base + gtid, base + gtid < a.m, x, oldl);
      for (; base < a.m; base += tstep) {
        const long long i = base + gtid;
        const bool valid = i < a.m;
        float xx = 0.f;
#pragma unroll
        for (int d = 0; d < GR; ++d)
          if (d < rho) xx = fmaf(x[d], x[d], xx);
        // A operand: row = this thread's TMEM lane, columns (x_0 .. x_rho-1, 1, 0 ...), hi then lo;
        // hi = x rounded to TF32 (integer round-half-up), lo = x - hi exactly (read by truncation)
#pragma unroll
        for (int c = 0; c < KC; ++c) {
          if (16 * c < KU) {
            float h[16], l[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int d = 16 * c + e;
              float v = 0.f;
              if (d < GR) v = x[d < GR ? d : 0];
              if (d == rho) v = 1.f;
              h[e] = __uint_as_float((__float_as_uint(v) + 0x1000u) & 0xffffe000u);
              l[e] = v - h[e];
            }
            umma::st_32x32b_x16(a_hi + lane_base + (uint32_t)(16 * c), h);
            umma::st_32x32b_x16(a_lo + lane_base + (uint32_t)(16 * c), l);
          }
        }
        umma::st_wait();
        umma::fence_before();
        asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
        // the group's first warp issues, converged, one elected lane per MMA (mma_tf32_ts_elect);
        // wu is the warp index as a value the compiler knows to be warp-uniform
        auto issue = [&](auto gc) {
          constexpr int G = decltype(gc)::value;
          umma::fence_after();
          const uint32_t d0 = (uint32_t)(G * tcols);
          const uint32_t ah = d0 + (uint32_t)((NU + 31) & ~31), al = ah + (uint32_t)((KU + 31) & ~31);
          uint32_t acc = 0;
#pragma unroll 1
          for (int pass = 0; pass < 3; ++pass) {
            const uint32_t A = pass == 1 ? al : ah;
            uint64_t B = pass == 2 ? desc_l : desc_h;
#pragma unroll 1
            for (int kk = 0; kk < KU / 8; ++kk, B += desc_step) {
              umma::mma_tf32_ts_elect(d0, A + (uint32_t)(8 * kk), B, idesc, acc);
              acc = 1;
            }
          }
          umma::commit_elect(&tc_bar[G]);
        };
        if (wu == 0) issue(std::integral_constant<int, 0>{});
        if (wu == 4) issue(std::integral_constant<int, 1>{});
        // the next tile's coordinates travel while the tensor core and the re-check work
        float xn[GR];
        int oldn;
        load_pt(i + tstep, i + tstep < a.m, xn, oldn);
        umma::mbar_wait(&tc_bar[g], tc_phase);
        tc_phase ^= 1u;
        umma::fence_after();
        // smallest and second-smallest approximate distance (minus |x|^2) with the argmin: nearly
        // every point has one candidate within 2 delta, re-checked without divergence
        // (four interleaved chains: a single running minimum is a 3-deep dependent select per column)
        float m4[4] = {INFINITY, INFINITY, INFINITY, INFINITY}, s4[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
        int j4[4] = {0, 0, 0, 0};
        for (int c = 0; c < NU / 16; ++c) {
          float v[16];
          umma::ld_32x32b_x16(dcol + lane_base + (uint32_t)(16 * c), v);
          umma::ld_wait();
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int j = 16 * c + e;
            const float ve = j < m0 ? v[e] : INFINITY;
            const int q = e & 3;
            if (ve < m4[q]) {
              s4[q] = m4[q];
              m4[q] = ve;
              j4[q] = j;
            } else {
              s4[q] = fminf(s4[q], ve);
            }
          }
        }
        float mn = m4[0], mn2 = s4[0];
        int jmin = j4[0];
#pragma unroll
        for (int q = 1; q < 4; ++q) {  // merge: smallest value (lowest index on ties), second smallest
          if (m4[q] < mn || (m4[q] == mn && j4[q] < jmin)) {
            mn2 = fminf(fminf(mn2, s4[q]), mn);
            mn = m4[q];
            jmin = j4[q];
          } else {
            mn2 = fminf(fminf(mn2, s4[q]), m4[q]);
          }
        }
        // delta: 3 K FP32 accumulation roundings, the dropped lo.lo products and the truncated lo
        // operands bound |D_j + |x|^2 - d2| by ~7e-6 (|x|^2 + 2 max|c|^2); 3e-5 keeps a 4x margin
        const float lim = mn + 2.f * (3e-5f * (xx + 2.f * ccmax) + 1e-30f);
        float best = d2_f32<GR>(x, rho, Cf + (size_t)jmin * rhop);
        int arg = jmin;
        if (__any_sync(0xffffffffu, mn2 <= lim)) {  // rare: several candidates, ascending j with first-index ties
          // (tcgen05.ld is warp-collective: every lane drains, the lanes with one candidate skip the math)
          for (int c = 0; c < NU / 16; ++c) {
            float v[16];
            umma::ld_32x32b_x16(dcol + lane_base + (uint32_t)(16 * c), v);
            umma::ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int j = 16 * c + e;
              if (mn2 <= lim && j < m0 && j != jmin && v[e] <= lim) {
                const float d2 = d2_f32<GR>(x, rho, Cf + (size_t)j * rhop);
                if (d2 < best || (d2 == best && j < arg)) {
                  best = d2;
                  arg = j;
                }
              }
            }
          }
        }
        bool chg = false;
        if (valid) {
          near_sum += (double)best;
          chg = oldl != arg;
          if (chg) {
            changed += 1.0;
            a.labels[i] = arg;
          }
        }
        warp_accumulate_fx<GR>(x, rho, arg, valid && chg, scale, 1, myacc, mycnt);
        warp_accumulate_fx<GR>(x, rho, oldl, valid && chg && oldl >= 0, scale, -1, myacc, mycnt);
        umma::fence_before();
        asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");  // the group's TMEM reads are done
        umma::fence_after();
#pragma unroll
        for (int d = 0; d < GR; ++d) x[d] = xn[d];
        oldl = oldn;
      }
      nlist = 0;  // phase B has nothing left
    } else if (!full_pass) {
      // phase A: warp w tests its contiguous sub-range; failures go to its list segment in point order
      // PA chunks of 32 points in flight per warp: their point, label and bound
      // loads are issued together (the per-chunk loads are otherwise two
      // dependent L2 round trips each), then tested in point order
      constexpr int PA = GR <= 4 ? 4 : 2;
      int nl = 0;
      for (long long base = wlo; base < whi; base += 32 * PA) {
        float x[PA][GR], lbv[PA];
        int lab[PA];
#pragma unroll
        for (int u = 0; u < PA; ++u) {
          const long long v = base + 32 * u + lane;
          const long long i = gmap(v);
          const bool valid = v < whi && i < a.m;
#pragma unroll
          for (int d = 0; d < GR; ++d) x[u][d] = (valid && d < rho) ? __ldg(a.pts + d * a.ps + i) : 0.f;
          lab[u] = valid ? a.labels[i] : 0;
          lbv[u] = valid ? a.lb[i] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < PA; ++u) {
          const long long v = base + 32 * u + lane;
          const long long i = gmap(v);
          bool need = false;
          if (v < whi && i < a.m) {
            const float d2a = d2_f32<GR>(x[u], rho, Cf + (size_t)lab[u] * rhop);
            const double lbe = (double)lbv[u] - dcum;
            if (lbe > 0.0 && (double)d2a * (1.0 + LB_EPS) < lbe * lbe * (1.0 - LB_EPS)) near_sum += (double)d2a;
            else need = true;
          }
          const unsigned bal = __ballot_sync(0xffffffffu, need);
          if (need) a.list[wlo + nl + __popc(bal & ((1u << lane) - 1u))] = (int)i;
          nl += __popc(bal);
        }
      }
      if (lane == 0) wlen[w] = nl;
      __syncthreads();
      if (threadIdx.x == 0) {
        wpre[0] = 0;
        for (int q = 0; q < nw; ++q) wpre[q + 1] = wpre[q] + wlen[q];
      }
      __syncthreads();
      nlist = wpre[nw];
    }
    // phase B: the m0-way search (every point on full passes, else the listed ones)
    int sgc = 0;  // list segment of this thread's last point: q only grows, so the scan resumes there
    for (long long q0 = (long long)w * 32 * HH; q0 < nlist; q0 += (long long)nw * 32 * HH) {
      float x[HH][GR];
      float best[HH], second[HH];
      int arg[HH], oldl[HH];
      long long idx[HH];
      bool valid[HH];
#pragma unroll
      for (int h = 0; h < HH; ++h) {
        best[h] = second[h] = INFINITY;
        arg[h] = 0;
        const long long q = q0 + 32 * h + lane;
        valid[h] = q < nlist;
        long long i = 0;
        if (valid[h]) {
          if (full_pass) {
            i = gmap(lo + q);
            valid[h] = i < a.m;
            if (!valid[h]) i = 0;
          } else {
            while (q >= wpre[sgc + 1]) ++sgc;
            i = a.list[min(hi, lo + sgc * cw) + (q - wpre[sgc])];
          }
        }
        idx[h] = i;
#pragma unroll
        for (int d = 0; d < GR; ++d) x[h][d] = (valid[h] && d < rho) ? __ldg(a.pts + d * a.ps + i) : 0.f;
        oldl[h] = (valid[h] && it > 0) ? a.labels[i] : -1;  // issued with the point loads, used after the search
      }
      for (int j0 = 0; j0 < m0; j0 += JJ) {
        float d2[JJ][HH];
#pragma unroll
        for (int jj = 0; jj < JJ; ++jj)
#pragma unroll
          for (int h = 0; h < HH; ++h) d2[jj][h] = 0.f;
#pragma unroll
        for (int d4 = 0; d4 < (GR + 3) / 4; ++d4) {
          if (4 * d4 < rho) {
            float cc[JJ][4];
#pragma unroll
            for (int jj = 0; jj < JJ; ++jj) {
              const float4 c4 = reinterpret_cast<const float4*>(Cf + (size_t)(j0 + jj) * rhop)[d4];
              cc[jj][0] = c4.x;
              cc[jj][1] = c4.y;
              cc[jj][2] = c4.z;
              cc[jj][3] = c4.w;
            }
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (4 * d4 + e < GR && 4 * d4 + e < rho) {
#pragma unroll
                for (int jj = 0; jj < JJ; ++jj)
#pragma unroll
                  for (int h = 0; h < HH; ++h) {
                    const float t = x[h][4 * d4 + e] - cc[jj][e];
                    d2[jj][h] = fmaf(t, t, d2[jj][h]);
                  }
              }
          }
        }
#pragma unroll
        for (int jj = 0; jj < JJ; ++jj)
#pragma unroll
          for (int h = 0; h < HH; ++h) {
            const float v = d2[jj][h];
            if (v < best[h]) {  // strict, ascending j: first index wins ties (np.argmin)
              second[h] = best[h];
              best[h] = v;
              arg[h] = j0 + jj;
            } else {
              second[h] = fminf(second[h], v);
            }
          }
      }
#pragma unroll
      for (int h = 0; h < HH; ++h) {
        const long long i = idx[h];
        int old = -1;
        bool chg = false;
        if (valid[h]) {
          near_sum += (double)best[h];
          old = oldl[h];
          chg = old != arg[h];
          if (chg) {
            changed += 1.0;
            a.labels[i] = arg[h];
          }
          // drift-adjusted lower bound on the distance to the second-closest centroid
          const double lbv = (double)sqrtf(second[h]) * (1.0 - LB_EPS) + dcum;
          a.lb[i] = second[h] < INFINITY ? __double2float_rd(lbv) : 3.0e38f;
        }
        warp_accumulate_fx<GR>(x[h], rho, arg[h], valid[h] && chg, scale, 1, myacc, mycnt);
        warp_accumulate_fx<GR>(x[h], rho, old, valid[h] && chg && old >= 0, scale, -1, myacc, mycnt);
      }
    }
    near_sum = warp_sum(near_sum);
    changed = warp_sum(changed);
    if (lane == 0) {
      extra[0][w] = near_sum;
      extra[1][w] = changed;
    }
    __syncthreads();
    // block deltas -> global exact integer accumulators (order-independent, two's complement)
    for (int k = threadIdx.x; k < msl; k += blockDim.x) {
      unsigned long long t = 0;
      for (int q = 0; q < nw; ++q) t += wacc[(size_t)q * msl + k];
      if constexpr (GRID) {
        for (int q = 0; q < nw; ++q) {
          const int* l = wlim + ((size_t)q * msl + k) * 3;
          t += (unsigned long long)((long long)l[0] + ((long long)l[1] << 21) + ((long long)l[2] << 42));
        }
      }
      if (t) atomicAdd(D + k, t);
    }
    for (int k = threadIdx.x; k < m0; k += blockDim.x) {
      long long t = 0;
      for (int q = 0; q < nw; ++q) t += wcnt[(size_t)q * m0 + k];
      if (t) atomicAdd(D + msl + k, (unsigned long long)t);
    }
    double* P = a.part + (size_t)par * nb * 2;
    if (threadIdx.x == 0) {
      double e = 0.0, c = 0.0;
      for (int q = 0; q < nw; ++q) {
        e += extra[0][q];
        c += extra[1][q];
      }
      P[2 * b] = e;
      P[2 * b + 1] = c;
    }
    grid.sync();
    // every block: running exact totals, objective/changed in fixed block order
    for (int k = threadIdx.x; k < gstride; k += blockDim.x) T[k] += (long long)__ldcg(D + k);
    {
      double e = 0.0, c = 0.0;
      for (int q = threadIdx.x; q < nb; q += blockDim.x) {
        e += __ldcg(P + 2 * q);
        c += __ldcg(P + 2 * q + 1);
      }
      e = block_sum(e, sh);
      if (threadIdx.x == 0) misc[0] = e;
      c = block_sum(c, sh);
      if (threadIdx.x == 0) misc[1] = c;
    }
    __syncthreads();
    const double chg = misc[1];
    if (b == 0 && threadIdx.x == 0) {
      a.errors[it] = misc[0];
      a.st->iters = it + 1;
      a.st->changed = (long long)chg;
    }
    if (it > 0 && chg == 0.0) {
      if (b == 0 && threadIdx.x == 0) a.st->converged = 1;
      break;  // uniform: every block read the same total
    }
    for (int k = threadIdx.x; k < msl; k += blockDim.x) {
      Cp[k] = Cd[k];
      const int j = k / rho;
      const double cnt = (double)T[msl + j];
      if (cnt > 0.0) Cd[k] = ((double)T[k] * inv_scale) / cnt;
    }
    __syncthreads();
    // empty clusters, ascending j: farthest remaining point from its old centroid
    int nex = 0;
    bool mine_empty = false;
    for (int j = threadIdx.x; j < m0; j += blockDim.x) mine_empty |= T[msl + j] <= 0;
    const int jend = __syncthreads_or(mine_empty) ? m0 : 0;  // (the common case: none, no serial scan)
    for (int j = 0; j < jend; ++j) {
      if (T[msl + j] > 0) continue;
      double bv = -INFINITY;
      long long bi = a.m;
      for (long long i = clo + threadIdx.x; i < chi; i += blockDim.x) {
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
    // next iteration's FP32 centroids and the largest centroid movement (rounded up)
    for (int k = threadIdx.x; k < m0p * rhop; k += blockDim.x) {
      Cfo[k] = Cf[k];
      const int j = k / rhop, d = k - j * rhop;
      Cf[k] = j >= m0 ? 3.0e38f : (d < rho ? (float)Cd[j * rho + d] : 0.f);
    }
    __syncthreads();
    double mv = 0.0;
    if constexpr (!gridmode && !TC)  // (the cell-pruned / tensor-core searches keep no drift-adjusted bounds)
    for (int j = threadIdx.x; j < m0; j += blockDim.x) {
      double s2 = 0.0;
      for (int d = 0; d < rho; ++d) {
        const double t = (double)Cf[j * rhop + d] - (double)Cfo[j * rhop + d];
        s2 += t * t;
      }
      mv = fmax(mv, sqrt(s2));
    }
    if constexpr (!gridmode && !TC) {
      for (int o = 16; o > 0; o >>= 1) mv = fmax(mv, __shfl_xor_sync(0xffffffffu, mv, o));
      if (lane == 0) sh[w] = mv;
      __syncthreads();
      if (threadIdx.x == 0) {
        double mx = 0.0;
        for (int q = 0; q < nw; ++q) mx = fmax(mx, sh[q]);
        dcum_sh = dcum + mx * (1.0 + 1e-9) + 1e-30;  // monotone, never understated
      }
      __syncthreads();
    }
    if (gridmode && it + 1 < a.max_iter) {
      if constexpr (GRID) build_grid();
      grid.sync();
    }
  }
  if constexpr (TC) {
    umma::fence_before();
    __syncthreads();
    if (w == 0) umma::tmem_dealloc(tc_tmem, (uint32_t)tc_alloc);
  }
  if (b == 0)
    for (int k = threadIdx.x; k < msl; k += blockDim.x) a.C[k] = Cd[k];
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
int launch_seed_coop(const float* pts, long long ps, long long m, int rho, int m0, const double* uniforms_dev,
                     double* C, long long* seeds, char* ws, const KLayout& L, cudaStream_t s) {
  if (m0 < 2) return NYS_OK;
  if (!coop_supported() || rho > NYS_MAX_RHO) return NYS_EUNSUPPORTED;  // wide guides: step-wise seeding
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
  a.flag = seed_flag(ws, L);  // zeroed by k_seed_prologue
  void* args[] = {&a};
  const char* v1 = getenv("NYS_SEED_V1");
  const bool runs = !(v1 && atoi(v1));
  const char* sm_e = getenv("NYS_SEED_MODE");
  a.mode = sm_e ? (atoi(sm_e) ? 1 : 0) : 1;
  auto go = [&](auto kern_v1, auto kern_runs) -> int {
    // one block per SM; the block's D^2 chunk lives in shared memory when it fits
    const int nb = (int)std::max<long long>(1, std::min<long long>((long long)sms(), ceil_div(m, 512)));
    const long long chunk = ceil_div(m, (long long)nb);
    size_t smem;
    void* kern;
    if (runs) {
      a.per = (int)ceil_div(chunk, 512);
      a.pp = reinterpret_cast<float*>(ws + L.off_pp);
      a.pps = L.m_pad;
      a.tsum = reinterpret_cast<double*>(ws + L.off_tsum);
      const size_t hist = (size_t)m0 * rho * 8 + (size_t)a.per * 8;  // centroid history + owning run
      smem = (size_t)a.per * 512 * 8 + hist;
      a.d2_in_smem = smem <= 200 * 1024;
      if (!a.d2_in_smem) smem = hist;
      kern = (void*)kern_runs;
    } else {
      smem = (size_t)chunk * 8;
      a.d2_in_smem = smem <= 200 * 1024;
      if (!a.d2_in_smem) smem = 0;
      kern = (void*)kern_v1;
    }
    int per_sm = 0;
    NYS_CUDA_TRY(coop_blocks_per_sm(kern, 512, smem, &per_sm));
    if (per_sm < 1) return NYS_EUNSUPPORTED;
    count_launch();
    NYS_CUDA_TRY(cudaLaunchCooperativeKernel(kern, dim3(nb), dim3(512), args, smem, s));
    return NYS_OK;
  };
#define NYS_SEED_GO(GR, RX) go(k_seed_coop<GR, RX>, k_seed_runs<GR, RX>)
  switch (rho) {
    case 1: return NYS_SEED_GO(4, 1);
    case 2: return NYS_SEED_GO(4, 2);
    case 3: return NYS_SEED_GO(4, 3);
    case 4: return NYS_SEED_GO(4, 4);
    default: break;
  }
  switch (rho) {  // exact compile-time dimensions of the BASELINE guides
    case 16: return NYS_SEED_GO(16, 16);
    case 27: return NYS_SEED_GO(32, 27);
    case 31: return NYS_SEED_GO(32, 31);
    default: break;
  }
  if (rho <= 16) return NYS_SEED_GO(16, 0);
  if (rho <= 32) return NYS_SEED_GO(32, 0);
  return NYS_SEED_GO(64, 0);
#undef NYS_SEED_GO
}

int launch_lloyd_coop(const float* pts, long long ps, long long m, int rho, int m0, int max_iter, double* C,
                      double* errors, char* ws, const KLayout& L, cudaStream_t s, bool prezeroed) {
  if (!coop_supported() || rho > NYS_MAX_RHO) return NYS_EUNSUPPORTED;
  const int msl = m0 * rho;
  const size_t fixed = (size_t)msl * 8 * 2 + (size_t)(msl + m0) * 8 + (size_t)m0 * 8 +
                       2 * (size_t)((m0 + 3) & ~3) * ((rho + 3) & ~3) * 4 + 96;
  const char* eg = getenv("NYS_KM_NOGRID");
  const bool gridmode = rho <= 3 && m0 <= 64 && !(eg && atoi(eg));
  size_t gcells = 1;
  for (int d = 0; d < rho; ++d) gcells *= KM_NG;
  const size_t gsm = gridmode ? gcells * 8 + 16 + 64 + (size_t)8 * msl * 3 * 4 : 0;  // masks, box, limb tables
  // tensor-core search for wide guides: (x, 1) needs K = rho + 1 padded to 8, N = m0 padded to 16,
  // two groups' D / A_hi / A_lo columns in the 512-column TMEM
  // NYS_KM_TC_COOP = 1 / 0 forces it on / off.  Default: on where it measured faster than the bounds
  // kernel -- the bounds kernel's full searches grow with m0 * rho, the tensor-core tiles hardly do:
  // cfg 3 (m0 64, rho 27) 6.5 -> 5.9 ms clustering, cfg 4 (m0 48, rho 31) 4.6 -> 4.8 ms
  const char* etc = getenv("NYS_KM_TC_COOP");
  const bool tc_wanted = etc ? atoi(etc) != 0 : (long long)m0 * rho >= 1600;
  const int KUt = (int)ceil_div(rho + 1, 8) * 8, NUt = (int)ceil_div(m0, 16) * 16;
  bool use_tc = rho >= 16 && tc_wanted && NUt <= 256 &&
                2 * (((NUt + 31) & ~31) + 2 * ((KUt + 31) & ~31)) <= 512;
  const size_t tsm = use_tc ? (size_t)2 * NUt * KUt * 4 + 128 : 0;
  auto need = [&](int nw) { return (size_t)nw * msl * 8 + (((size_t)nw * m0 + 1) & ~size_t(1)) * 4 + fixed + gsm + tsm; };
  int nw = 8;
  while (nw > 1 && need(nw) > 200 * 1024) --nw;
  const size_t smem = need(nw);
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
  a.gacc = reinterpret_cast<unsigned long long*>(ws + L.off_tot);
  a.part = reinterpret_cast<double*>(ws + L.off_part);
  a.arg = reinterpret_cast<double*>(ws + L.off_arg);
  a.errors = errors;
  a.st = reinterpret_cast<KState*>(ws + L.off_state);
  a.maxabs_bits = reinterpret_cast<unsigned*>(ws + L.off_idx);
  a.nw = nw;
  // the seeding D^2 array is dead during Lloyd: bounds in its first half, work lists in the second
  a.lb = reinterpret_cast<float*>(ws + L.off_d2);
  a.list = reinterpret_cast<int*>(ws + L.off_d2 + (size_t)m * 4);
  {
    const char* e = getenv("NYS_KM_NOBOUNDS");
    a.bounds = (e && atoi(e)) ? 0 : 1;
  }
  const bool use_grid = gridmode && a.bounds;  // candidate masks in place of the bound / list arrays
  // the first delta buffer starts at zero (the kernel zeroes each next one) and max|x| at +0
  if (!prezeroed) {  // else k_seed_prologue zeroed both
    NYS_CUDA_TRY(cudaMemsetAsync(a.gacc, 0, (size_t)(msl + m0) * 8, s));
    NYS_CUDA_TRY(cudaMemsetAsync(a.maxabs_bits, 0, 7 * sizeof(unsigned), s));  // max|x| and the bounding box words
  }
  void* args[] = {&a};
  auto go = [&](auto kern) -> int {
    int per_sm = 0;
    NYS_CUDA_TRY(coop_blocks_per_sm((const void*)kern, nw * 32, smem, &per_sm));
    if (per_sm < 1) return NYS_EUNSUPPORTED;
    const int nb = (int)std::max<long long>(
        1, std::min<long long>({(long long)per_sm * sms(), (long long)L.nb_coop, ceil_div(m, (long long)nw * 64)}));
    count_launch();
    NYS_CUDA_TRY(cudaLaunchCooperativeKernel((void*)kern, dim3(nb), dim3(nw * 32), args, smem, s));
    return NYS_OK;
  };
  if (use_tc && a.bounds && nw == 8) {  // (fewer warps: the per-warp tables did not fit; FP32 bounds kernel)
    switch (rho) {
      case 16: return go(k_lloyd_coop<16, 16, false, true>);
      case 27: return go(k_lloyd_coop<32, 27, false, true>);
      case 31: return go(k_lloyd_coop<32, 31, false, true>);
      default: break;
    }
    if (rho <= 32) return go(k_lloyd_coop<32, 0, false, true>);
    return go(k_lloyd_coop<64, 0, false, true>);
  }
  if (use_grid) {
    switch (rho) {
      case 1: return go(k_lloyd_coop<4, 1, true>);
      case 2: return go(k_lloyd_coop<4, 2, true>);
      default: return go(k_lloyd_coop<4, 3, true>);
    }
  }
  switch (rho) {
    case 1: return go(k_lloyd_coop<4, 1>);
    case 2: return go(k_lloyd_coop<4, 2>);
    case 3: return go(k_lloyd_coop<4, 3>);
    case 4: return go(k_lloyd_coop<4, 4>);
    default: break;
  }
  switch (rho) {  // exact compile-time dimensions of the BASELINE guides
    case 16: return go(k_lloyd_coop<16, 16>);
    case 27: return go(k_lloyd_coop<32, 27>);
    case 31: return go(k_lloyd_coop<32, 31>);
    default: break;
  }
  if (rho <= 16) return go(k_lloyd_coop<16, 0>);
  if (rho <= 32) return go(k_lloyd_coop<32, 0>);
  return go(k_lloyd_coop<64, 0>);
}

}  // namespace nys
