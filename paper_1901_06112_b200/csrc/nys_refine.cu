// Near-guard FP64 refinement + filter statistics (nys_filter_finish).
//
// Reference region: filters.py:223-257 -- zeta, eta and the guarded ratio are
// formed in FP64 there.  K3 forms them in FP32 (y-form), which
// is ~1e-6 accurate wherever the ratio is well conditioned.  Where it is not --
// |eta| small against its own scale S = sum_i b_i |conv(y_i)|, or a guard
// decision (|eta| < eps_den, |eta_lead| >= eps_den) within FP32 error of its
// threshold -- K3 queues the pixel (near_guard, nys_filter_common.cuh) and this
// kernel re-evaluates it from the inputs alone, in FP64, by direct window
// summation:
//
//   eta(x)    = sum_y w(x-y) b(x)^T M b(y)        zeta_c(x) = same with f_c(y)
//   eta_l(x)  = s0(x) sum_y w(x-y) s0(y) / alpha_1,  s0 = u0 . b
//
// with M the FP64 mixing matrix (= sum_k w_k w_k^T / alpha_k, the reference's
// sum over retained eigenpairs of alpha_k v_k(x) v_k(y)) and the FP64
// landmarks, then applies the reference's guard in FP64 and overwrites the
// pixel.  One CTA per queued pixel (grid-strided); per window pixel b(y) costs
// m0 (2 rho + exp) FP64 operations.  The last CTA publishes min|eta| and the
// guarded count (K3 left the queued pixels out of both).
#include "nys_filter_common.cuh"

namespace nys {

constexpr int RF_THREADS = 256;
constexpr int RF_QPT = 4;  // window sums per thread: 2 (n + 1) <= 1024

struct RArgs {
  const float* f;
  const float* g;
  float* out;
  long long fps, gps, ops;
  int n, rho, H, W, m0, R, gkind, rlo, rhi, c_in_smem, nch, out64;
  const double* D;    // FP64 block: C64, U064, SC64 (filter_layout)
  const double* M64;  // m0 x m0 row-major
  const unsigned* list;
  unsigned cap;
  unsigned* chunk_cnt;  // per queued pixel: window chunks done
  double* part;         // per queued pixel: nch x 2(n+1) window partial sums
  int d_u0, d_sc;
  FilterStats* stats;
  double* stats_out;  // nullable: {min|eta|, guarded (int64 bits)}
  double inv;         // 1 / (2 theta^2), nystrom.py:48
  double taps[NYS_MAX_TAPS];
};

__device__ __forceinline__ float guide_val(const RArgs& a, int k, int row, int x) {
  if (a.gkind == 0) return __ldg(a.g + (long long)k * a.gps + (long long)row * a.W + x);
  const int c = k / 9, q = k - c * 9, dy = q / 3 - 1, dx = q - (q / 3) * 3 - 1;
  const int yy = clampi(row + dy, 0, a.H - 1), xx = clampi(x + dx, 0, a.W - 1);
  return __ldg(a.f + (long long)c * a.fps + (long long)yy * a.W + xx);
}

// Work item = (queued pixel e, window chunk k): the (2S+1)^2 window of a pixel is split over
// nch CTAs so a handful of queued pixels still spread over the GPU.  Each item writes its
// 2(n+1) partial sums; the CTA that completes a pixel's last chunk adds the partials in chunk
// order (deterministic), applies the guard and overwrites the pixel.
__global__ void __launch_bounds__(RF_THREADS) k_finish(const RArgs a) {
  extern __shared__ __align__(16) double rsm[];
  const int tid = threadIdx.x;
  const int m0 = a.m0, rho = a.rho, n = a.n, NQ = 2 * (n + 1), nch = a.nch;
  double* z = rsm;                // m0: M b(x)
  double* u0 = z + m0;            // m0
  double* bx = u0 + m0;           // m0
  double* gx = bx + m0;           // rho
  double* tw = gx + rho;          // 256: w(x-y) b(x)^T M b(y)
  double* tl = tw + RF_THREADS;   // 256: w(x-y) s0(y)
  double* res = tl + RF_THREADS;  // NQ
  double* Cs = res + NQ;          // m0 x rho (when c_in_smem)
  int* pos = reinterpret_cast<int*>(Cs + (a.c_in_smem ? (size_t)m0 * rho : 0));  // 256 (row, x) packed
  float* gy = reinterpret_cast<float*>(pos + RF_THREADS);                        // [rho][256]
  __shared__ double s0x_sh;
  __shared__ bool last_chunk;

  const double* C = a.c_in_smem ? Cs : a.D;
  for (int k = tid; k < m0; k += RF_THREADS) u0[k] = a.D[a.d_u0 + k];
  if (a.c_in_smem)
    for (int k = tid; k < m0 * rho; k += RF_THREADS) Cs[k] = a.D[k];
  const double inv_a1 = a.D[a.d_sc], eps = a.D[a.d_sc + 1];
  const unsigned cnt = min(*(volatile unsigned*)&a.stats->flagged, a.cap);
  const int R = a.R, T = 2 * R + 1, NP = T * T;
  const unsigned items = cnt * (unsigned)nch;
  __syncthreads();

  for (unsigned item = blockIdx.x; item < items; item += gridDim.x) {
    const unsigned e = item / (unsigned)nch;
    const int k = (int)(item - e * (unsigned)nch);
    const unsigned idx = a.list[e];
    const int row = (int)(idx / (unsigned)a.W), x = (int)(idx - (unsigned)row * (unsigned)a.W);
    for (int q = tid; q < rho; q += RF_THREADS) gx[q] = (double)guide_val(a, q, row, x);
    __syncthreads();
    for (int i = tid; i < m0; i += RF_THREADS) {
      double d2 = 0.0;
      for (int q = 0; q < rho; ++q) {
        const double t = gx[q] - C[(size_t)i * rho + q];
        d2 = fma(t, t, d2);
      }
      bx[i] = exp(-d2 * a.inv);
    }
    __syncthreads();
    for (int i = tid; i < m0; i += RF_THREADS) {
      double s = 0.0;
      const double* Mi = a.M64 + (size_t)i * m0;
      for (int j = 0; j < m0; ++j) s = fma(Mi[j], bx[j], s);
      z[i] = s;
    }
    if (tid < 32) {
      double s = 0.0;
      for (int j = tid; j < m0; j += 32) s = fma(u0[j], bx[j], s);
      s = warp_sum(s);
      if (tid == 0) s0x_sh = s;
    }
    // thread t owns the quantities q = t, t + 256, ... (c, kind) = (q % (n+1), q / (n+1)); NQ <= 1024
    double acc[RF_QPT] = {0.0, 0.0, 0.0, 0.0};
    const int p_lo = (int)((long long)NP * k / nch), p_hi = (int)((long long)NP * (k + 1) / nch);
    for (int base = p_lo; base < p_hi; base += RF_THREADS) {
      const int p = base + tid;
      __syncthreads();  // tw / tl / pos of the previous block consumed; z ready
      if (p < p_hi) {
        const int dy = p / T, dx = p - dy * T;
        const int yy = clampi(clampi(row + dy - R, 0, a.H - 1), a.rlo, a.rhi - 1);
        const int xx = clampi(x + dx - R, 0, a.W - 1);
        for (int q = 0; q < rho; ++q) gy[q * RF_THREADS + tid] = guide_val(a, q, yy, xx);
        double kz0 = 0.0, ks0 = 0.0, kz1 = 0.0, ks1 = 0.0;  // two landmark chains for ILP
        int i = 0;
        for (; i + 1 < m0; i += 2) {
          double d0 = 0.0, d1 = 0.0;
          for (int q = 0; q < rho; ++q) {
            const double gq = (double)gy[q * RF_THREADS + tid];
            const double t0 = gq - C[(size_t)i * rho + q], t1 = gq - C[(size_t)(i + 1) * rho + q];
            d0 = fma(t0, t0, d0);
            d1 = fma(t1, t1, d1);
          }
          const double b0 = exp(-d0 * a.inv), b1 = exp(-d1 * a.inv);
          kz0 = fma(z[i], b0, kz0);
          ks0 = fma(u0[i], b0, ks0);
          kz1 = fma(z[i + 1], b1, kz1);
          ks1 = fma(u0[i + 1], b1, ks1);
        }
        if (i < m0) {
          double d0 = 0.0;
          for (int q = 0; q < rho; ++q) {
            const double t0 = (double)gy[q * RF_THREADS + tid] - C[(size_t)i * rho + q];
            d0 = fma(t0, t0, d0);
          }
          const double b0 = exp(-d0 * a.inv);
          kz0 = fma(z[i], b0, kz0);
          ks0 = fma(u0[i], b0, ks0);
        }
        const double w = a.taps[dy] * a.taps[dx];
        tw[tid] = w * (kz0 + kz1);
        tl[tid] = w * (ks0 + ks1);
        pos[tid] = yy * a.W + xx;
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < RF_QPT; ++u) {
        const int qq = tid + u * RF_THREADS;
        if (qq < NQ) {
          const int c = qq % (n + 1), kind = qq / (n + 1);
          const double* t = kind ? tl : tw;
          const int lim = min(RF_THREADS, p_hi - base);
          for (int q = 0; q < lim; ++q) {
            const double fv = c < n ? (double)__ldg(a.f + (long long)c * a.fps + pos[q]) : 1.0;
            acc[u] = fma(t[q], fv, acc[u]);
          }
        }
      }
    }
    double* mine = a.part + ((size_t)e * nch + k) * NQ;
#pragma unroll
    for (int u = 0; u < RF_QPT; ++u)
      if (tid + u * RF_THREADS < NQ) mine[tid + u * RF_THREADS] = acc[u];
    __threadfence();
    __syncthreads();
    if (tid == 0) last_chunk = atomicAdd(&a.chunk_cnt[e], 1u) == (unsigned)nch - 1;
    __syncthreads();
    if (last_chunk) {
      __threadfence();
      const volatile double* pe = a.part + (size_t)e * nch * NQ;
      for (int qq = tid; qq < NQ; qq += RF_THREADS) {
        double s = 0.0;
        for (int kk = 0; kk < nch; ++kk) s += pe[(size_t)kk * NQ + qq];  // chunk order: deterministic
        res[qq] = s;
      }
      __syncthreads();
      const double eta = res[n];
      const double s0x = s0x_sh;
      const double eta_l = s0x * res[2 * n + 1] * inv_a1;
      for (int c = tid; c < n; c += RF_THREADS) {  // the reference's guard (filters.py:241-257), in FP64
        double o;
        if (fabs(eta) >= eps) o = res[c] / eta;
        else if (fabs(eta_l) >= eps) o = (s0x * res[n + 1 + c] * inv_a1) / eta_l;
        else o = (double)__ldg(a.f + (long long)c * a.fps + (long long)row * a.W + x);
        const long long oi = (long long)c * a.ops + (long long)row * a.W + x;
        if (a.out64) reinterpret_cast<double*>(a.out)[oi] = (double)(float)o;  // as K3 stores it
        else a.out[oi] = (float)o;
      }
      if (tid == 0) {
        atomicMin(&a.stats->min_abs_eta_bits, __float_as_uint((float)fabs(eta)));
        if (fabs(eta) < eps) {
          atomicAdd(&a.stats->guarded, 1ull);
          atomicAdd(&a.stats->refined_guarded, 1u);
        }
        a.chunk_cnt[e] = 0u;  // ready for the next filter
      }
    }
    __syncthreads();  // gx / bx / z / res reused by the next item
  }
  // the last CTA publishes the statistics
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (tid == 0) last = atomicAdd(&a.stats->finish_done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last && tid == 0) {
    __threadfence();
    volatile FilterStats* s = a.stats;
    if (a.stats_out) {
      if (s->gate_timeout) {  // the in-stream plan never arrived: the outputs are meaningless
        a.stats_out[0] = __longlong_as_double(0x7ff8000000000000ll);
        reinterpret_cast<long long*>(a.stats_out)[1] = -1ll;
      } else {
        a.stats_out[0] = (double)__uint_as_float(s->min_abs_eta_bits);
        reinterpret_cast<long long*>(a.stats_out)[1] = (long long)s->guarded;
      }
    }
    s->finish_done = 0u;
  }
}

}  // namespace nys

using namespace nys;

extern "C" {

int nys_filter_finish(const nys_filter_desc* d, const float* f, int64_t f_plane_stride, const float* guide,
                      int64_t guide_plane_stride, float* out, int64_t out_plane_stride, const void* workspace,
                      void* stats_out, void* stream) {
  int st = validate_tiled(d);
  if (st) return st;
  if (!f || !out || !workspace || (d->guide_kind == 0 && !guide)) return NYS_EINVAL;
  const FilterLayout L = filter_layout(d);
  RArgs a;
  memset(&a, 0, sizeof(a));
  a.f = f;
  a.g = d->guide_kind == 0 ? guide : f;
  a.out = out;
  a.fps = f_plane_stride;
  a.gps = d->guide_kind == 0 ? guide_plane_stride : f_plane_stride;
  a.ops = out_plane_stride;
  a.n = d->n;
  a.rho = d->rho;
  a.H = d->H;
  a.W = d->W;
  a.m0 = d->m0;
  a.R = d->radius;
  a.gkind = d->guide_kind;
  a.out64 = d->out_f64 != 0;
  a.rlo = std::max(0, d->row_lo);
  a.rhi = d->row_hi > 0 ? std::min(d->H, d->row_hi) : d->H;
  const char* ws = static_cast<const char*>(workspace);
  a.D = reinterpret_cast<const double*>(ws + L.off_D * sizeof(float));
  a.M64 = reinterpret_cast<const double*>(ws + L.m64_off_bytes);
  a.list = reinterpret_cast<const unsigned*>(ws + L.list_off_bytes);
  a.cap = L.list_cap;
  a.chunk_cnt = reinterpret_cast<unsigned*>(const_cast<char*>(ws) + L.cnt_off_bytes);
  a.part = reinterpret_cast<double*>(const_cast<char*>(ws) + L.part_off_bytes);
  {
    const int NP = (2 * d->radius + 1) * (2 * d->radius + 1);
    a.nch = std::max(1, std::min(kRefineChunks, (NP + RF_THREADS - 1) / RF_THREADS));
  }
  a.d_u0 = (int)L.d_U064;
  a.d_sc = (int)L.d_SC64;
  a.stats = reinterpret_cast<FilterStats*>(const_cast<char*>(ws) + L.stats_off_bytes);
  a.stats_out = static_cast<double*>(stats_out);
  a.inv = 1.0 / (2.0 * d->theta * d->theta);
  const int T = 2 * d->radius + 1;
  for (int t = 0; t < NYS_MAX_TAPS; ++t) a.taps[t] = 0.0;
  for (int t = 0; t < T; ++t) {
    const double u = (double)(t - d->radius);
    a.taps[t] = d->spatial_kind == NYS_SPATIAL_BOX ? 1.0 : std::exp(-(u * u) / (2.0 * d->sigma * d->sigma));
  }
  const size_t base = (size_t)(3 * d->m0 + d->rho + 2 * RF_THREADS + 2 * (d->n + 1)) * sizeof(double) +
                      RF_THREADS * sizeof(int) + (size_t)d->rho * RF_THREADS * sizeof(float);
  const size_t csz = (size_t)d->m0 * d->rho * sizeof(double);
  a.c_in_smem = base + csz <= 160 * 1024;
  const size_t smem = base + (a.c_in_smem ? csz : 0);
  if (smem > 227 * 1024) return NYS_EUNSUPPORTED;
  NYS_CUDA_TRY(cudaFuncSetAttribute(k_finish, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  count_launch();
  k_finish<<<2 * num_sms(), RF_THREADS, smem, (cudaStream_t)stream>>>(a);
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

}  // extern "C"
