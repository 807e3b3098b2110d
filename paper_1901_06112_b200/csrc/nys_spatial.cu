// Stand-alone separable spatial filters on FP64 plane stacks (the reference's
// public spatial.py API: apply_planes, box_filter, gaussian_fir,
// gaussian_recursive; spatial.py:91-109, 149-234).
//
// Row pass then column pass with edge-replicate borders, in FP64 like the
// reference (these are utility entry points, not the filter's hot path, which
// fuses the passes into K2/K3 / R1-R4):
//   box / FIR   one thread per output sample, taps from the kernel parameters
//               (the box is the unnormalised (2S+1)-sum; the reference's cumsum
//               difference equals it up to FP64 rounding);
//   recursive   one thread per (plane, row) then per (plane, column): the
//               fifth-order causal + anticausal recursion of _vyv_scan, then the
//               squared truncated-FIR mass; sigma < 1 is the FIR at ceil(3 sigma).
#include "nys_filter_common.cuh"

namespace nys {

struct SpTaps {
  double w[NYS_MAX_TAPS];
};

// out[p][y][x] = sum_t w[t] in[p][y][clamp(x - R + t)]   (rows == 1)  or along y (rows == 0)
__global__ void k_sp_fir(const double* __restrict__ in, double* __restrict__ out, long long P, int H, int W, int R,
                         int along_rows, const SpTaps tp) {
  const long long n = P * H * W;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const long long p = e / ((long long)H * W);
    const int rem = (int)(e - p * H * W), y = rem / W, x = rem - y * W;
    const double* base = in + p * H * W;
    double acc = 0.0;
    for (int t = 0; t <= 2 * R; ++t) {
      const double v = along_rows ? base[(long long)y * W + clampi(x - R + t, 0, W - 1)]
                                  : base[(long long)clampi(y - R + t, 0, H - 1) * W + x];
      acc = fma(tp.w[t], v, acc);
    }
    out[e] = acc;
  }
}

struct SpRec {
  double g, a1, a2, a3, a4, a5;
};

// causal then anticausal recursion along rows (along_rows) or columns, in place
__global__ void k_sp_rec(double* __restrict__ a, long long P, int H, int W, int along_rows, const SpRec c) {
  const long long lines = along_rows ? P * H : P * W;
  const long long li = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (li >= lines) return;
  const int N = along_rows ? W : H;
  const long long stride = along_rows ? 1 : W;
  double* base = along_rows ? a + li * W : a + (li / W) * (long long)H * W + (li % W);
  for (int pass = 0; pass < 2; ++pass) {
    const bool rev = pass == 1;
    double w1 = base[(rev ? N - 1 : 0) * stride], w2 = w1, w3 = w1, w4 = w1, w5 = w1;
    for (int i = 0; i < N; ++i) {
      const long long k = (long long)(rev ? N - 1 - i : i) * stride;
      const double cur = c.g * base[k] - (c.a1 * w1 + c.a2 * w2 + c.a3 * w3 + c.a4 * w4 + c.a5 * w5);
      base[k] = cur;
      w5 = w4;
      w4 = w3;
      w3 = w2;
      w2 = w1;
      w1 = cur;
    }
  }
}

__global__ void k_sp_scale(double* __restrict__ a, long long n, double s) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    a[e] *= s;
}

}  // namespace nys

using namespace nys;

extern "C" int nys_spatial_planes(const double* in, double* out, int64_t P, int H, int W, int kind, double sigma,
                                  int radius, double* scratch, void* stream) {
  if (!in || !out || P < 1 || H < 1 || W < 1) return NYS_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  const long long n = (long long)P * H * W;
  const int grid = (int)std::min<long long>(ceil_div(n, 256), (long long)num_sms() * 16);
  const bool rec = kind == NYS_SPATIAL_GAUSSIAN_RECURSIVE;
  if (rec && !(sigma > 0.0)) return NYS_EINVAL;
  if (rec && sigma >= 1.0) {
    double cf[6];
    const int st = nys_vyv_coeffs(sigma, cf);
    if (st) return st;
    const SpRec c{cf[0], cf[1], cf[2], cf[3], cf[4], cf[5]};
    NYS_CUDA_TRY(cudaMemcpyAsync(out, in, (size_t)n * 8, cudaMemcpyDeviceToDevice, s));
    count_launch();
    k_sp_rec<<<(unsigned)ceil_div((long long)P * H, 128), 128, 0, s>>>(out, P, H, W, 1, c);
    NYS_LAUNCH_CHECK();
    count_launch();
    k_sp_rec<<<(unsigned)ceil_div((long long)P * W, 128), 128, 0, s>>>(out, P, H, W, 0, c);
    NYS_LAUNCH_CHECK();
    const int Rm = (int)std::ceil(3.0 * sigma);
    double mass = 0.0;
    for (int t = -Rm; t <= Rm; ++t) mass += std::exp(-((double)t * t) / (2.0 * sigma * sigma));
    count_launch();
    k_sp_scale<<<grid, 256, 0, s>>>(out, n, mass * mass);
    NYS_LAUNCH_CHECK();
    return NYS_OK;
  }
  if (!scratch) return NYS_EINVAL;
  int R = radius;
  if (rec) R = (int)std::ceil(3.0 * sigma);  // sigma < 1: the FIR at ceil(3 sigma) (spatial.py:206-208)
  if (kind == NYS_SPATIAL_BOX) {
    if (R < 0) return NYS_EINVAL;
  } else if (kind == NYS_SPATIAL_GAUSSIAN_FIR || rec) {
    if (!(sigma > 0.0) || R < 1) return NYS_EINVAL;
  } else {
    return NYS_EINVAL;
  }
  if (R > NYS_MAX_RADIUS) return NYS_EUNSUPPORTED;
  SpTaps tp{};
  for (int t = 0; t <= 2 * R; ++t) {
    const double u = (double)(t - R);
    tp.w[t] = kind == NYS_SPATIAL_BOX ? 1.0 : std::exp(-(u * u) / (2.0 * sigma * sigma));  // spatial.py:72-75
  }
  count_launch();
  k_sp_fir<<<grid, 256, 0, s>>>(in, scratch, P, H, W, R, 1, tp);
  NYS_LAUNCH_CHECK();
  count_launch();
  k_sp_fir<<<grid, 256, 0, s>>>(scratch, out, P, H, W, R, 0, tp);
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}
