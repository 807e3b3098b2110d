// Image quality metrics on the device: per-plane sums of
// squared differences (MSE / PSNR) and single-scale SSIM.
//
// Reference region replaced: metrics.py:37-122.
//   mse  = mean((a - b)^2) over every sample (metrics.py:37-40)
//   psnr = 10 log10(R^2 / mse), per band or global, capped at 99 dB (host)
//   ssim = per plane: 11x11 Gaussian window (sigma 1.5, normalised), C1 =
//          (0.01 R)^2, C2 = (0.03 R)^2, evaluated where the whole window fits,
//          averaged over positions and then over planes; planes smaller than
//          the window use whole-plane statistics (metrics.py:74-108).
// Everything accumulates in FP64 like the reference; the inputs may be
// float32 or float64 planes.  Reductions are deterministic: fixed per-block
// partials, then one fixed-order pass.
#include "nys_filter_common.cuh"

namespace nys {

constexpr int QM_THREADS = 256;
constexpr int QM_BLOCKS = 592;  // 4 x 148 SMs
constexpr int SSIM_WIN = 11;

template <typename T>
__device__ __forceinline__ double ld(const void* p, long long i) {
  return (double)__ldg(static_cast<const T*>(p) + i);
}

__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
  __syncthreads();
  return t;
}

// partial[c * gridDim.x + block] = Σ over this block's samples of plane c
template <typename T>
__global__ void __launch_bounds__(QM_THREADS) k_sq_diff(const void* a, long long aps, const void* b, long long bps,
                                                        long long npx, double* partial) {
  __shared__ double sh[32];
  const int c = blockIdx.y;
  double acc = 0.0;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < npx; p += (long long)gridDim.x * blockDim.x) {
    const double d = ld<T>(a, c * aps + p) - ld<T>(b, c * bps + p);
    acc = fma(d, d, acc);
  }
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) partial[(long long)c * gridDim.x + blockIdx.x] = t;
}

struct SsimConsts {
  double w[SSIM_WIN * SSIM_WIN];
  double c1, c2;
};

// mean of the SSIM map over the valid positions of plane blockIdx.y
template <typename T>
__global__ void __launch_bounds__(QM_THREADS) k_ssim_map(const void* a, long long aps, const void* b, long long bps,
                                                         int H, int W, const SsimConsts k, double* partial) {
  __shared__ double sh[32];
  const int c = blockIdx.y;
  const int Hv = H - SSIM_WIN + 1, Wv = W - SSIM_WIN + 1;
  const long long nv = (long long)Hv * Wv;
  double acc = 0.0;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (long long)gridDim.x * blockDim.x) {
    const int y = (int)(v / Wv), x = (int)(v - (long long)y * Wv);
    double mx = 0, my = 0, xx = 0, yy = 0, xy = 0;
    for (int dy = 0; dy < SSIM_WIN; ++dy) {
      const long long r = (long long)(y + dy) * W + x;
#pragma unroll
      for (int dx = 0; dx < SSIM_WIN; ++dx) {
        const double wv = k.w[dy * SSIM_WIN + dx];
        const double xs = ld<T>(a, c * aps + r + dx), ys = ld<T>(b, c * bps + r + dx);
        mx = fma(wv, xs, mx);
        my = fma(wv, ys, my);
        xx = fma(wv * xs, xs, xx);
        yy = fma(wv * ys, ys, yy);
        xy = fma(wv * xs, ys, xy);
      }
    }
    const double vx = xx - mx * mx, vy = yy - my * my, cv = xy - mx * my;
    acc += ((2 * mx * my + k.c1) * (2 * cv + k.c2)) / ((mx * mx + my * my + k.c1) * (vx + vy + k.c2));
  }
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) partial[(long long)c * gridDim.x + blockIdx.x] = t;
}

// whole-plane statistics for planes smaller than the window (metrics.py:78-86)
template <typename T>
__global__ void __launch_bounds__(QM_THREADS) k_ssim_global(const void* a, long long aps, const void* b,
                                                            long long bps, long long npx, double c1, double c2,
                                                            double* out) {
  __shared__ double sh[32];
  __shared__ double mu[2];
  const int c = blockIdx.x;
  double sx = 0, sy = 0;
  for (long long p = threadIdx.x; p < npx; p += blockDim.x) {
    sx += ld<T>(a, c * aps + p);
    sy += ld<T>(b, c * bps + p);
  }
  sx = block_sum(sx, sh);
  sy = block_sum(sy, sh);
  if (threadIdx.x == 0) {
    mu[0] = sx / (double)npx;
    mu[1] = sy / (double)npx;
  }
  __syncthreads();
  const double mx = mu[0], my = mu[1];
  double vx = 0, vy = 0, cv = 0;
  for (long long p = threadIdx.x; p < npx; p += blockDim.x) {
    const double dx = ld<T>(a, c * aps + p) - mx, dy = ld<T>(b, c * bps + p) - my;
    vx = fma(dx, dx, vx);
    vy = fma(dy, dy, vy);
    cv = fma(dx, dy, cv);
  }
  vx = block_sum(vx, sh) / (double)npx;
  vy = block_sum(vy, sh) / (double)npx;
  cv = block_sum(cv, sh) / (double)npx;
  if (threadIdx.x == 0)
    out[c] = ((2 * mx * my + c1) * (2 * cv + c2)) / ((mx * mx + my * my + c1) * (vx + vy + c2));
}

// out[c] = scale * Σ_b partial[c][b] in block order
__global__ void k_sum_partials(const double* partial, int nblocks, double scale, double* out) {
  const int c = blockIdx.x;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int b = 0; b < nblocks; ++b) t += partial[(long long)c * nblocks + b];
    out[c] = t * scale;
  }
}

template <typename T>
int quality_impl(const void* a, int64_t aps, const void* b, int64_t bps, int n, int H, int W, double range_max,
                 double* sq, double* ssim, double* ws, cudaStream_t s) {
  const long long npx = (long long)H * W;
  count_launch();
  k_sq_diff<T><<<dim3(QM_BLOCKS, n), QM_THREADS, 0, s>>>(a, aps, b, bps, npx, ws);
  NYS_LAUNCH_CHECK();
  count_launch();
  k_sum_partials<<<n, 32, 0, s>>>(ws, QM_BLOCKS, 1.0, sq);
  NYS_LAUNCH_CHECK();
  if (!ssim) return NYS_OK;
  const double c1 = (0.01 * range_max) * (0.01 * range_max), c2 = (0.03 * range_max) * (0.03 * range_max);
  if (H < SSIM_WIN || W < SSIM_WIN) {
    count_launch();
    k_ssim_global<T><<<n, QM_THREADS, 0, s>>>(a, aps, b, bps, npx, c1, c2, ssim);
    NYS_LAUNCH_CHECK();
    return NYS_OK;
  }
  SsimConsts k;
  double w1[SSIM_WIN], tot = 0.0;
  for (int t = 0; t < SSIM_WIN; ++t) {
    const double u = (double)(t - SSIM_WIN / 2);
    w1[t] = std::exp(-(u * u) / (2.0 * 1.5 * 1.5));
  }
  for (int i = 0; i < SSIM_WIN; ++i)
    for (int j = 0; j < SSIM_WIN; ++j) tot += w1[i] * w1[j];
  for (int i = 0; i < SSIM_WIN; ++i)
    for (int j = 0; j < SSIM_WIN; ++j) k.w[i * SSIM_WIN + j] = (w1[i] * w1[j]) / tot;
  k.c1 = c1;
  k.c2 = c2;
  const long long nv = (long long)(H - SSIM_WIN + 1) * (W - SSIM_WIN + 1);
  count_launch();
  k_ssim_map<T><<<dim3(QM_BLOCKS, n), QM_THREADS, 0, s>>>(a, aps, b, bps, H, W, k, ws);
  NYS_LAUNCH_CHECK();
  count_launch();
  k_sum_partials<<<n, 32, 0, s>>>(ws, QM_BLOCKS, 1.0 / (double)nv, ssim);
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

}  // namespace nys

using namespace nys;

extern "C" {

size_t nys_quality_workspace_bytes(int n) { return (size_t)(n > 0 ? n : 1) * QM_BLOCKS * sizeof(double); }

int nys_quality_planes(const void* a, int64_t a_plane_stride, const void* b, int64_t b_plane_stride, int elem_bytes,
                       int n, int H, int W, double range_max, double* sq_sums_out, double* ssim_out, void* workspace,
                       size_t workspace_bytes, void* stream) {
  if (!a || !b || !sq_sums_out || !workspace || n < 1 || H < 1 || W < 1) return NYS_EINVAL;
  if (elem_bytes != 4 && elem_bytes != 8) return NYS_EINVAL;
  if (workspace_bytes < nys_quality_workspace_bytes(n)) return NYS_EINVAL;
  if (n > 65535) return NYS_EUNSUPPORTED;
  cudaStream_t s = (cudaStream_t)stream;
  double* ws = static_cast<double*>(workspace);
  return elem_bytes == 4
             ? quality_impl<float>(a, a_plane_stride, b, b_plane_stride, n, H, W, range_max, sq_sums_out, ssim_out, ws, s)
             : quality_impl<double>(a, a_plane_stride, b, b_plane_stride, n, H, W, range_max, sq_sums_out, ssim_out, ws, s);
}

}  // extern "C"
