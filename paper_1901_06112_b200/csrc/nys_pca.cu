// PCA patch guide: the NLM guide with pca_dim < n(2r+1)^2.
//
// Reference region replaced: filters.py:161-187 (pca_patch_guide):
//   X[p, :]  = the (2r+1)^2 patch of every channel at pixel p, channel-major,
//              then dy, then dx, edge replicate (filters.py:174-181)
//   mu       = X.mean(0);  Xc = X - mu
//   cov      = Xc^T Xc / m   (SymMatrix)  -> jacobi_eig (host, m x m tiny)
//   guide    = Xc @ V[:, :pca_dim], planar (pca_dim, H, W)
// The patch matrix X is never stored: every kernel gathers patches from the
// image (L1/L2-resident neighbourhoods).
//   P0 k_patch_sums   per-dimension sums (FP64, deterministic block partials)
//   P1 k_patch_gram   centred Gram matrix in FP64: each thread owns a 4x4
//                     register tile of the upper triangle, CTAs stage 32-pixel
//                     chunks of centred patches in shared memory
//   P2 k_sum_splits   fixed-order reduction of the per-CTA partials
//   (host: eigendecomposition + sign convention, paper_1901_06112_b200/pca.py)
//   P3 k_pca_project  per pixel: centred patch (shared memory) x V[:, :k]
#include "nys_filter_common.cuh"

namespace nys {

constexpr int PC_THREADS = 256;
constexpr int PC_CHUNK = 32;  // pixels staged per step
constexpr int PC_MAXDIM = 1024;  // e.g. 31 bands x 5x5 patches = 775

__device__ __forceinline__ float patch_at(const float* __restrict__ f, long long fps, int side, int r, int d,
                                          int y, int x, int H, int W) {
  const int s2 = side * side, c = d / s2, k = d - c * s2, dy = k / side - r, dx = k - (k / side) * side - r;
  return __ldg(f + (long long)c * fps + (long long)clampi(y + dy, 0, H - 1) * W + clampi(x + dx, 0, W - 1));
}

// partial[blockIdx.x][d] = Σ over this CTA's pixels of patch coordinate d
__global__ void __launch_bounds__(PC_THREADS) k_patch_sums(const float* __restrict__ f, long long fps, int side,
                                                           int r, int dim, int H, int W, long long per_block,
                                                           double* __restrict__ partial) {
  extern __shared__ float xsum[];  // [PC_CHUNK][dim]
  float* xs = xsum;
  const long long npx = (long long)H * W;
  const long long p0 = (long long)blockIdx.x * per_block, p1 = min(npx, p0 + per_block);
  double acc[PC_MAXDIM / PC_THREADS] = {};  // coordinates threadIdx.x + k * PC_THREADS
  for (long long c0 = p0; c0 < p1; c0 += PC_CHUNK) {
    const int cnt = (int)min((long long)PC_CHUNK, p1 - c0);
    for (int k = threadIdx.x; k < cnt * dim; k += blockDim.x) {
      const int i = k / dim, d = k - i * dim;
      const long long p = c0 + i;
      const int y = (int)(p / W), x = (int)(p - (long long)y * W);
      xs[i * dim + d] = patch_at(f, fps, side, r, d, y, x, H, W);
    }
    __syncthreads();
    for (int dd = threadIdx.x; dd < dim; dd += blockDim.x) {  // coordinate dd: this thread's running sum
      double v = 0.0;
      for (int i = 0; i < cnt; ++i) v += (double)xs[i * dim + dd];
      acc[dd / PC_THREADS] += v;
    }
    __syncthreads();
  }
  for (int dd = threadIdx.x; dd < dim; dd += blockDim.x) partial[(long long)blockIdx.x * dim + dd] = acc[dd / PC_THREADS];
}

// upper-triangle 4x4 tile t -> (ti, tj), ti <= tj, row-major over ti
__device__ __forceinline__ void tile_of(int t, int nt, int& ti, int& tj) {
  ti = 0;
  while (t >= nt - ti) {
    t -= nt - ti;
    ++ti;
  }
  tj = ti + t;
}

// partial[blockIdx.x][tile][16] = Σ over this CTA's pixels of the centred
// outer-product tile; blockIdx.y selects 256 tiles
__global__ void __launch_bounds__(PC_THREADS) k_patch_gram(const float* __restrict__ f, long long fps, int side,
                                                           int r, int dim, int H, int W, long long per_block,
                                                           const double* __restrict__ mu, int ntiles, int chunk,
                                                           double* __restrict__ partial) {
  extern __shared__ double xs[];  // [chunk][dimp]
  const int dimp = (dim + 3) & ~3, nt = dimp / 4;
  const int t = blockIdx.y * PC_THREADS + threadIdx.x;
  const bool active = t < ntiles;
  int ti = 0, tj = 0;
  if (active) tile_of(t, nt, ti, tj);
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  const long long npx = (long long)H * W;
  const long long p0 = (long long)blockIdx.x * per_block, p1 = min(npx, p0 + per_block);
  for (long long c0 = p0; c0 < p1; c0 += chunk) {
    const int cnt = (int)min((long long)chunk, p1 - c0);
    for (int k = threadIdx.x; k < chunk * dimp; k += blockDim.x) {
      const int i = k / dimp, d = k - i * dimp;
      double v = 0.0;
      if (i < cnt && d < dim) {
        const long long p = c0 + i;
        const int y = (int)(p / W), x = (int)(p - (long long)y * W);
        v = (double)patch_at(f, fps, side, r, d, y, x, H, W) - mu[d];
      }
      xs[i * dimp + d] = v;
    }
    __syncthreads();
    if (active) {
      for (int i = 0; i < cnt; ++i) {
        const double2 a01 = *reinterpret_cast<const double2*>(xs + i * dimp + 4 * ti);
        const double2 a23 = *reinterpret_cast<const double2*>(xs + i * dimp + 4 * ti + 2);
        const double2 b01 = *reinterpret_cast<const double2*>(xs + i * dimp + 4 * tj);
        const double2 b23 = *reinterpret_cast<const double2*>(xs + i * dimp + 4 * tj + 2);
        const double av[4] = {a01.x, a01.y, a23.x, a23.y}, bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
      }
    }
    __syncthreads();
  }
  if (active) {
    double* dst = partial + ((long long)blockIdx.x * ntiles + t) * 16;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) dst[a * 4 + b] = acc[a][b];
  }
}

// out[e] = scale * Σ_s partial[s][e], s in order
__global__ void k_sum_splits(const double* __restrict__ partial, int nsplit, long long len, double scale,
                             double* __restrict__ out) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < len; e += (long long)gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int s = 0; s < nsplit; ++s) t += partial[(long long)s * len + e];
    out[e] = t * scale;
  }
}

// guide[k][p] = Σ_d (patch_d(p) - mu_d) V[d][k], k < kdim
__global__ void __launch_bounds__(128) k_pca_project(const float* __restrict__ f, long long fps, int side, int r,
                                                     int dim, int H, int W, const float* __restrict__ mu,
                                                     const float* __restrict__ V /*[dim][kdim]*/, int kdim,
                                                     float* __restrict__ out, long long ops) {
  extern __shared__ float xc[];  // [dim][blockDim]
  const int BT = blockDim.x;
  const long long npx = (long long)H * W;
  const long long p = (long long)blockIdx.x * BT + threadIdx.x;
  if (p >= npx) return;
  const int y = (int)(p / W), x = (int)(p - (long long)y * W);
  for (int d = 0; d < dim; ++d) xc[d * BT + threadIdx.x] = patch_at(f, fps, side, r, d, y, x, H, W) - __ldg(mu + d);
  for (int k0 = 0; k0 < kdim; k0 += 4) {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    for (int d = 0; d < dim; ++d) {
      const float v = xc[d * BT + threadIdx.x];
      const float* vr = V + (long long)d * kdim + k0;
      a0 = fmaf(v, __ldg(vr), a0);
      if (k0 + 1 < kdim) a1 = fmaf(v, __ldg(vr + 1), a1);
      if (k0 + 2 < kdim) a2 = fmaf(v, __ldg(vr + 2), a2);
      if (k0 + 3 < kdim) a3 = fmaf(v, __ldg(vr + 3), a3);
    }
    out[(long long)k0 * ops + p] = a0;
    if (k0 + 1 < kdim) out[(long long)(k0 + 1) * ops + p] = a1;
    if (k0 + 2 < kdim) out[(long long)(k0 + 2) * ops + p] = a2;
    if (k0 + 3 < kdim) out[(long long)(k0 + 3) * ops + p] = a3;
  }
}

inline int pca_ntiles(int dim);
inline int pca_splits(long long npx, int dim) {
  const long long cap = pca_ntiles(dim) > 4096 ? 32 : 2 * num_sms();  // bound the partials for large patches
  return (int)std::max<long long>(1, std::min<long long>(cap, ceil_div(npx, 256)));
}
inline int pca_ntiles(int dim) {
  const int nt = (int)ceil_div(dim, 4);
  return nt * (nt + 1) / 2;
}

}  // namespace nys

using namespace nys;

extern "C" {

size_t nys_patch_moments_workspace_bytes(int n, int H, int W, int r) {
  const int dim = n * (2 * r + 1) * (2 * r + 1);
  if (n < 1 || r < 0 || dim > PC_MAXDIM || H < 1 || W < 1) return 0;
  const int ns = pca_splits((long long)H * W, dim);
  return (size_t)ns * ((size_t)pca_ntiles(dim) * 16 + dim) * sizeof(double);
}

int nys_patch_moments(const float* f, int64_t f_plane_stride, int n, int H, int W, int r, double* mean_out,
                      double* gram_tiles_out, void* workspace, size_t workspace_bytes, void* stream) {
  const int side = 2 * r + 1, dim = n * side * side;
  if (!f || !mean_out || !gram_tiles_out || !workspace || n < 1 || r < 0 || H < 1 || W < 1) return NYS_EINVAL;
  if (dim > PC_MAXDIM) return NYS_EUNSUPPORTED;
  if (workspace_bytes < nys_patch_moments_workspace_bytes(n, H, W, r)) return NYS_EINVAL;
  const long long npx = (long long)H * W;
  const int ns = pca_splits(npx, dim);
  const long long per = ceil_div(npx, ns);
  const int ntiles = pca_ntiles(dim);
  double* part = static_cast<double*>(workspace);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t smem_s = (size_t)PC_CHUNK * dim * sizeof(float);
  NYS_CUDA_TRY(cudaFuncSetAttribute(k_patch_sums, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_s));
  count_launch();
  k_patch_sums<<<ns, PC_THREADS, smem_s, s>>>(f, f_plane_stride, side, r, dim, H, W, per, part);
  NYS_LAUNCH_CHECK();
  count_launch();
  k_sum_splits<<<1, 256, 0, s>>>(part, ns, dim, 1.0 / (double)npx, mean_out);
  NYS_LAUNCH_CHECK();
  const int gchunk = (int)std::max<size_t>(1, std::min<size_t>(PC_CHUNK, (200 * 1024) / (((size_t)dim + 3) / 4 * 4 * 8)));
  const size_t smem = (size_t)gchunk * ((dim + 3) & ~3) * sizeof(double);
  NYS_CUDA_TRY(cudaFuncSetAttribute(k_patch_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  count_launch();
  k_patch_gram<<<dim3(ns, (unsigned)ceil_div(ntiles, PC_THREADS)), PC_THREADS, smem, s>>>(
      f, f_plane_stride, side, r, dim, H, W, per, mean_out, ntiles, gchunk, part);
  NYS_LAUNCH_CHECK();
  count_launch();
  k_sum_splits<<<(unsigned)ceil_div((long long)ntiles * 16, 256), 256, 0, s>>>(part, ns, (long long)ntiles * 16, 1.0,
                                                                             gram_tiles_out);
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

int nys_pca_project(const float* f, int64_t f_plane_stride, int n, int H, int W, int r, const float* mean,
                    const float* basis, int pca_dim, float* out, int64_t out_plane_stride, void* stream) {
  const int side = 2 * r + 1, dim = n * side * side;
  if (!f || !mean || !basis || !out || n < 1 || r < 0 || H < 1 || W < 1 || pca_dim < 1 || pca_dim > dim)
    return NYS_EINVAL;
  if (dim > PC_MAXDIM) return NYS_EUNSUPPORTED;
  const int bt = std::max(32, std::min(128, (int)((200 * 1024) / ((size_t)dim * 4)) & ~31));  // patch rows in SMEM
  const size_t smem = (size_t)dim * bt * sizeof(float);
  NYS_CUDA_TRY(cudaFuncSetAttribute(k_pca_project, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  count_launch();
  k_pca_project<<<(unsigned)ceil_div((long long)H * W, bt), bt, smem, (cudaStream_t)stream>>>(
      f, f_plane_stride, side, r, dim, H, W, mean, basis, pca_dim, out, out_plane_stride);
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

}  // extern "C"
