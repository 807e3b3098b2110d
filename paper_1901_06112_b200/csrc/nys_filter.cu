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
// pixel.  K2 evaluates b and y per source pixel (a register-blocked
// [px x m0] x [m0 x (m0+1)] product, the extra column being the lead
// projection s0 = w_1.b) and runs the horizontal pass of the (m0+1)(n+1)
// planes y_i f_c, y_i.  K3 TMA-stages tiles of those planes, runs the vertical
// pass, contracts with b_i(x) recomputed at the centre pixel, and applies the
// guard and division.  Only the horizontally filtered planes touch HBM.
//
// Plane buffer layout: plane p = i*(n+1) + c, each plane `rows + 2R` virtual
// rows of pitch Wp = roundup(W, 4) floats; virtual row v maps to image row
// clamp(v, 0, H-1), so K3 never clamps (replicate borders, spatial.py:85-88).
#include "nys_filter_common.cuh"

namespace nys {

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

// M = A^{-1} = L^{-T} L^{-1} from the host's Cholesky factor, FP64, into the FP32
// [M | u0]^T block (MT[j][i] = M[i][j]); one CTA, n <= 90 (L and X in shared memory)
__global__ void __launch_bounds__(1024) k_inverse_cholesky(const double* __restrict__ Lg, int n, float* __restrict__ MT,
                                                          int m0q) {
  extern __shared__ double cs[];
  double* Ls = cs;          // n x n
  double* X = cs + n * n;   // n x n, X = L^{-1} (lower)
  for (int k = threadIdx.x; k < n * n; k += blockDim.x) {
    Ls[k] = Lg[k];
    X[k] = 0.0;
  }
  __syncthreads();
  if ((int)threadIdx.x < n) {  // column j of L^{-1} by forward substitution
    const int j = threadIdx.x;
    X[j * n + j] = 1.0 / Ls[j * n + j];
    for (int i = j + 1; i < n; ++i) {
      double t = 0.0;
      for (int k = j; k < i; ++k) t = fma(Ls[i * n + k], X[k * n + j], t);
      X[i * n + j] = -t / Ls[i * n + i];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    double t = 0.0;
    for (int k = max(i, j); k < n; ++k) t = fma(X[k * n + i], X[k * n + j], t);
    MT[(size_t)j * m0q + i] = (float)t;
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

}  // namespace nys

using namespace nys;

extern "C" {

size_t nys_filter_planes_bytes(const nys_filter_desc* d, int rows) {
  if (validate_tiled(d) != NYS_OK) return 0;
  return (size_t)(rows + 2 * d->radius) * (size_t)plane_row_stride(d->W, buffer_planes(d)) * sizeof(float);
}

int64_t nys_filter_plane_row_stride(const nys_filter_desc* d) {
  if (validate_tiled(d) != NYS_OK) return 0;
  return plane_row_stride(d->W, buffer_planes(d));
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
  for (int j = 0; j < d->m0; ++j)
    for (int k = 0; k < d->rho; ++k) h[L.off_C + (size_t)j * L.rhop + k] = (float)d->centroids[(size_t)j * d->rho + k];
  const bool chol = d->M_is_cholesky != 0;
  if (chol && (d->phi_form || d->m0 > 90)) return NYS_EINVAL;
  for (int j = 0; j < d->m0; ++j) {
    if (!chol)
      for (int i = 0; i < d->m0; ++i) h[L.off_MT + (size_t)j * L.m0q + i] = (float)d->M[(size_t)i * d->m0 + j];
    h[L.off_MT + (size_t)j * L.m0q + d->m0] = (float)d->u0[j];
    // K3 forms s0 = U0 . (stored feature planes): u0 . b, or sqrt(alpha_1) phi_0 in the phi-form
    h[L.off_U0 + j] = d->phi_form ? (j == 0 ? (float)std::sqrt(d->alpha0) : 0.f) : (float)d->u0[j];
  }
  cudaStream_t s = (cudaStream_t)stream;
  // pageable H2D: the runtime stages `h` before returning, so it may go away
  // right after (no stream synchronisation: the caller keeps queueing work)
  NYS_CUDA_TRY(cudaMemcpyAsync(workspace, h.data(), L.n_floats * sizeof(float), cudaMemcpyHostToDevice, s));
  if (chol) {  // M = A^{-1} from the Cholesky factor, on the device (after the block above lands)
    double* Ld = reinterpret_cast<double*>((char*)workspace + L.chol_off_bytes);
    NYS_CUDA_TRY(cudaMemcpyAsync(Ld, d->M, (size_t)d->m0 * d->m0 * sizeof(double), cudaMemcpyHostToDevice, s));
    const size_t smem = 2 * (size_t)d->m0 * d->m0 * sizeof(double);
    NYS_CUDA_TRY(cudaFuncSetAttribute(k_inverse_cholesky, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    count_launch();
    k_inverse_cholesky<<<1, 1024, smem, s>>>(Ld, d->m0, static_cast<float*>(workspace) + L.off_MT, L.m0q);
    NYS_LAUNCH_CHECK();
  }
  count_launch();
  k_reset_stats<<<1, 1, 0, s>>>(reinterpret_cast<FilterStats*>((char*)workspace + L.stats_off_bytes));
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

int nys_filter_stats(const nys_filter_desc* d, const void* workspace, void* stats_out, void* stream) {
  int st = validate(d);
  if (st) return st;
  if (!workspace || !stats_out) return NYS_EINVAL;
  const FilterLayout L = filter_layout(d);
  count_launch();
  k_copy_stats<<<1, 1, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const FilterStats*>((const char*)workspace + L.stats_off_bytes),
      reinterpret_cast<double*>(stats_out));
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

int nys_device_view(const void* p, void** device_ptr_out) {
  if (!p || !device_ptr_out) return NYS_EINVAL;
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return NYS_EINVAL;
  }
  if (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged) {
    *device_ptr_out = const_cast<void*>(p);
    return NYS_OK;
  }
  if (attr.type == cudaMemoryTypeHost && attr.devicePointer) {
    // attr describes the allocation's base: keep p's offset within it
    *device_ptr_out = static_cast<char*>(attr.devicePointer) +
                      (static_cast<const char*>(p) - static_cast<const char*>(attr.hostPointer));
    return NYS_OK;
  }
  return NYS_EINVAL;
}

int nys_patch_guide(const float* f, int64_t f_plane_stride, int n, int H, int W, int r, float* out,
                    int64_t out_plane_stride, void* stream) {
  if (!f || !out || n < 1 || H < 1 || W < 1 || r < 0) return NYS_EINVAL;
  const long long total = (long long)H * W * n * (2 * r + 1) * (2 * r + 1);
  const int grid = (int)std::min<long long>(ceil_div(total, 256), (long long)num_sms() * 16);
  count_launch();
  k_patch_guide<<<grid, 256, 0, (cudaStream_t)stream>>>(f, f_plane_stride, n, H, W, r, out, out_plane_stride);
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

}  // extern "C"
