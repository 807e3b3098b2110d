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
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstddef>
#include <deque>
#include <mutex>
#include <thread>

#include "nys_filter_common.cuh"
#include "nys_inverse.cuh"
#include "nys_host_internal.h"

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

__global__ void k_reset_stats(FilterStats* s) { reset_filter_stats(reinterpret_cast<unsigned*>(s), false); }

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

int nys_filter_workspace_layout(const nys_filter_desc* d, int64_t* out) {
  if (!out || validate(d) != NYS_OK) return NYS_EINVAL;
  const FilterLayout L = filter_layout(d);
  const int64_t v[8] = {(int64_t)(L.off_D * sizeof(float)), (int64_t)L.stats_off_bytes, (int64_t)L.chol_off_bytes,
                        (int64_t)L.m64_off_bytes, (int64_t)L.list_off_bytes, (int64_t)L.cnt_off_bytes,
                        (int64_t)L.part_off_bytes, (int64_t)L.total_bytes};
  for (int k = 0; k < 8; ++k) out[k] = v[k];
  return NYS_OK;
}

}  // extern "C"

namespace {
// M = A^{-1} from the Cholesky factor (m0 <= 64): read at chol_off_bytes of the workspace,
// or -- img_src non-null -- of the mapped pinned image, which the kernel first copies into
// the workspace; then the statistics reset
int launch_inverse_and_reset(const nys_filter_desc* d, const FilterLayout& L, void* workspace, bool chol,
                             cudaStream_t s, const void* img_src = nullptr, const unsigned* gate = nullptr,
                             unsigned seq = 0, bool reset = true) {
  if (chol) {
    const char* base = img_src ? static_cast<const char*>(img_src) : static_cast<const char*>(workspace);
    const double* Ld = reinterpret_cast<const double*>(base + L.chol_off_bytes);
    static std::atomic<unsigned long long> attr_set{0};  // one bit per device
    int dev = 0;
    NYS_CUDA_TRY(cudaGetDevice(&dev));
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_set.load() & bit)) {
      NYS_CUDA_TRY(cudaFuncSetAttribute(k_inverse_cholesky, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)kInvSmemBytes));
      attr_set.fetch_or(bit);
    }
    count_launch();
    k_inverse_cholesky<<<1, 1024, kInvSmemBytes, s>>>(Ld, d->m0, static_cast<float*>(workspace) + L.off_MT, L.m0q,
                                                      reinterpret_cast<double*>((char*)workspace + L.m64_off_bytes),
                                                      static_cast<const float4*>(img_src),
                                                      static_cast<float4*>(workspace), (int)(L.n_floats / 4),
                                                      reinterpret_cast<unsigned*>((char*)workspace + L.stats_off_bytes),
                                                      gate, seq);
    NYS_LAUNCH_CHECK();
    return NYS_OK;  // the inverse kernel also reset the statistics
  }
  if (!reset) return NYS_OK;  // k_wait_gate reset them (keeping a gate-timeout mark)
  count_launch();
  k_reset_stats<<<1, 1, 0, s>>>(reinterpret_cast<FilterStats*>((char*)workspace + L.stats_off_bytes));
  NYS_LAUNCH_CHECK();
  return NYS_OK;
}

// ---------------------------------------------------------------------------
// In-stream plan (nys_filter_plan_async / nys_filter_prepare_join).  The pinned
// staging buffer starts with this job record; the workspace image follows at
// kStagingHeader bytes.
//
// Two pinned words in the job: the caller's stream writes `ready` (cuStreamWriteValue32)
// once the landmarks' copy has completed; a persistent native worker thread polls it
// with plain loads (no CUDA call: it never queues behind other driver users), runs the
// lite plan, fills the image and publishes `done`; the first kernel after the join (the
// device inverse) polls `done` itself (an active wait: a cuStreamWaitValue32 gate sometimes
// noticed it milliseconds late), then pulls the image in.  The worker
// depends only on work queued before the gate and always publishes `done` (with an
// error status on failure or a 60 s timeout), so the gate cannot deadlock.  A
// cudaLaunchHostFunc chain did the same with ~0.3 ms of dispatch latency.
// ---------------------------------------------------------------------------
constexpr size_t kStagingHeader = 512;
struct PlanJob {
  const double* centroids;
  int m0, rho, S, device;
  double theta, eps_drop, phi_cond;
  FilterLayout L;
  size_t image_bytes;
  nys_plan_result result;
  unsigned seq;
  volatile unsigned ready;  // written by the stream (cuStreamWriteValue32) once the landmarks landed
  volatile unsigned done;   // the stream waits for done >= seq
};
static_assert(sizeof(PlanJob) <= kStagingHeader, "plan job record outgrew its header");

void run_plan(PlanJob* j, const nys_plan_exec* ex) {
  const auto t0 = std::chrono::steady_clock::now();
  const int n = j->m0, rho = j->rho;
  const FilterLayout& L = j->L;
  float* img = reinterpret_cast<float*>(reinterpret_cast<char*>(j) + kStagingHeader);
  std::vector<double> info(n), Lc((size_t)n * n), u0(n);
  int rank = 0;
  const bool chol = n <= kInvN;  // else the host forms M and the image carries it
  const int rc = nys_mixing_plan_lite_ex(j->centroids, n, rho, j->theta, j->eps_drop, j->phi_cond, chol ? 1 : 0,
                                         info.data(), &rank, Lc.data(), u0.data(), ex);
  j->result.status = rc;
  j->result.rank = rc == NYS_OK ? n : 0;
  if (rc == NYS_OK) {
    const double a1 = info[0];
    j->result.alpha0 = a1;
    j->result.eps_den = 1e-12 * (double)((2 * j->S + 1) * (2 * j->S + 1)) * a1;  // filters.py:241-243
    for (int q = 0; q < n; ++q) {
      for (int k = 0; k < rho; ++k) img[L.off_C + (size_t)q * L.rhop + k] = (float)j->centroids[(size_t)q * rho + k];
      img[L.off_MT + (size_t)q * L.m0q + n] = (float)u0[q];
      img[L.off_U0 + q] = (float)u0[q];
    }
    img[L.off_SC] = (float)(1.0 / a1);
    img[L.off_SC + 1] = (float)j->result.eps_den;
    // FP64 constants of the near-guard refinement (nys_filter_finish)
    double* D = reinterpret_cast<double*>(img + L.off_D);
    std::memcpy(D + L.d_C64, j->centroids, (size_t)n * rho * sizeof(double));
    std::memcpy(D + L.d_U064, u0.data(), (size_t)n * sizeof(double));
    D[L.d_SC64] = 1.0 / a1;
    D[L.d_SC64 + 1] = j->result.eps_den;
    D[L.d_SC64 + 2] = a1;
    D[L.d_SC64 + 3] = 0.0;
    if (chol)
      std::memcpy(reinterpret_cast<char*>(img) + L.chol_off_bytes, Lc.data(), (size_t)n * n * sizeof(double));
    else {
      for (int q = 0; q < n; ++q)
        for (int i = 0; i < n; ++i) img[L.off_MT + (size_t)q * L.m0q + i] = (float)Lc[(size_t)i * n + q];
      std::memcpy(reinterpret_cast<char*>(img) + L.m64_off_bytes, Lc.data(), (size_t)n * n * sizeof(double));
    }
  }
  j->result.host_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
}

// One worker serves every host thread and stream.  It never blocks on one job: it scans its
// pending jobs and runs whichever has its landmarks (a job's `ready` word), so a job whose
// stream is stuck behind another job's device gate (e.g. a cooperative k-means launch that
// cannot start while another stream's k_inverse_cholesky spins on an SM) cannot hold up the
// plan that gate waits for.
class PlanWorker {
 public:
  PlanWorker() { std::thread([this] { loop(); }).detach(); }
  void post(PlanJob* j) {
    {
      std::lock_guard<std::mutex> g(mu_);
      q_.push_back(Pending{j, std::chrono::steady_clock::now()});
    }
    cv_.notify_one();
  }

 private:
  struct Pending {
    PlanJob* job;
    std::chrono::steady_clock::time_point posted;
  };
  void loop() {
    std::vector<Pending> mine;  // jobs taken from the queue, waiting for their landmarks
    for (;;) {
      {
        std::unique_lock<std::mutex> g(mu_);
        if (mine.empty()) cv_.wait(g, [this] { return !q_.empty(); });
        while (!q_.empty()) {
          mine.push_back(q_.front());
          q_.pop_front();
        }
      }
      bool ran = false;
      const auto now = std::chrono::steady_clock::now();
      for (size_t k = 0; k < mine.size();) {
        PlanJob* j = mine[k].job;
        const bool ready = j->ready == j->seq;  // plain load of a pinned word the stream writes
        const double us = std::chrono::duration<double, std::micro>(now - mine[k].posted).count();
        if (!ready && us <= 60e6) {
          ++k;
          continue;
        }
        std::atomic_thread_fence(std::memory_order_seq_cst);
        // sequential plan: a helper thread for the Gram rows / Cholesky (nys_plan_exec) made the
        // plan slower and erratic (76-133 us) where the host threads contend for cores
        if (ready) run_plan(j, nullptr);
        else j->result.status = NYS_ECUDA;  // the stream never got there (an error upstream)
        std::atomic_thread_fence(std::memory_order_seq_cst);
        j->done = j->seq;  // releases the device gate
        std::atomic_thread_fence(std::memory_order_seq_cst);
        mine.erase(mine.begin() + (long)k);
        ran = true;
      }
      // spin while a job is young, then back off
      if (!ran && !mine.empty()) {
        const double oldest =
            std::chrono::duration<double, std::micro>(now - mine.front().posted).count();
        if (oldest > 5000.0) std::this_thread::sleep_for(std::chrono::microseconds(20));
      }
    }
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<Pending> q_;
};

PlanWorker& plan_worker() {
  static PlanWorker* w = new PlanWorker();  // never destroyed: the thread outlives static teardown
  return *w;
}

typedef CUresult (*StreamWaitValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
StreamWaitValue32Fn write_value_fn() {  // cuStreamWriteValue32
  static StreamWaitValue32Fn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<StreamWaitValue32Fn>(p);
  }
  return fn;
}

size_t plan_image_bytes(const FilterLayout& L, int m0) { return L.m64_off_bytes + (size_t)m0 * m0 * sizeof(double); }
}  // namespace

extern "C" {

size_t nys_filter_plan_staging_bytes(const nys_filter_desc* d) {
  if (validate(d) != NYS_OK) return 0;
  return kStagingHeader + plan_image_bytes(filter_layout(d), d->m0);
}

int nys_filter_plan_async(const nys_filter_desc* d, const double* centroids, double eps_drop, double phi_cond,
                          void* staging, size_t staging_bytes, void* workspace, size_t workspace_bytes,
                          void* stream) {
  int st = validate(d);
  if (st) return st;
  if (!centroids || !staging || !workspace || !(phi_cond > 1.0)) return NYS_EINVAL;
  const FilterLayout L = filter_layout(d);
  if (staging_bytes < kStagingHeader + plan_image_bytes(L, d->m0) || workspace_bytes < L.total_bytes)
    return NYS_EINVAL;
  if (!write_value_fn()) return NYS_EUNSUPPORTED;
  void* dv = nullptr;  // the gate words must be device-visible (mapped pinned memory)
  if (nys_device_view(staging, &dv) != NYS_OK) return NYS_EINVAL;
  PlanJob* j = static_cast<PlanJob*>(staging);
  if (j->seq != j->done) {
    // the previous plan on this buffer is still pending (its caller stopped before its final
    // wait, e.g. on an exception): it depends only on GPU work queued before it, so wait
    const auto t0 = std::chrono::steady_clock::now();
    while (j->seq != j->done) {
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(60)) return NYS_EINVAL;
      std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
  }
  j->centroids = centroids;
  j->m0 = d->m0;
  j->rho = d->rho;
  j->S = d->radius;
  NYS_CUDA_TRY(cudaGetDevice(&j->device));
  j->theta = d->theta;
  j->eps_drop = eps_drop;
  j->phi_cond = phi_cond;
  j->L = L;
  j->image_bytes = plan_image_bytes(L, d->m0);
  j->result = nys_plan_result{NYS_ECUDA, 0, 0.0, 0.0, 0.0};  // overwritten by the worker
  j->seq = j->seq + 1;
  // stream-ordered: written (behind a memory fence) once the landmarks' copy has completed
  const CUdeviceptr ready = reinterpret_cast<CUdeviceptr>(dv) + offsetof(PlanJob, ready);
  if (write_value_fn()(reinterpret_cast<CUstream>(stream), ready, j->seq, 0) != CUDA_SUCCESS) {
    j->seq = j->seq - 1;
    return NYS_ECUDA;
  }
  plan_worker().post(j);
  return NYS_OK;
}

int nys_filter_prepare_join(const nys_filter_desc* d, void* staging, void* workspace, void* stream) {
  int st = validate(d);
  if (st) return st;
  if (!staging || !workspace) return NYS_EINVAL;
  const PlanJob* j = static_cast<const PlanJob*>(staging);
  if (j->m0 != d->m0) return NYS_EINVAL;
  void* dv = nullptr;
  if (nys_device_view(staging, &dv) != NYS_OK) return NYS_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  // the gate is polled by the first kernel after it (k_inverse_cholesky, or k_wait_gate when
  // the image carries M): an active wait notices the worker's `done` within a microsecond
  const unsigned* gate = reinterpret_cast<const unsigned*>(static_cast<const char*>(dv) + offsetof(PlanJob, done));
  const FilterLayout L = filter_layout(d);
  const char* img = static_cast<const char*>(dv) + kStagingHeader;
  if (d->m0 <= kInvN) return launch_inverse_and_reset(d, L, workspace, true, s, img, gate, j->seq);
  count_launch();
  k_wait_gate<<<1, 32, 0, s>>>(gate, j->seq, reinterpret_cast<unsigned*>((char*)workspace + L.stats_off_bytes));
  NYS_LAUNCH_CHECK();
  const char* src = static_cast<const char*>(staging) + kStagingHeader;
  NYS_CUDA_TRY(cudaMemcpyAsync(workspace, src, L.n_floats * sizeof(float), cudaMemcpyHostToDevice, s));
  NYS_CUDA_TRY(cudaMemcpyAsync((char*)workspace + L.m64_off_bytes, src + L.m64_off_bytes,
                               (size_t)d->m0 * d->m0 * sizeof(double), cudaMemcpyHostToDevice, s));
  return launch_inverse_and_reset(d, L, workspace, false, s, nullptr, nullptr, 0, /*reset=*/false);
}

int nys_filter_plan_result(const void* staging, nys_plan_result* out) {
  if (!staging || !out) return NYS_EINVAL;
  const PlanJob* j = static_cast<const PlanJob*>(staging);
  if (j->done != j->seq) return NYS_EINVAL;  // not finished
  std::atomic_thread_fence(std::memory_order_seq_cst);
  *out = j->result;
  return NYS_OK;
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
  if (chol && (d->phi_form || d->m0 > kInvN)) return NYS_EINVAL;
  for (int j = 0; j < d->m0; ++j) {
    if (!chol)
      for (int i = 0; i < d->m0; ++i) h[L.off_MT + (size_t)j * L.m0q + i] = (float)d->M[(size_t)i * d->m0 + j];
    h[L.off_MT + (size_t)j * L.m0q + d->m0] = (float)d->u0[j];
    // K3 forms s0 = U0 . (stored feature planes): u0 . b, or sqrt(alpha_1) phi_0 in the phi-form
    h[L.off_U0 + j] = d->phi_form ? (j == 0 ? (float)std::sqrt(d->alpha0) : 0.f) : (float)d->u0[j];
  }
  h[L.off_SC] = (float)(1.0 / d->alpha0);
  h[L.off_SC + 1] = (float)d->eps_den;
  {  // FP64 constants of the near-guard refinement (nys_filter_finish)
    double* D = reinterpret_cast<double*>(h.data() + L.off_D);
    std::memcpy(D + L.d_C64, d->centroids, (size_t)d->m0 * d->rho * sizeof(double));
    std::memcpy(D + L.d_U064, d->u0, (size_t)d->m0 * sizeof(double));
    D[L.d_SC64] = 1.0 / d->alpha0;
    D[L.d_SC64 + 1] = d->eps_den;
    D[L.d_SC64 + 2] = d->alpha0;
    D[L.d_SC64 + 3] = 0.0;
  }
  cudaStream_t s = (cudaStream_t)stream;
  // one upload: the float block, the stats slot (reset below), the Cholesky factor (FP64 at
  // chol_off_bytes) and M64 -- which the device inverse forms itself from the factor
  h.resize((L.m64_off_bytes + (size_t)d->m0 * d->m0 * sizeof(double)) / sizeof(float), 0.f);
  if (chol) std::memcpy(reinterpret_cast<char*>(h.data()) + L.chol_off_bytes, d->M, (size_t)d->m0 * d->m0 * sizeof(double));
  else {
    const int m = d->m0;
    double* M64 = reinterpret_cast<double*>(reinterpret_cast<char*>(h.data()) + L.m64_off_bytes);
    if (!d->phi_form) {
      std::memcpy(M64, d->M, (size_t)m * m * sizeof(double));
    } else {  // eta = sum_y w phi(x).phi(y) = b(x)^T (P^T P) b(y)
      for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) {
          double acc = 0.0;
          for (int k = 0; k < m; ++k) acc += d->M[(size_t)k * m + i] * d->M[(size_t)k * m + j];
          M64[(size_t)i * m + j] = acc;
        }
    }
  }
  // pageable H2D: the runtime stages `h` before returning, so it may go away
  // right after (no stream synchronisation: the caller keeps queueing work); the
  // stats block it overwrites is reset below
  NYS_CUDA_TRY(cudaMemcpyAsync(workspace, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice, s));
  return launch_inverse_and_reset(d, L, workspace, chol, s);
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
