/*
 * nysfilter_b200.h -- C ABI of the B200-native Nystrom kernel-filter hot path.
 *
 * The reference (`nysfilter` 0.1.0, /root/reference/pkg/src/nysfilter) is pure
 * Python; it has no FFI.  Each entry point below replaces the NumPy region of
 * the reference named in its comment, so a Python (ctypes) or C/C++ host can
 * bind them directly.  Conventions:
 *   - every pointer marked [dev] is CUDA device memory, [host] is host memory;
 *   - images are planar float32, plane c at `base + c * plane_stride`, rows of
 *     `W` contiguous floats (reference layout: image.py:33-72, data[c, y, x]);
 *   - the library never allocates or frees device memory: callers pass
 *     workspaces sized by the matching *_workspace_bytes() query;
 *   - all work is enqueued on `stream` (a cudaStream_t passed as void*);
 *     nothing synchronises the host unless documented;
 *   - the return value is 0 on success, NYS_EINVAL / NYS_EUNSUPPORTED for bad
 *     arguments (checked before any launch), or NYS_ECUDA + cudaError_t.
 */
#ifndef NYSFILTER_B200_H
#define NYSFILTER_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NYS_OK 0
#define NYS_EINVAL 1
#define NYS_EUNSUPPORTED 2
#define NYS_ECUDA 1000

#define NYS_SPATIAL_BOX 0          /* spatial.py:32 kind "box" */
#define NYS_SPATIAL_GAUSSIAN_FIR 1 /* spatial.py:32 kind "gaussian_fir" */
#define NYS_SPATIAL_GAUSSIAN_RECURSIVE 2 /* spatial.py:32 kind "gaussian_recursive" (sigma >= 1;
                                            sigma < 1 is the FIR path, spatial.py:206-208) */

#define NYS_MAX_RADIUS 64          /* taps = 2R+1 <= 129 */
#define NYS_MAX_M0 256
#define NYS_MAX_RHO 64        /* guide dimensions held in registers by the fast kernels */
#define NYS_MAX_RHO_WIDE 1024 /* wider guides (e.g. 103 hyperspectral bands, 147-dim r = 3 patches)
                                 take the generic paths: step-wise k-means, features written
                                 as planes by a separate pass before K2 */
#define NYS_MAX_CHANNELS 64       /* filtered channels held in registers (brute force) */
#define NYS_MAX_CHANNELS_WIDE 511 /* filtered channels of the Nystrom path (e.g. all 103 bands of a cube) */

/* Library ABI version (major*100 + minor). */
int nys_abi_version(void);

/* Kernels launched by this library since load (all entry points, all streams). */
uint64_t nys_kernel_launches(void);

/* ---------------------------------------------------------------------- */
/* Landmarks: k-means++ seeding + Lloyd (landmarks.py:60-129)             */
/* ---------------------------------------------------------------------- */

/* Bytes of device workspace needed by nys_kmeans_run / nys_kmeans_* for m
 * points of dimension rho and m0 centroids. */
size_t nys_kmeans_workspace_bytes(int64_t m, int rho, int m0);

/*
 * Full k-means on one device, replacing kmeans_landmarks (landmarks.py:76-129):
 *  - k-means++ seeding in FP64 (landmarks.py:60-73).  The host supplies the
 *    random stream it drew from numpy's default_rng(seed):  first_index =
 *    rng.integers(m), then uniforms[j-1] = rng.random() for draw j = 1..m0-1
 *    (Generator.choice(m, p) == searchsorted(cdf, random(), 'right')).
 *  - Lloyd iterations (<= max_iter) with the reference's break rule
 *    (labels unchanged -> stop before the update) and empty-cluster repair.
 *  - the final exact (differenced) assignment and quant_error.
 * points [dev]: planar (rho, m) float32 with plane stride `plane_stride`.
 * centroids_out [dev]: m0*rho float64 row-major.
 * errors_out [dev]: max_iter float64 (Σ nearest after each assignment step).
 * stats_out [dev]: int64[4] = {iterations_run, first_zero_total_draw (or -1),
 *                              last_changed_count, empty_repairs}.
 * quant_error_out [dev]: float64[1].  assignment_out [dev] (nullable): int64[m].
 * When quant_error_out and assignment_out are both null the final exact pass
 * is skipped (the caller runs nys_kmeans_exact itself, e.g. overlapped with
 * its host-side work on the centroids).
 * seed_indices_out [dev] (nullable): int64[m0], the k-means++ picks.
 * If stats_out[1] >= 0 the k-means++ stream hit sum(d2) == 0 at that draw; the
 * reference then switches to rng.integers(m) (landmarks.py:69-70) and the
 * caller must re-run with nys_kmeans_run_seeded() using seed_indices_out[<j]
 * followed by its own integers(m) draws.
 */
int nys_kmeans_run(const float* points, int64_t plane_stride, int64_t m, int rho,
                   int m0, int max_iter, int64_t first_index, const double* uniforms /*[host] m0-1*/,
                   double* centroids_out, double* errors_out, int64_t* stats_out,
                   double* quant_error_out, int64_t* assignment_out, int64_t* seed_indices_out,
                   void* workspace, size_t workspace_bytes, void* stream);

/* Same, but with all m0 seed indices already chosen by the host
 * (seed_indices [host] int64[m0]); used for the sum(d2)==0 corner case. */
int nys_kmeans_run_seeded(const float* points, int64_t plane_stride, int64_t m, int rho,
                          int m0, int max_iter, const int64_t* seed_indices,
                          double* centroids_out, double* errors_out, int64_t* stats_out,
                          double* quant_error_out, int64_t* assignment_out,
                          void* workspace, size_t workspace_bytes, void* stream);

/* --- step-wise k-means for the row-band-sharded multi-GPU driver --------- */
/* Per-rank partial results are combined by the caller (NCCL all-reduce) in a
 * fixed order; these helpers expose exactly the per-rank reductions.        */

/* d2 := min(d2, |x - c|^2) (or := when init != 0) in FP64 over the local
 * points; writes the local FP64 sum of d2 to sum_out [dev] (1 double). */
int nys_kmeanspp_update(const float* points, int64_t plane_stride, int64_t m, int rho,
                        const double* c /*[dev] rho*/, int init, double* d2,
                        double* sum_out, void* workspace, size_t workspace_bytes, void* stream);

/* First local index i with prefix_sum(d2)[i] > target (FP64); -1 if none.
 * index_out [dev] int64[1]. */
int nys_kmeanspp_pick(const double* d2, int64_t m, double target, int64_t* index_out,
                      void* workspace, size_t workspace_bytes, void* stream);

/* One Lloyd assignment pass over the local points against centroids (FP64
 * [dev] m0*rho).  labels [dev] int32[m] is read (previous) and rewritten.
 * acc_out [dev] float64[m0*(rho+1) + 2]: per-cluster coordinate sums and
 * counts (cluster j at j*(rho+1): rho sums then count), then Σ nearest, then
 * the number of changed labels.  first_pass != 0 counts every label as
 * changed. */
int nys_kmeans_assign(const float* points, int64_t plane_stride, int64_t m, int rho,
                      const double* centroids, int m0, int32_t* labels, int first_pass,
                      double* acc_out, void* workspace, size_t workspace_bytes, void* stream);

/* Exact (differenced) FP64 nearest distance and Σ (landmarks.py:121-129);
 * assignment_out nullable. sum_out [dev] 1 double. */
int nys_kmeans_exact(const float* points, int64_t plane_stride, int64_t m, int rho,
                     const double* centroids, int m0, int64_t* assignment_out,
                     double* sum_out, void* workspace, size_t workspace_bytes, void* stream);

/* Local maximum of `nearest` recomputed against `centroids` for the points
 * labelled `labels`, excluding indices listed in excluded [dev] int64[n_excl];
 * writes {value, local index} as two doubles to out [dev].  Used for the
 * empty-cluster repair (landmarks.py:114-119). */
int nys_kmeans_farthest(const float* points, int64_t plane_stride, int64_t m, int rho,
                        const double* centroids, int m0, const int32_t* labels,
                        const int64_t* excluded, int n_excl, double* out,
                        void* workspace, size_t workspace_bytes, void* stream);

/* --- device-resident sharded k-means (parallel.device_distributed_kmeans) ----
 * The same global semantics as the host-orchestrated step-wise calls above, with
 * every per-draw / per-iteration decision taken on the device so a rank never
 * waits on the host between collectives (all-gather / all-reduce on device
 * buffers in between, stream-ordered):
 *   state_init; k-means++: per draw j = 1..m0-1 nys_kmeanspp_update (local D^2,
 *   local total) -> all-gather of the totals -> nys_kmeanspp_owner_pick (every
 *   rank resolves the owner of u_j * total from the totals in rank order; the
 *   owner writes point + global index into cand[rho+1], the others zeros) ->
 *   all-reduce(sum) of cand;  Lloyd: per iteration nys_kmeans_lloyd_local (local
 *   sums / counts / objective / changed, zero work once converged) -> all-reduce
 *   (sum) -> nys_kmeans_lloyd_update (the reference's update and break rule);
 *   nys_kmeans_state_read at the end.  stats[1] >= 0 (a zero D^2 total) or
 *   stats[3] == -1 (an empty cluster, whose repair needs the global farthest
 *   point) tell the caller to rerun the host-orchestrated path. */
int nys_kmeans_state_init(void* workspace, size_t workspace_bytes, int64_t m, int rho, int m0, void* stream);
int nys_kmeans_state_read(const void* workspace, int64_t m, int rho, int m0, int64_t* stats_out /*[dev] 4*/,
                          void* stream);
int nys_kmeanspp_owner_pick(const float* points, int64_t plane_stride, int64_t m, int rho, int m0, const double* d2,
                            const double* totals /*[dev] world*/, int world, int rank, int64_t my_offset,
                            double u, int draw, double* cand_out /*[dev] rho+1*/, void* workspace,
                            size_t workspace_bytes, void* stream);
/* Cluster sums are exact fixed-point integers, x * 2^sexp rounded once per point, with
 * sexp = 60 - ilogb(max|x| * m) over ALL ranks' points (max|x| all-reduced, m the global
 * count): integer all-reduce, so the centroids are bit-identical to the single-device
 * cooperative kernel's.  tot_out [dev] int64[m0*rho + m0 + 1] (sums, counts, changed),
 * obj_out [dev] 1 double (objective). */
int nys_kmeans_lloyd_local(const float* points, int64_t plane_stride, int64_t m, int rho, const double* centroids,
                           int m0, int it, int sexp, int64_t* tot_out, double* obj_out, void* workspace,
                           size_t workspace_bytes, void* stream);
int nys_kmeans_lloyd_update(int64_t m, int rho, int m0, int it, int sexp, const int64_t* tot, const double* obj,
                            double* centroids, double* errors, void* workspace, size_t workspace_bytes, void* stream);

/* Gather point `index` (rho coordinates, FP64) into dst [dev]. */
int nys_gather_point(const float* points, int64_t plane_stride, int rho, int64_t index,
                     double* dst, void* stream);

/* ---------------------------------------------------------------------- */
/* Filter (filters.py:214-257 + spatial.py:194-209 + nystrom.py:43-114)   */
/* ---------------------------------------------------------------------- */

/* Everything one filter launch needs.  Host-side struct; the library copies
 * the constants into kernel parameters / device constants itself. */
typedef struct nys_filter_desc {
    /* geometry */
    int n;          /* filtered channels (f) */
    int rho;        /* guide dimension (p); for guide_kind==1 must be n*9 */
    int H, W;       /* full image size (the borders replicate at 0 and H-1/W-1) */
    int guide_kind; /* 0: planar guide (rho planes); 1: raw 3x3 patches of f
                       gathered on the fly (channel, dy, dx order, edge-replicated,
                       filters.py:174-181) */
    /* spatial kernel */
    int spatial_kind;   /* NYS_SPATIAL_BOX | NYS_SPATIAL_GAUSSIAN_FIR */
    int radius;         /* R (box radius or FIR truncation radius) */
    double sigma;       /* FIR sigma (ignored for box) */
    /* range kernel and landmarks */
    int m0;             /* landmarks */
    double theta;       /* Gaussian range scale: kappa = exp(-|s-t|^2/(2 theta^2)) */
    /* Nystrom algebra, computed on the host in FP64 (nystrom.py:67-114):
     * M = sum_{k retained} w_k w_k^T / alpha_k, u0 = w_0, alpha0 = alpha_1 */
    const double* centroids; /* [host] m0*rho */
    const double* M;         /* [host] m0*m0 row-major */
    const double* u0;        /* [host] m0 */
    double alpha0;
    double eps_den;          /* 1e-12 * (2S+1)^2 * max|alpha| (filters.py:242) */
    /* rows [row_lo, row_hi) of the image are present in the f / guide buffers
     * (base pointers still address image row 0); row_hi == 0 means all H rows.
     * Used by the row-band-sharded multi-GPU path, whose ranks hold their rows
     * plus R (+1) halo rows; reads never leave this range. */
    int row_lo, row_hi;
    /* 0: y-form (M = sum_k w_k w_k^T / alpha_k, contraction with the raw
     * features b(x)).  1: phi-form for ill-conditioned landmark kernels: M holds
     * P = Lambda^{-1/2} W^T (rows >= rank zero), so y = phi = P b, the planes
     * are phi_k f, and the contraction weights are phi(x) itself (K2 stores
     * them as the raw-feature planes).  Same reference quantity
     * (filters.py:227-238); FP32 error no longer grows with cond(A). */
    int phi_form;
    /* 1: M holds the lower Cholesky factor L of A (row-major) instead of M;
     * nys_filter_prepare forms M = A^{-1} = L^{-T} L^{-1} on the device in FP64
     * (y-form, nothing dropped, m0 <= 64).  0: M as above. */
    int M_is_cholesky;
    /* 1: the `out` pointers of nys_filter_vpass / nys_filter_finish address
     * float64 planes (e.g. a page-locked host array for the reference's FP64
     * Image); 0: float32. */
    int out_f64;
} nys_filter_desc;

/* Size of the horizontal-pass plane buffer for a band of `rows` output rows:
 * (m0+1)*(n+1) planes of (rows + 2R) virtual rows x Wp floats, Wp = W rounded
 * up to a multiple of 4.  Virtual row v of a band starting at out0 holds the
 * row-filtered planes of image row clamp(out0 - R + v, 0, H-1), so the
 * vertical pass never clamps (replicate borders, spatial.py:85-88). */
size_t nys_filter_planes_bytes(const nys_filter_desc* d, int rows);

/* Floats per virtual row of the plane buffer ([row][x/32][plane][32]); pass
 * it (or more) as planes_stride.  Includes the raw-feature planes K2 stores
 * for K3 when the guide is high-dimensional (rho > 8) or the NLM patch guide. */
int64_t nys_filter_plane_row_stride(const nys_filter_desc* d);

/* Device bytes for the filter's constant block + reduction scratch. */
size_t nys_filter_workspace_bytes(const nys_filter_desc* d);

/* Byte offsets of the workspace regions (diagnostics / tests): out[8] =
 * {FP64 constants (landmarks, u0, 1/alpha_1, eps_den, alpha_1), statistics,
 *  Cholesky factor, FP64 M, queued-pixel list, per-pixel chunk counters,
 *  window partial sums, total bytes}. */
int nys_filter_workspace_layout(const nys_filter_desc* d, int64_t* out);

/* Upload the per-call constants (centroids, M, u0) into `workspace` and reset
 * the min|eta| / guarded-pixel accumulators.  Call once per filter before the
 * band passes below.  Asynchronous: the host constants are staged by the
 * runtime before the call returns. */
int nys_filter_prepare(const nys_filter_desc* d, void* workspace, size_t workspace_bytes,
                       void* stream);

/*
 * In-stream (speculative) mixing plan: the host never waits for the landmarks.
 *
 * nys_filter_plan_async forks from `stream` at the point of the call: once the
 * landmark coordinates have landed in `centroids` [pinned host, m0 x rho FP64,
 * written by an earlier copy on `stream`], a host function on a side stream
 * runs the lite plan (nys_mixing_plan_lite, Cholesky factor) into the pinned
 * `staging` image of the workspace constants (the stream signals it with a
 * stream-ordered write of a pinned word; the worker makes no CUDA call).
 * Work queued on `stream` between this call and nys_filter_prepare_join (e.g.
 * the k-means exact pass) overlaps the plan.  The desc's M / u0 / alpha0 /
 * eps_den / phi_form / M_is_cholesky are ignored (the plan supplies them).
 *
 * nys_filter_prepare_join queues the kernel that waits on the device for the
 * plan (it polls the staging buffer's `done` word), pulls the image into
 * `workspace`, forms M = A^{-1} and resets the statistics; the band passes
 * follow as usual.
 *
 * The speculation is the y-form with nothing dropped (cond(A) <= phi_cond).
 * Read the verdict with nys_filter_plan_result once `stream` has passed the
 * join: status NYS_OK means the passes used the exact plan; NYS_EUNSUPPORTED
 * means the plan needs drops or the phi-form -- rerun with nys_filter_prepare
 * and a plan from nys_mixing_plan (the speculative outputs are meaningless).
 * `staging` [pinned, nys_filter_plan_staging_bytes(d), zero-filled once] and
 * `centroids` must stay untouched until then; a new plan on a staging buffer
 * whose previous plan is still pending waits for it (up to 60 s, then EINVAL).  For m0 <= 64 the device forms
 * M from the Cholesky factor (and copies the image itself from the mapped
 * staging buffer); larger m0 carry M formed on the host.
 */
typedef struct nys_plan_result {
    int status;      /* NYS_OK, NYS_EUNSUPPORTED (fall back), or an error code */
    int rank;        /* retained eigenpairs (m0 on NYS_OK) */
    double alpha0;   /* largest eigenvalue of A */
    double eps_den;  /* guard threshold used by the passes */
    double host_us;  /* wall time of the plan inside the host function */
} nys_plan_result;
size_t nys_filter_plan_staging_bytes(const nys_filter_desc* d);
int nys_filter_plan_async(const nys_filter_desc* d, const double* centroids, double eps_drop, double phi_cond,
                          void* staging, size_t staging_bytes, void* workspace, size_t workspace_bytes,
                          void* stream);
int nys_filter_prepare_join(const nys_filter_desc* d, void* staging, void* workspace, void* stream);
int nys_filter_plan_result(const void* staging, nys_plan_result* out);

/*
 * K2: range features + horizontal pass for the band of output rows
 * [out0, out0+out_rows) (computes its rows + 2R virtual halo rows).
 * f [dev] (n,H,W) planar, f_plane_stride; guide [dev] (rho,H,W) (ignored for
 * guide_kind 1; may alias f).  planes [dev] 16-byte aligned: (m0+1)*(n+1)
 * planes, plane stride planes_stride (multiple of 4, >= (out_rows+2R)*Wp).
 * Plane (i*(n+1)+c) holds the row-filtered y_i*f_c (c<n) or y_i (c==n), with
 * y = M b(x) for i<m0 and y_{m0} = u0.b(x) (the rank-1 lead term).
 */
int nys_filter_hpass(const nys_filter_desc* d, const float* f, int64_t f_plane_stride,
                     const float* guide, int64_t guide_plane_stride,
                     int out0, int out_rows, float* planes, int64_t planes_stride,
                     const void* workspace, void* stream);

/*
 * K3: vertical pass + per-pixel reconstruction, guard and division for the
 * band [out0, out0+out_rows) whose planes K2 produced.  The plane stack is
 * read through a TMA descriptor (cp.async.bulk.tensor).  out [dev] (n,H,W)
 * planar with out_plane_stride.  Accumulates min|eta| and the guarded-pixel
 * count into the workspace.
 */
int nys_filter_vpass(const nys_filter_desc* d, const float* f, int64_t f_plane_stride,
                     const float* guide, int64_t guide_plane_stride,
                     const float* planes, int64_t planes_stride,
                     int out0, int out_rows, float* out, int64_t out_plane_stride,
                     const void* workspace, void* stream);

/* Copy {min|eta| (float64), guarded pixels (int64 bit pattern in a double
 * slot)} into stats_out [dev] (2 x 8 bytes). */
int nys_filter_stats(const nys_filter_desc* d, const void* workspace, void* stats_out, void* stream);

/*
 * Near-guard refinement + statistics; call once after the last band's
 * nys_filter_vpass (replaces nys_filter_stats on the tiled path).
 * K3 forms zeta, eta and the guard decisions in FP32; the reference forms
 * them in FP64 (filters.py:223-257).  Where the FP32 ratio is ill-conditioned
 * (|eta| small against its scale sum_i b_i |conv(y_i)|) or a guard decision
 * lies within FP32 error of eps_den, K3 queued the pixel; this call
 * re-evaluates each queued pixel in FP64 by direct window summation,
 * eta(x) = sum_y w(x-y) b(x)^T M b(y) (and zeta_c, eta_lead, zeta_lead alike),
 * applies the guard in FP64 and overwrites the pixel in `out` (same pointer
 * conventions as nys_filter_vpass).  Then it writes {min|eta| (float64),
 * guarded pixels (int64 bit pattern)} to stats_out [dev or mapped pinned]
 * (nullable).  When the in-stream plan's gate timed out, stats_out receives
 * {NaN, -1}: the step's outputs are invalid.
 */
int nys_filter_finish(const nys_filter_desc* d, const float* f, int64_t f_plane_stride,
                      const float* guide, int64_t guide_plane_stride, float* out, int64_t out_plane_stride,
                      const void* workspace, void* stats_out, void* stream);

/* ---------------------------------------------------------------------- */
/* Recursive Gaussian spatial kernel (spatial.py:114-191)    */
/* ---------------------------------------------------------------------- */

/* {gain, a1..a5} of the fifth-order van Vliet/Young/Verbeek recursion whose
 * forward/backward cascade has impulse-response variance sigma^2
 * (_vyv_coeffs, spatial.py:132-146).  [host] coeffs_out[6]. */
int nys_vyv_coeffs(double sigma, double* coeffs_out);

/* Device scratch for nys_filter_recursive with landmark bands of
 * `groups_per_band` groups (each group = the n+1 planes of one landmark or
 * the lead projection; <= 0 means all m0+1 groups in one band).  Larger
 * scratch -> fewer bands (each band re-reads the per-pixel features). */
size_t nys_filter_recursive_scratch_bytes(const nys_filter_desc* d, int groups_per_band);

/*
 * The whole filter with d->spatial_kind == NYS_SPATIAL_GAUSSIAN_RECURSIVE
 * (replaces filters.py:214-257 with spatial.py:179-191 as the convolution):
 * features, row recursion, column recursion fused with the contraction, the
 * (fir_mass)^2 scale, guard and division.  d->eps_den must use the radius
 * ceil(3 sigma) (spatial.py:66-69).  Whole images only (row_lo == 0,
 * row_hi in {0, H}): the recursion couples every row of a column.
 * Call nys_filter_prepare first; statistics via nys_filter_stats.
 * scratch [dev] of at least nys_filter_recursive_scratch_bytes(d, 1) bytes.
 */
int nys_filter_recursive(const nys_filter_desc* d, const float* f, int64_t f_plane_stride,
                         const float* guide, int64_t guide_plane_stride,
                         float* out, int64_t out_plane_stride, void* scratch, size_t scratch_bytes,
                         const void* workspace, void* stream);

/* ---------------------------------------------------------------------- */
/* PCA patch guide (filters.py:161-187)                      */
/* ---------------------------------------------------------------------- */

/* Workspace for nys_patch_moments (0 if n(2r+1)^2 > 1024). */
size_t nys_patch_moments_workspace_bytes(int n, int H, int W, int r);

/* First and centred second moments of the (2r+1)^2-per-channel patch
 * vectors (channel-major, dy, dx, edge replicate; filters.py:174-181) of
 * f [dev] (n,H,W), in FP64, deterministic:
 *   mean_out [dev] dim doubles (dim = n(2r+1)^2),
 *   gram_tiles_out [dev] T*16 doubles, T = t(t+1)/2, t = ceil(dim/4): the
 *   4x4 tiles (ti <= tj, row-major over ti) of Σ_p (x_p - mean)(x_p - mean)^T.
 * The covariance of the reference is that Gram / (H W). */
int nys_patch_moments(const float* f, int64_t f_plane_stride, int n, int H, int W, int r, double* mean_out,
                      double* gram_tiles_out, void* workspace, size_t workspace_bytes, void* stream);

/* guide [dev] (pca_dim, H, W): out[k](p) = Σ_d (x_p[d] - mean[d]) basis[d*pca_dim + k]
 * with mean [dev] dim floats and basis [dev] dim x pca_dim floats (the
 * leading covariance eigenvectors as columns). */
int nys_pca_project(const float* f, int64_t f_plane_stride, int n, int H, int W, int r, const float* mean,
                    const float* basis, int pca_dim, float* out, int64_t out_plane_stride, void* stream);

/* Stand-alone separable filtering of an FP64 plane stack (spatial.py:194-234:
 * apply_planes / box_filter / gaussian_fir / gaussian_recursive): in, out [dev]
 * (P, H, W) float64; kind NYS_SPATIAL_*; radius for box / FIR; sigma for FIR
 * and recursive (sigma < 1: the FIR at ceil(3 sigma)); scratch [dev] P*H*W
 * doubles for the box / FIR passes (unused by the recursive kind).  Row pass
 * then column pass, edge replicate, FP64. */
int nys_spatial_planes(const double* in, double* out, int64_t P, int H, int W, int kind, double sigma, int radius,
                       double* scratch, void* stream);

/* ---------------------------------------------------------------------- */
/* Direct (brute-force) kernel filter, Eq. (1) (filters.py:107-138), §8 f1 */
/* ---------------------------------------------------------------------- */

/* out(x) = Σ_d w(d) κ(p(x+d)-p(x)) f(x+d) / Σ_d w(d) κ(p(x+d)-p(x)) over the
 * (2S+1)^2 window with edge replicate; w = outer product of the unnormalised
 * Gaussian taps (box: ones), S = d->radius, or ceil(3 sigma) for the
 * recursive kind (evaluated as its FIR counterpart).  Uses d->n, rho, H, W,
 * spatial_kind, radius, sigma, theta; guide_kind must be 0 (materialise a
 * patch guide with nys_patch_guide first).  FP32, no workspace. */
int nys_brute_force_filter(const nys_filter_desc* d, const float* f, int64_t f_plane_stride,
                           const float* guide, int64_t guide_plane_stride, float* out,
                           int64_t out_plane_stride, void* stream);

/* ---------------------------------------------------------------------- */
/* Quality metrics (metrics.py:37-122), §8 f4                              */
/* ---------------------------------------------------------------------- */

/* Device workspace for nys_quality_planes over n planes. */
size_t nys_quality_workspace_bytes(int n);

/* Per plane c of a and b ([dev] planar, float32 (elem_bytes 4) or float64
 * (elem_bytes 8)): sq_sums_out[c] = Σ (a-b)^2 (FP64, [dev] n doubles) and,
 * when ssim_out [dev] is non-null, the mean single-scale SSIM of the plane
 * (11x11 Gaussian window sigma 1.5, C1 = (0.01 R)^2, C2 = (0.03 R)^2, valid
 * positions only; whole-plane statistics below 11x11).  Deterministic. */
int nys_quality_planes(const void* a, int64_t a_plane_stride, const void* b, int64_t b_plane_stride,
                       int elem_bytes, int n, int H, int W, double range_max, double* sq_sums_out,
                       double* ssim_out, void* workspace, size_t workspace_bytes, void* stream);

/* Device-side address of a buffer for the kernels' pointer arguments: device
 * memory maps to itself, page-locked host memory to its mapped device view
 * (so K3 can write the filtered image straight into a pinned host buffer,
 * overlapping the device->host transfer with the vertical pass).  NYS_EINVAL
 * when `p` is not device-accessible. */
int nys_device_view(const void* p, void** device_ptr_out);

/* Materialise the raw (2r+1)^2*n patch guide (filters.py:174-181) as planes:
 * out [dev] (n*(2r+1)^2, H, W). */
int nys_patch_guide(const float* f, int64_t f_plane_stride, int n, int H, int W, int r,
                    float* out, int64_t out_plane_stride, void* stream);

/* ---------------------------------------------------------------------- */
/* Host FP64 helpers (symeig.py, nystrom.py)                               */
/* ---------------------------------------------------------------------- */

/* Cyclic Jacobi eigendecomposition of a symmetric k x k matrix (row-major,
 * symmetrised as (A+A^T)/2), descending eigenvalues, largest-|.| entry of
 * each eigenvector non-negative (symeig.py:58-125).  vectors_out column j
 * pairs with values_out[j].  Returns the number of sweeps in *sweeps. */
int nys_jacobi_eig(const double* a, int k, double* values_out, double* vectors_out, int* sweeps);

/* Fast symmetric eigensolver used on the hot path (Householder tridiagonal +
 * implicit QL): same eigenpairs as nys_jacobi_eig up to rounding, basis and
 * signs; descending eigenvalues, eigenvectors as columns. */
int nys_sym_eig(const double* a, int k, double* values_out, double* vectors_out);

/* The m0 x m0 host products the kernels consume, in one call (replaces
 * nystrom.py:67-69 build_A, 97-109 eigendecomposition + drop rule, and the
 * filters.py:214-219 mixing products):
 *   A = exp(-|c_i - c_j|^2 / (2 theta^2)), eigenvalues alpha_1 >= ... ,
 *   retained alpha_k > eps_drop * alpha_1, M = sum_retained w_k w_k^T / alpha_k,
 *   u0 = w_1.
 * When nothing is dropped M = A^{-1} (Cholesky) and u0 comes from inverse
 * iteration on the eigenvalues of a values-only QL, ~4x cheaper than the full
 * eigensystem; otherwise the full eigensystem (nys_sym_eig) is used.
 * alphas_out: m0 (first *rank_out valid, descending); M_out: m0 x m0; u0_out: m0.
 * Returns NYS_EDEGENERATE when alpha_1 <= 0. */
#define NYS_EDEGENERATE 3
/* Hot-path variant: alpha_1 by Sturm bisection on the tridiagonal plus two Sturm
 * counts instead of every eigenvalue.  Returns NYS_EUNSUPPORTED (nothing
 * written but possibly M/u0 scratch) when an eigenpair would be dropped
 * (alpha <= eps_drop alpha_1) or cond(A) > phi_cond -- the caller then uses
 * nys_mixing_plan.  Otherwise rank = m0, M = A^{-1}, u0 = w_1, info_out[0] = alpha_1. */
int nys_mixing_plan_lite(const double* centroids, int m0, int rho, double theta, double eps_drop, double phi_cond,
                         int chol_only, double* info_out, int* rank_out, double* M_out, double* u0_out);
/* chol_only != 0: M_out receives the lower Cholesky factor of A instead of
 * A^{-1} (pass it with nys_filter_desc.M_is_cholesky = 1). */
int nys_mixing_plan(const double* centroids, int m0, int rho, double theta, double eps_drop, double* alphas_out,
                    int* rank_out, double* M_out, double* u0_out);

#ifdef __cplusplus
}
#endif

#endif /* NYSFILTER_B200_H */
