"""Filter API (drop-in mirror of reference ``filters.py``).

``fast_filter(f, p, params) -> FilterReport`` keeps the reference's contract
(filters.py:199-274): same parameters, same validation errors, same report
fields and timing keys.  The work runs on the B200:

  k-means++ + Lloyd  -> K0/K1 kernels (landmarks.py)
  A, eig, drop rule  -> host FP64 (nystrom.mixing_plan), m0 x m0 only
  features + H-pass  -> K2  nys_filter_hpass
  V-pass + Σ_k + guard + division -> K3  nys_filter_vpass

There is no CPU fallback: without the native library or a GPU every call
raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _native
from ._device import StageTimer, ptr, require_cuda, stamp, stream_ptr, to_device_f32, workspace
from .bands import Band, plan_bands
from .image import Image
from .landmarks import DEFAULT_MAX_ITER, exact_assignment, exact_assignment_async, kmeans_device
from .nystrom import DEFAULT_EPS_DROP, PHI_FORM_COND, MixingPlan, RangeKernel, mixing_plan
from .spatial import BOX, GAUSSIAN_FIR, GAUSSIAN_RECURSIVE, SpatialKernel

MODE_BILATERAL = "bilateral"
MODE_JOINT = "joint"
MODE_NLM = "nlm"
STRATEGY_KMEANS = "kmeans"
STRATEGY_UNIFORM = "uniform"
DENOMINATOR_EPS_SCALE = 1e-12

# default cap on the horizontal-pass plane buffer (bytes); bands are planned
# so that one band's planes fit (bands.plan_bands)
PLANE_BUDGET_BYTES = 64 << 30
SMALL_PLANES_BYTES = 8 << 30


@dataclass(frozen=True)
class FilterParams:
    """Everything that determines a filtering run (filters.py:57-86)."""

    spatial: SpatialKernel
    theta: float
    m0: int = 15
    seed: int = 0
    landmark_strategy: str = STRATEGY_KMEANS
    mode: str = MODE_BILATERAL
    patch_radius: int = 3
    pca_dim: int = 25
    eps_drop: float = DEFAULT_EPS_DROP
    kmeans_max_iter: int = DEFAULT_MAX_ITER

    def __post_init__(self) -> None:
        if self.theta <= 0:
            raise ValueError("theta must be positive")
        if self.m0 < 1:
            raise ValueError("m0 must be >= 1")
        if self.landmark_strategy not in (STRATEGY_KMEANS, STRATEGY_UNIFORM):
            raise ValueError(f"unknown landmark strategy {self.landmark_strategy!r}")
        if self.mode not in (MODE_BILATERAL, MODE_JOINT, MODE_NLM):
            raise ValueError(f"unknown mode {self.mode!r}")
        if not 0.0 <= self.eps_drop < 1.0:
            raise ValueError("eps_drop must lie in [0, 1)")

    @property
    def range_kernel(self) -> RangeKernel:
        return RangeKernel(theta=self.theta)


@dataclass
class FilterReport:
    """filters.py:89-96 plus the landmarks actually used."""

    output: Image
    timings: dict = field(default_factory=dict)
    retained_rank: int = 0
    quant_error: float = 0.0
    min_denominator: float = 0.0
    guarded_pixels: int = 0
    centroids: np.ndarray | None = None


class PatchGuide:
    """Lazy NLM guide: the raw (2r+1)^2 patches of ``source`` per pixel
    (channel-major, then dy, then dx, edge-replicated: filters.py:174-181).

    With ``pca_dim`` equal to the full patch dimension the reference's PCA
    guide is a centring plus an orthonormal rotation of these patches, which
    leaves every guide-space distance -- and therefore k-means, the range
    kernel and the filter output -- unchanged (survey probe: 6.9e-10), so the
    kernels gather raw patches straight from the image instead of storing a
    dim-channel guide.  Landmark coordinates are then in raw-patch space.
    """

    def __init__(self, source: Image, patch_radius: int):
        self.source = source
        self.patch_radius = int(patch_radius)
        self.range_max = source.range_max

    @property
    def channels(self) -> int:
        return self.source.channels * (2 * self.patch_radius + 1) ** 2

    @property
    def height(self) -> int:
        return self.source.height

    @property
    def width(self) -> int:
        return self.source.width

    def device_planes(self, f_dev: torch.Tensor | None = None) -> torch.Tensor:
        f_dev = to_device_f32(self.source.data) if f_dev is None else f_dev
        n, H, W = f_dev.shape
        out = torch.empty((self.channels, H, W), dtype=torch.float32, device=f_dev.device)
        _native.call("nys_patch_guide", ptr(f_dev), H * W, n, H, W, self.patch_radius, ptr(out), H * W,
                     stream_ptr())
        return out

    @property
    def data(self):
        planes = self.device_planes()
        return planes if self.source.on_device else planes.double().cpu().numpy()


def _check_sizes(f, p) -> None:
    if (f.width, f.height) != (p.width, p.height):
        raise ValueError(f"input {f.width}x{f.height} and guide {p.width}x{p.height} must share the spatial size")


def build_guide(f: Image, mode: str = MODE_BILATERAL, guide: Image | None = None, patch_radius: int = 3,
                pca_dim: int = 25):
    """Guide for the requested mode (filters.py:141-158)."""
    if mode == MODE_BILATERAL:
        return f
    if mode == MODE_JOINT:
        if guide is None:
            raise ValueError("joint mode requires an external guide image")
        _check_sizes(f, guide)
        return guide
    if mode == MODE_NLM:
        return pca_patch_guide(f, patch_radius, pca_dim)
    raise ValueError(f"unknown mode {mode!r}")


def pca_patch_guide(f: Image, patch_radius: int, pca_dim: int):
    """PCA patch guide (filters.py:161-187).  The full-dimension case (the
    configuration BASELINE cfg 3 uses) is served by ``PatchGuide`` (a rotation
    of the raw patches leaves every guide distance unchanged); a truncated
    projection (pca_dim < n(2r+1)^2, §8 row f3) is computed on the device by
    ``pca.pca_patch_guide``: FP64 patch moments, host eig, projection."""
    dim = f.channels * (2 * patch_radius + 1) ** 2
    if not 1 <= pca_dim <= dim:
        raise ValueError(f"pca_dim must lie in [1, {dim}], got {pca_dim}")
    if pca_dim == dim:
        return PatchGuide(f, patch_radius)
    from .pca import pca_patch_guide as _pca

    return _pca(f, patch_radius, pca_dim)


def _desc(n: int, rho: int, H: int, W: int, gkind: int, spatial: SpatialKernel, theta: float,
          C_: np.ndarray, plan, keep: list) -> _native.FilterDesc:
    d = _native.FilterDesc()
    d.n, d.rho, d.H, d.W, d.guide_kind = n, rho, H, W, gkind
    if spatial.kind == BOX:
        d.spatial_kind, d.radius, d.sigma = _native.NYS_SPATIAL_BOX, spatial.radius, 0.0
    elif spatial.kind == GAUSSIAN_FIR:
        d.spatial_kind, d.radius, d.sigma = _native.NYS_SPATIAL_GAUSSIAN_FIR, spatial.radius, spatial.sigma
    else:
        d.spatial_kind, d.radius, d.sigma = (_native.NYS_SPATIAL_GAUSSIAN_RECURSIVE, spatial.effective_radius(),
                                             spatial.sigma)
    d.m0 = C_.shape[0]
    d.theta = theta
    arrs = [np.ascontiguousarray(C_, dtype=np.float64), np.ascontiguousarray(plan.M, dtype=np.float64),
            np.ascontiguousarray(plan.u0, dtype=np.float64)]
    keep.extend(arrs)
    d.centroids = arrs[0].ctypes.data_as(C.POINTER(C.c_double))
    d.M = arrs[1].ctypes.data_as(C.POINTER(C.c_double))
    d.u0 = arrs[2].ctypes.data_as(C.POINTER(C.c_double))
    d.alpha0 = plan.alpha0
    d.eps_den = plan.eps_den
    d.phi_form = 1 if plan.phi_form else 0
    d.M_is_cholesky = 1 if plan.M_is_cholesky else 0
    return d


@dataclass
class _Inputs:
    f: torch.Tensor          # (n, H, W) float32
    guide: torch.Tensor      # planar guide for the kernels (== f for BLF / patch-on-the-fly)
    gkind: int               # 0 planar, 1 3x3 patches gathered from f
    points: torch.Tensor     # (rho, m) planar k-means points
    rho: int


def _prepare_inputs(f: Image, p) -> _Inputs:
    f_dev = to_device_f32(f.data)
    n, H, W = f_dev.shape
    if p is f or (isinstance(p, Image) and p.data is f.data):
        return _Inputs(f_dev, f_dev, 0, f_dev.reshape(n, H * W), n)
    if isinstance(p, PatchGuide):
        planes = p.device_planes(f_dev if p.source is f else None)
        rho = planes.shape[0]
        if p.patch_radius == 1 and p.source is f:
            return _Inputs(f_dev, f_dev, 1, planes.reshape(rho, H * W), rho)
        return _Inputs(f_dev, planes, 0, planes.reshape(rho, H * W), rho)
    g_dev = to_device_f32(p.data)
    return _Inputs(f_dev, g_dev, 0, g_dev.reshape(g_dev.shape[0], H * W), g_dev.shape[0])


@dataclass
class _Inflight:
    """In-stream plan for run_filter: the landmarks arrive in ``kmeans.host``
    (pinned) during the step; ``between()`` queues work that overlaps the plan
    (the k-means exact pass).  run_filter fills ``staging`` and ``keep``."""
    kmeans: object
    between: object
    staging: torch.Tensor | None = None
    keep: list | None = None

    def result(self) -> _native.PlanResult:
        r = _native.PlanResult()
        _native.check(_native.lib().nys_filter_plan_result(ptr(self.staging), C.byref(r)), "nys_filter_plan_result")
        return r


_TLS = threading.local()  # per host thread: released with the thread


def _tls_dict(name: str) -> dict:
    d = getattr(_TLS, name, None)
    if d is None:
        d = {}
        setattr(_TLS, name, d)
    return d


class _StagingCache(dict):
    """A thread's staging buffers; when the thread ends, a plan it left pending (a call that
    raised before its final wait) is waited for before the pinned memory is released, since
    the worker thread may still be writing into it."""

    def __del__(self):
        try:
            import time

            r = _native.PlanResult()
            for buf in self.values():
                t0 = time.monotonic()
                while (_native.lib().nys_filter_plan_result(buf.data_ptr(), C.byref(r)) != _native.NYS_OK
                       and time.monotonic() - t0 < 10.0):
                    time.sleep(1e-4)
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


def _plan_staging(nbytes: int) -> torch.Tensor:
    """Reused zero-filled page-locked staging buffer for nys_filter_plan_async, one per
    (host thread, size): a buffer is busy from the fork until the call's final wait."""
    cache = getattr(_TLS, "staging", None)
    if cache is None:
        cache = _TLS.staging = _StagingCache()
    buf = cache.get(nbytes)
    if buf is None:
        buf = torch.zeros(nbytes, dtype=torch.uint8, pin_memory=True)
        cache[nbytes] = buf
    return buf


def plan_staging_buffers() -> list:
    """This thread's in-stream plan staging buffers (read with nys_filter_plan_result)."""
    return list(getattr(_TLS, "staging", {}).values())


def run_filter(inp: _Inputs, centroids: np.ndarray | None, params: FilterParams, timer: StageTimer | None = None,
               plane_budget: int | None = None, out: torch.Tensor | None = None,
               kernel_events: list | None = None, rows: tuple[int, int] | None = None, row_origin: int = 0,
               H_global: int | None = None, inflight: _Inflight | None = None, stats_ptr: int | None = None):
    """K2/K3 over row bands given landmarks; returns (out, plan, stats).

    ``kernel_events`` (optional list) receives (name, start, end) CUDA events
    recorded on the launching stream around every K2/K3 launch.

    Row sharding (parallel.py): ``inp.f``/``inp.guide`` hold image rows
    [row_origin, row_origin + rows_local) of an image of ``H_global`` rows and
    only output rows ``rows = (lo, hi)`` are produced (``out`` is then
    (n, hi-lo, W)).  Kernel pointers are rebased so rows stay global."""
    if params.spatial.kind == GAUSSIAN_RECURSIVE:
        if params.spatial.sigma < 1.0:
            # spatial.py:206-208: below sigma 1 the reference filters with the FIR at radius ceil(3 sigma)
            params = replace(params, spatial=SpatialKernel.gaussian(params.spatial.sigma))
        else:
            if rows is not None or row_origin != 0 or H_global is not None:
                raise NotImplementedError("the recursive Gaussian couples whole columns; row-band sharding "
                                          "covers the box / FIR kernels only")
            return _run_filter_recursive(inp, centroids, params, timer, plane_budget, out, kernel_events)
    n, h_local, W = inp.f.shape
    H = H_global if H_global is not None else h_local
    lo, hi = rows if rows is not None else (0, H)
    S = params.spatial.effective_radius()
    keep: list = []
    lib = _native.lib()
    s = stream_ptr()
    if inflight is not None:
        # the plan is computed in-stream from the landmarks as they land (nys_filter_plan_async);
        # the placeholder M / u0 below are ignored by the native side
        km = inflight.kmeans
        plan = _PENDING_PLAN.get(km.m0)
        if plan is None:
            plan = _PENDING_PLAN[km.m0] = MixingPlan(alphas=np.ones(1), M=np.zeros((km.m0, km.m0)),
                                                     u0=np.zeros(km.m0), alpha0=1.0, eps_den=0.0, rank=km.m0)
        d = _desc(n, inp.rho, H, W, inp.gkind, params.spatial, params.theta, np.zeros((km.m0, km.rho)), plan, keep)
    else:
        plan = mixing_plan(np.asarray(centroids, np.float64), params.theta, params.eps_drop, S, lite=True,
                           device_inverse=True)
        d = _desc(n, inp.rho, H, W, inp.gkind, params.spatial, params.theta, centroids, plan, keep)
    d.row_lo, d.row_hi = row_origin, row_origin + h_local
    wsb = int(lib.nys_filter_workspace_bytes(C.byref(d)))
    if wsb == 0:
        raise NotImplementedError(f"filter shape n={n} rho={inp.rho} m0={d.m0} R={d.radius} not supported")
    ws = workspace(wsb)
    if inflight is not None:
        sb = int(lib.nys_filter_plan_staging_bytes(C.byref(d)))
        inflight.staging = _plan_staging(sb)
        inflight.keep = [ws, keep]
        _native.check(lib.nys_filter_plan_async(C.byref(d), km.centroids_ptr(), float(params.eps_drop), PHI_FORM_COND,
                                                ptr(inflight.staging), sb, ptr(ws), wsb, s), "nys_filter_plan_async")
        inflight.between()
        _native.check(lib.nys_filter_prepare_join(C.byref(d), ptr(inflight.staging), ptr(ws), s),
                      "nys_filter_prepare_join")
    else:
        _native.check(lib.nys_filter_prepare(C.byref(d), ptr(ws), wsb, s), "nys_filter_prepare")
    if timer:
        timer.mark("extrapolation")
    rs = int(lib.nys_filter_plane_row_stride(C.byref(d)))   # [row][x/32][plane][32] (+ raw b planes)
    row_bytes = rs * 4
    if plane_budget is not None:
        budget = plane_budget
    elif (hi - lo + 2 * d.radius) * row_bytes <= SMALL_PLANES_BYTES:
        budget = SMALL_PLANES_BYTES  # single band; skip the (synchronising) free-memory query
    else:
        budget = _plane_budget()
    bands = [Band(b.out0 + lo, b.out_rows, b.hp0 + lo, b.hp_rows)
             for b in plan_bands(hi - lo, d.radius, row_bytes, budget)]
    max_rows = max(b.hp_rows for b in bands)
    planes = torch.empty((max_rows, rs), dtype=torch.float32, device=inp.f.device)
    hps = rs
    if out is None:
        out = torch.empty((n, hi - lo, W), dtype=torch.float32, device=inp.f.device)
    # rebased pointers: image row r of the inputs is local row r - row_origin,
    # output row r is local row r - lo
    f_ptr = ptr(inp.f) - row_origin * W * 4
    g_ptr = ptr(inp.guide) - row_origin * W * 4
    d.out_f64 = 1 if out.dtype == torch.float64 else 0
    o_ptr = _device_view(out) - lo * W * out.element_size()  # a pinned host `out` is written by K3 directly
    f_ps = g_ps = h_local * W
    o_ps = (hi - lo) * W

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    for b in bands:
        e0 = ev() if kernel_events is not None else None
        _native.check(lib.nys_filter_hpass(C.byref(d), f_ptr, f_ps, g_ptr, g_ps, b.out0, b.out_rows,
                                           ptr(planes), hps, ptr(ws), s), "nys_filter_hpass")
        e1 = ev() if kernel_events is not None else None
        _native.check(lib.nys_filter_vpass(C.byref(d), f_ptr, f_ps, g_ptr, g_ps, ptr(planes), hps,
                                           b.out0, b.out_rows, o_ptr, o_ps, ptr(ws), s), "nys_filter_vpass")
        if kernel_events is not None:
            e2 = ev()
            kernel_events.append(("k_feat_hpass", e0, e1, b))
            kernel_events.append(("k_vpass", e1, e2, b))
    if timer:
        timer.mark("convolutions")
    # near-guard FP64 refinement of the pixels K3 queued, then the statistics; stats_ptr: the two
    # doubles go straight to that address (mapped pinned memory), no tensor
    stats = torch.empty(2, dtype=torch.float64, device=inp.f.device) if stats_ptr is None else None
    _native.check(lib.nys_filter_finish(C.byref(d), f_ptr, f_ps, g_ptr, g_ps, o_ptr, o_ps, ptr(ws),
                                        ptr(stats) if stats is not None else stats_ptr, s), "nys_filter_finish")
    del keep
    return out, plan, stats


_PENDING_PLAN: dict = {}


def _run_filter_recursive(inp: _Inputs, centroids: np.ndarray, params: FilterParams, timer, plane_budget, out,
                          kernel_events):
    """Recursive-Gaussian filter (spatial.py:179-191 as the convolution of
    filters.py:223-257): features, row recursion, column recursion fused with
    the contraction, mass^2 scale, guard and division (csrc/nys_recursive.cu).
    Landmark bands are sized so the plane buffer fits ``plane_budget``."""
    n, H, W = inp.f.shape
    S = params.spatial.effective_radius()
    plan = mixing_plan(np.asarray(centroids, np.float64), params.theta, params.eps_drop, S, lite=True,
                       device_inverse=True)
    keep: list = []
    d = _desc(n, inp.rho, H, W, inp.gkind, params.spatial, params.theta, centroids, plan, keep)
    lib = _native.lib()
    wsb = int(lib.nys_filter_workspace_bytes(C.byref(d)))
    if wsb == 0:
        raise NotImplementedError(f"filter shape n={n} rho={inp.rho} m0={d.m0} not supported")
    ws = workspace(wsb)
    s = stream_ptr()
    _native.check(lib.nys_filter_prepare(C.byref(d), ptr(ws), wsb, s), "nys_filter_prepare")
    if timer:
        timer.mark("extrapolation")
    budget = plane_budget if plane_budget is not None else SMALL_PLANES_BYTES
    full = int(lib.nys_filter_recursive_scratch_bytes(C.byref(d), 0))  # preferred path, all landmarks at once
    if full > budget and plane_budget is None:
        budget = max(budget, _plane_budget())
    if full <= budget:
        sb = full
    else:  # banded global-memory path
        nb = d.m0 + 1
        while nb > 1 and int(lib.nys_filter_recursive_scratch_bytes(C.byref(d), nb)) > budget:
            nb = max(1, nb // 2) if nb > 8 else nb - 1
        sb = int(lib.nys_filter_recursive_scratch_bytes(C.byref(d), nb))
    scratch = torch.empty(sb, dtype=torch.uint8, device=inp.f.device)
    if out is None:
        out = torch.empty((n, H, W), dtype=torch.float32, device=inp.f.device)
    e0 = torch.cuda.Event(enable_timing=True) if kernel_events is not None else None
    if e0 is not None:
        e0.record()
    _native.check(lib.nys_filter_recursive(C.byref(d), ptr(inp.f), H * W, ptr(inp.guide), H * W,
                                           _device_view(out), H * W, ptr(scratch), sb, ptr(ws), s),
                  "nys_filter_recursive")
    if kernel_events is not None:
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        kernel_events.append(("k_recursive", e0, e1, None))
    if timer:
        timer.mark("convolutions")
    stats = torch.empty(2, dtype=torch.float64, device=inp.f.device)
    _native.check(lib.nys_filter_stats(C.byref(d), ptr(ws), ptr(stats), s), "nys_filter_stats")
    del keep
    return out, plan, stats


def _plane_budget() -> int:
    free, _total = torch.cuda.mem_get_info()
    return int(min(PLANE_BUDGET_BYTES, max(256 << 20, free * 0.7)))


def _stats_host(stats: torch.Tensor) -> tuple[float, int]:
    h = stats.cpu()
    return float(h[0]), int(h[1:].view(torch.int64)[0])


def _device_view(t: torch.Tensor) -> int:
    if t.is_cuda:
        return ptr(t)
    dev = C.c_void_p()
    _native.check(_native.lib().nys_device_view(ptr(t), C.byref(dev)), "nys_device_view (pinned host output)")
    return int(dev.value)


def _output_buffer(f: Image, out: torch.Tensor | None, params: FilterParams | None = None) -> torch.Tensor | None:
    """Where K3 writes: the caller's `out` (device or page-locked host float32
    (n, H, W)), else a fresh page-locked host tensor for pinned host input (the
    device->host transfer then overlaps the vertical pass), else -- for the
    reference's NumPy float64 Image -- a page-locked float64 host array that K3
    fills directly (no device->host copy, no host cast), else None (device
    buffer from run_filter)."""
    shape = (f.channels, f.height, f.width)
    if out is not None:
        if (not isinstance(out, torch.Tensor) or out.dtype != torch.float32 or tuple(out.shape) != shape
                or not out.is_contiguous() or not (out.is_cuda or out.is_pinned())):
            raise ValueError(f"out must be a contiguous float32 {shape} CUDA or pinned host tensor")
        return out
    if f.is_tensor and not f.on_device and f.data.is_pinned():
        return torch.empty(shape, dtype=torch.float32, pin_memory=True)
    if not f.is_tensor and (params is None or params.spatial.kind != GAUSSIAN_RECURSIVE
                            or params.spatial.sigma < 1.0):
        # K3 writes the float64 planes in HBM; one DMA (queued before the step's wait,
        # _queue_host_copy) brings them to page-locked host memory -- scattered 32-byte writes
        # over PCIe from K3 itself ran at a fraction of the DMA rate
        return torch.empty(shape, dtype=torch.float64, device=require_cuda())
    return None


def _queue_host_copy(out: torch.Tensor, f: Image) -> torch.Tensor:
    """For a NumPy input: queue the device float64 output's copy into page-locked host memory on
    the current stream (before the caller's wait) and return the host tensor."""
    if f.is_tensor or not out.is_cuda or out.dtype != torch.float64:
        return out
    host = torch.empty(out.shape, dtype=torch.float64, pin_memory=True)
    host.copy_(out, non_blocking=True)
    return host


def _output_image(out: torch.Tensor, f: Image, given: torch.Tensor | None = None) -> Image:
    """Output in the caller's container: device tensor stays on the device, a
    host tensor (e.g. pinned) gets a host float32 tensor, NumPy gets the
    reference's float64 ndarray."""
    if not out.is_cuda and out.dtype == torch.float64:  # the float64 planes, already in page-locked host memory
        return Image.trusted(out.numpy(), f.range_max)
    if given is not None or f.on_device or not out.is_cuda:  # caller's buffer / device in / pinned host in place
        return Image(data=out, range_max=f.range_max)
    if f.is_tensor:
        host = torch.empty(out.shape, dtype=torch.float32, pin_memory=f.data.is_pinned())
        host.copy_(out)
        return Image(data=host, range_max=f.range_max)
    return Image(data=out.double().cpu().numpy(), range_max=f.range_max)


def _select_landmarks(inp: _Inputs, params: FilterParams):
    """(centroids on the host, quant_error as a float or a pending device
    scalar).  For k-means the final exact pass is queued behind the centroids'
    device->host copy, so it runs while the host builds the mixing plan."""
    if params.landmark_strategy == STRATEGY_KMEANS:
        km = kmeans_device(inp.points, params.m0, seed=params.seed, max_iter=params.kmeans_max_iter,
                           queue_exact=True)
        return km.centroids, km.quant_error_dev
    rng = np.random.default_rng(params.seed)
    m = inp.points.shape[1]
    idx = rng.choice(m, size=params.m0, replace=False)
    centroids = inp.points[:, torch.as_tensor(idx, device=inp.points.device)].t().double().cpu().numpy()
    _, qe = exact_assignment(inp.points, centroids, want_assignment=False)
    return centroids, qe


def fast_filter(f: Image, p, params: FilterParams, *, kernel_events: list | None = None,
                out: torch.Tensor | None = None) -> FilterReport:
    """Low-rank kernel filter, Algorithm 1 (filters.py:199-274), on the B200.

    ``out`` (optional, an extension of the reference signature): a contiguous
    float32 (n, H, W) CUDA or page-locked host tensor that receives the output,
    e.g. a reused pinned buffer for streaming host frames."""
    stamp("fast_filter")
    _check_sizes(f, p)
    n, H, W = f.channels, f.height, f.width
    if params.m0 > H * W:
        raise ValueError(f"m0 = {params.m0} exceeds the pixel count {H * W}")
    require_cuda()
    timer = StageTimer()
    stamp("timer")
    timer.mark("start")
    stamp("mark start")
    inp = _prepare_inputs(f, p)
    stamp("prepare_inputs")
    if not (f.on_device and (p is f or getattr(p, "on_device", True))):
        timer.mark("upload")  # a host image was copied in (device inputs: upload is 0)
    stamp("mark upload")
    if _pipelined_ok(inp, params):
        rep = _fast_filter_pipelined(f, inp, params, timer, kernel_events, out)
        if rep is not None:
            return rep
        timer = StageTimer()  # the speculation missed (rare): the synchronous path below redoes the step
        timer.mark("start")
        timer.mark("upload")
    centroids, qe = _select_landmarks(inp, params)
    timer.mark("clustering")
    timer.mark("eigendecomposition")  # host eig happens inside run_filter's mixing_plan
    out_given = out
    out, plan, stats = run_filter(inp, centroids, params, timer, kernel_events=kernel_events,
                                  out=_output_buffer(f, out, params))
    out = _queue_host_copy(out, f)
    if isinstance(qe, torch.Tensor):  # the deferred exact pass rides along with the statistics copy
        stats = torch.cat([stats, qe])
        h = stats.cpu()
        qe = float(h[2])
        min_den, guarded = float(h[0]), int(h[1:2].view(torch.int64)[0])
    else:
        min_den, guarded = _stats_host(stats)  # synchronises: a host `out` is complete after this
    timer.mark("normalization")  # fused into K3
    t = timer.elapsed()
    timings = {k: t.get(k, 0.0) for k in ("clustering", "eigendecomposition", "extrapolation", "convolutions",
                                          "normalization")}
    timings["upload"] = t.get("upload", 0.0)
    timings["total"] = sum(t.values())
    return FilterReport(output=_output_image(out, f, given=out_given), timings=timings, retained_rank=plan.rank,
                        quant_error=qe, min_denominator=min_den, guarded_pixels=guarded, centroids=centroids)


def _result_slots() -> tuple[torch.Tensor, int]:
    """Per (host thread, stream) mapped pinned buffer of 3 doubles and its device address."""
    cache = _tls_dict("results")
    key = stream_ptr()
    e = cache.get(key)
    if e is None:
        t = torch.zeros(4, dtype=torch.float64, pin_memory=True)
        e = cache[key] = (t, _device_view(t))
    return e


def _pipelined_ok(inp: _Inputs, params: FilterParams) -> bool:
    """The whole step can be queued without the host waiting: k-means landmarks, a
    box / FIR spatial kernel."""
    sk = params.spatial
    if os.environ.get("NYS_PIPELINED", "1") == "0":  # A/B switch: the synchronous plan
        return False
    return params.landmark_strategy == STRATEGY_KMEANS and (sk.kind != GAUSSIAN_RECURSIVE or sk.sigma < 1.0)


def _fast_filter_pipelined(f: Image, inp: _Inputs, params: FilterParams, timer: StageTimer, kernel_events,
                           out) -> FilterReport | None:
    """fast_filter with the mixing plan computed in-stream (nys_filter_plan_async):
    k-means, the landmarks' copy to pinned memory, the plan on the library's worker thread
    overlapping the exact pass, the device inverse, K2 and K3 are all queued
    before the host waits once, for the statistics.  The plan speculates on the
    common case (nothing dropped, y-form); None when it missed or k-means++ hit
    a zero total (the caller then reruns the synchronous path)."""
    pk = kmeans_device(inp.points, params.m0, seed=params.seed, max_iter=params.kmeans_max_iter, pipelined=True)
    timer.mark("clustering")
    timer.mark("eigendecomposition")  # on the host, in-stream (the library's plan worker thread)
    n_events = len(kernel_events) if kernel_events is not None else 0
    # min|eta|, guarded count and quant_error land in one mapped pinned buffer, written by the
    # statistics kernel and the exact pass's final sum: no gather kernel, no copy at the end
    hres, hres_dev = _result_slots()
    # the exact pass is queued between the plan's fork and its join on the same stream, so it
    # runs while the worker computes the plan (a side stream for it let rare multi-ms stalls
    # into the second timed step: 2 of 9 bench runs, none of 9 on one stream)

    def between():
        exact_assignment_async(inp.points, pk.res, params.m0, pk.workspace, out_ptr=hres_dev + 16)

    fl = _Inflight(kmeans=pk, between=between)
    out_given = out
    out, _, _ = run_filter(inp, None, params, timer, kernel_events=kernel_events, out=_output_buffer(f, out, params),
                           inflight=fl, stats_ptr=hres_dev)
    timer.mark("normalization")  # fused into K3; stamped before the wait so elapsed() needs no further sync
    out = _queue_host_copy(out, f)
    timer.stream.synchronize()  # the step's only host wait
    h = hres.numpy().copy()
    res = fl.result()
    # guarded == -1: the device gate timed out waiting for the plan (nys_filter_finish sentinel)
    if res.status != _native.NYS_OK or pk.zero_total_draw() >= 0 or int(h[1:2].view(np.int64)[0]) < 0:
        if kernel_events is not None:
            del kernel_events[n_events:]
        return None
    m0, rho = params.m0, pk.rho
    centroids = pk.host[:m0 * rho].numpy().reshape(m0, rho).copy()
    return FilterReport(output=_output_image(out, f, given=out_given), timings=timer.lazy(_report_timings),
                        retained_rank=int(res.rank), quant_error=float(h[2]), min_denominator=float(h[0]),
                        guarded_pixels=int(h[1:2].view(np.int64)[0]), centroids=centroids)


def _report_timings(t: dict) -> dict:
    timings = {k: t.get(k, 0.0) for k in ("clustering", "eigendecomposition", "extrapolation", "convolutions",
                                          "normalization")}
    timings["upload"] = t.get("upload", 0.0)
    timings["total"] = sum(t.values())
    return timings


def filter_with_landmarks(f: Image, p, centroids, params: FilterParams) -> FilterReport:
    """Stage-1 parity boundary: the filter given landmarks
    (e.g. the reference's own k-means centroids)."""
    _check_sizes(f, p)
    require_cuda()
    timer = StageTimer()
    timer.mark("start")
    inp = _prepare_inputs(f, p)
    C_ = np.ascontiguousarray(np.asarray(centroids, dtype=np.float64))
    if C_.ndim != 2 or C_.shape[1] != inp.rho:
        raise ValueError(f"landmark dim {C_.shape[-1]} != guide dim {inp.rho}")
    timer.mark("upload")
    out, plan, stats = run_filter(inp, C_, params, timer, out=_output_buffer(f, None, params))
    out = _queue_host_copy(out, f)
    min_den, guarded = _stats_host(stats)
    _, qe = exact_assignment(inp.points, C_, want_assignment=False)
    timer.mark("normalization")
    t = timer.elapsed()
    t["total"] = sum(t.values())
    return FilterReport(output=_output_image(out, f), timings=t, retained_rank=plan.rank,
                        quant_error=qe, min_denominator=min_den, guarded_pixels=guarded, centroids=C_)


def brute_force_filter(f: Image, p, params: FilterParams) -> Image:
    """Direct evaluation of Eq. (1) over the (2S+1)^2 window, the exact
    filter the Nystrom path approximates (filters.py:116-138), on the B200
    (csrc/nys_brute.cu).  A recursive-Gaussian spatial kernel is evaluated as
    its truncated FIR counterpart at radius ceil(3 sigma), as in the
    reference.  Output container follows the input (see fast_filter)."""
    _check_sizes(f, p)
    require_cuda()
    f_dev = to_device_f32(f.data)
    n, H, W = f_dev.shape
    if isinstance(p, PatchGuide):
        g_dev = p.device_planes(f_dev if p.source is f else None)
    elif p is f or (isinstance(p, Image) and p.data is f.data):
        g_dev = f_dev
    else:
        g_dev = to_device_f32(p.data)
    rho = g_dev.shape[0]
    d = _native.FilterDesc()
    d.n, d.rho, d.H, d.W, d.guide_kind = n, rho, H, W, 0
    sp = params.spatial
    if sp.kind == BOX:
        d.spatial_kind, d.radius, d.sigma = _native.NYS_SPATIAL_BOX, sp.radius, 0.0
    elif sp.kind == GAUSSIAN_FIR:
        d.spatial_kind, d.radius, d.sigma = _native.NYS_SPATIAL_GAUSSIAN_FIR, sp.radius, sp.sigma
    else:  # the window is the FIR at ceil(3 sigma) for every sigma (filters.py:107-113)
        d.spatial_kind, d.radius, d.sigma = _native.NYS_SPATIAL_GAUSSIAN_FIR, sp.effective_radius(), sp.sigma
    d.m0, d.theta = 1, params.theta
    out = torch.empty((n, H, W), dtype=torch.float32, device=f_dev.device)
    _native.check(_native.lib().nys_brute_force_filter(C.byref(d), ptr(f_dev), H * W, ptr(g_dev), H * W, ptr(out),
                                                       H * W, stream_ptr()), "nys_brute_force_filter")
    return _output_image(out, f)
