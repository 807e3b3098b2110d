"""Landmark selection on the GPU (mirror of reference ``landmarks.py:18-148``).

``kmeans_landmarks`` keeps the reference's contract: k-means++ seeding from
``np.random.default_rng(seed)`` (the host draws exactly the reference's
stream: ``integers(m)`` then one ``random()`` per D^2 draw), Lloyd iterations
until the labels repeat or ``max_iter``, empty-cluster repair, and the final
exact assignment.  All passes over the points run in the K0/K1 CUDA kernels.
"""

from __future__ import annotations

import ctypes as C
import functools
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from ._device import ptr, require_cuda, stamp, stream_ptr, to_device_f32, workspace

DEFAULT_MAX_ITER = 50


@dataclass(frozen=True)
class LandmarkSet:
    """Centroids plus each point's nearest-centroid assignment (landmarks.py:18-34)."""

    centroids: np.ndarray
    assignment: np.ndarray
    quant_error: float
    errors: tuple = ()

    @property
    def count(self) -> int:
        return self.centroids.shape[0]


@dataclass
class DeviceKMeans:
    centroids: np.ndarray          # (m0, rho) float64, host
    quant_error: float
    errors: tuple
    iterations: int
    seed_indices: np.ndarray
    assignment: torch.Tensor | None  # int64 (m,) on device
    centroids_dev: torch.Tensor | None = None  # device result buffer; its first m0 * rho doubles are the centroids
    workspace: torch.Tensor | None = None      # reusable by exact_assignment_async (same m, rho, m0)
    quant_error_dev: torch.Tensor | None = None  # pending exact-pass result (queue_exact)


@functools.lru_cache(maxsize=64)
def _seed_stream_cached(m: int, m0: int, seed: int):
    rng = np.random.default_rng(seed)
    first = int(rng.integers(m))
    uniforms = np.ascontiguousarray(rng.random(m0 - 1) if m0 > 1 else np.zeros(1))
    uniforms.flags.writeable = False
    return first, uniforms


def _seed_stream(m: int, m0: int, seed: int):
    """The reference's k-means++ draws from default_rng(seed) (landmarks.py:63-70):
    integers(m), then one random() per draw.  A pure function of (m, m0, seed),
    cached: building the generator costs ~30 us per call."""
    return _seed_stream_cached(int(m), int(m0), int(seed))


def _replay_zero_total(m: int, m0: int, seed: int, j0: int, device_seeds: np.ndarray) -> np.ndarray:
    """Seed indices when sum(D^2) hit 0 at draw j0: the reference switches to
    rng.integers(m) for that and every later draw (landmarks.py:66-70)."""
    rng = np.random.default_rng(seed)
    rng.integers(m)
    for _ in range(1, j0):
        rng.random()
    seeds = np.array(device_seeds, dtype=np.int64).copy()
    for j in range(j0, m0):
        seeds[j] = int(rng.integers(m))
    return seeds


@dataclass
class PendingKMeans:
    """k-means whose results are still in flight (``kmeans_device(..., pipelined=True)``):
    ``host`` is the page-locked buffer the results land in (its first m0 * rho
    doubles are the centroids, usable by in-stream consumers such as
    nys_filter_plan_async); ``finish()`` parses it once the stream has passed."""
    host: torch.Tensor
    res: torch.Tensor
    workspace: torch.Tensor
    m0: int
    rho: int
    max_iter: int

    def centroids_ptr(self) -> int:
        return int(self.host.data_ptr())

    def zero_total_draw(self) -> int:
        """-1, or the k-means++ draw at which sum(D^2) hit 0 (the caller must redo the
        clustering with the synchronous path, which replays the reference's picks)."""
        o = self.m0 * self.rho + self.max_iter + 1
        return int(self.host[o:o + 4].numpy().view(np.int64)[1])

    def finish(self, quant_error: float | None) -> DeviceKMeans:
        h = self.host.numpy()
        m0, rho, mi = self.m0, self.rho, self.max_iter
        st = h[m0 * rho + mi + 1:m0 * rho + mi + 5].view(np.int64)
        iters = int(st[0])
        return DeviceKMeans(centroids=h[:m0 * rho].reshape(m0, rho).copy(), quant_error=quant_error,
                            errors=tuple(h[m0 * rho:m0 * rho + iters].tolist()), iterations=iters,
                            seed_indices=h[m0 * rho + mi + 5:].view(np.int64).copy(), assignment=None,
                            centroids_dev=self.res, workspace=self.workspace)


_TLS = threading.local()


def _pinned_tls_f64(n: int, key) -> torch.Tensor:
    """Page-locked buffer reused per (host thread, key); released with the thread."""
    cache = getattr(_TLS, "pinned", None)
    if cache is None:
        cache = _TLS.pinned = {}
    buf = cache.get(key)
    if buf is None or buf.numel() < n:
        buf = torch.empty(max(n, 64), dtype=torch.float64, pin_memory=True)
        cache[key] = buf
    return buf[:n]


def _pipelined_buffers(m: int, rho: int, m0: int, nres: int, dev) -> tuple[torch.Tensor, torch.Tensor]:
    cache = getattr(_TLS, "kmbufs", None)
    if cache is None:
        cache = _TLS.kmbufs = {}
    key = (stream_ptr(), m, rho, m0, nres, dev.index)
    e = cache.get(key)
    if e is None:
        if len(cache) > 8:
            cache.clear()
        wsb = int(_native.lib().nys_kmeans_workspace_bytes(m, rho, m0))
        e = cache[key] = (workspace(wsb), torch.empty(nres, dtype=torch.float64, device=dev))
    return e


def kmeans_device(points: torch.Tensor, m0: int, seed: int = 0, max_iter: int = DEFAULT_MAX_ITER,
                  want_assignment: bool = False, defer_exact: bool = False,
                  queue_exact: bool = False, pipelined: bool = False) -> DeviceKMeans | PendingKMeans:
    """k-means on planar device points ``(rho, m)`` float32 (rows may be any
    plane stride; the last dim must be contiguous).

    ``defer_exact``: skip the final exact pass (quant_error is then None);
    the caller launches it with ``exact_assignment_async`` once it has the
    centroids, so the pass overlaps its host-side work.

    ``queue_exact`` (implies defer_exact): the results are copied to a pinned
    host buffer behind an event, the exact pass is queued right after that copy
    (before the host waits), and only the copy is waited for -- the exact pass
    then runs while the caller works on the centroids, with no host gap in
    between.  Its pending result is ``DeviceKMeans.quant_error_dev``.

    ``pipelined`` (no assignment, no exact pass): queue the results' copy to a
    pinned buffer and return a ``PendingKMeans`` without waiting at all."""
    stamp("kmeans_device")
    require_cuda()
    if points.dim() != 2 or points.stride(1) != 1:
        raise ValueError("points must be a (rho, m) tensor with contiguous rows")
    rho, m = int(points.shape[0]), int(points.shape[1])
    if m0 < 1 or m0 > m:
        raise ValueError(f"m0 must be in [1, {m}], got {m0}")
    if max_iter < 1:
        raise ValueError("max_iter must be >= 1")
    if rho > _native.NYS_MAX_RHO_WIDE or m0 > _native.NYS_MAX_M0:
        raise NotImplementedError(f"rho <= {_native.NYS_MAX_RHO_WIDE} and m0 <= {_native.NYS_MAX_M0} on the B200 path")
    stamp("km checks")
    lib = _native.lib()
    dev = points.device
    ps = int(points.stride(0))
    # one device buffer for every small result -> a single D2H copy (one sync); every slot that is
    # read back is written by the kernels, so no zero fill; slots addressed by pointer arithmetic
    # (views cost ~5 us each on the critical path before the first launch)
    nres = m0 * rho + max_iter + 1 + 4 + m0
    if pipelined:
        # reused per (thread, stream, shape): the next call's kernels queue behind this one's
        ws, res = _pipelined_buffers(m, rho, m0, nres, dev)
        wsb = int(ws.numel())
    else:
        wsb = int(lib.nys_kmeans_workspace_bytes(m, rho, m0))
        ws = workspace(wsb)
        res = torch.empty(nres, dtype=torch.float64, device=dev)
    stamp("km workspace")
    base = res.data_ptr()
    Cd_p = base
    errs_p = base + 8 * m0 * rho
    qe_p = base + 8 * (m0 * rho + max_iter)
    stats_p = qe_p + 8
    seeds_p = stats_p + 8 * 4
    asg = torch.empty(m, dtype=torch.int64, device=dev) if want_assignment else None
    first, uniforms = _seed_stream(m, m0, seed)
    stamp("km res+seed")
    if (defer_exact or queue_exact or pipelined) and asg is None:
        qe_p = None
    if pipelined and (asg is not None or qe_p is not None):
        raise ValueError("pipelined k-means returns neither an assignment nor the exact pass")
    _native.check(lib.nys_kmeans_run(ptr(points), ps, m, rho, m0, max_iter, first,
                                     uniforms.ctypes.data, Cd_p, errs_p, stats_p, qe_p,
                                     ptr(asg), seeds_p, ptr(ws), wsb, stream_ptr()), "nys_kmeans_run")
    if pipelined:
        hbuf = _pinned_tls_f64(nres, stream_ptr())
        hbuf.copy_(res, non_blocking=True)
        return PendingKMeans(host=hbuf, res=res, workspace=ws, m0=m0, rho=rho, max_iter=max_iter)
    qe_dev = None
    if queue_exact and qe_p is None:
        hbuf = _pinned_tls_f64(nres, ("kmeans", stream_ptr()))  # per host thread: no cross-thread sharing
        hbuf.copy_(res, non_blocking=True)
        done = torch.cuda.Event()
        done.record()
        qe_dev = exact_assignment_async(points, res, m0, ws)
        done.synchronize()
        h = hbuf.numpy().copy()
    else:
        h = res.cpu().numpy()
    st = h[m0 * rho + max_iter + 1:m0 * rho + max_iter + 5].view(np.int64)
    seeds_h = h[m0 * rho + max_iter + 5:].view(np.int64).copy()
    if st[1] >= 0:  # sum(D^2) == 0 during seeding: redo with the reference's integers() picks
        sidx = _replay_zero_total(m, m0, seed, int(st[1]), seeds_h)
        sidx = np.ascontiguousarray(sidx, dtype=np.int64)
        _native.check(lib.nys_kmeans_run_seeded(ptr(points), ps, m, rho, m0, max_iter, sidx.ctypes.data,
                                                Cd_p, errs_p, stats_p, qe_p, ptr(asg),
                                                ptr(ws), wsb, stream_ptr()), "nys_kmeans_run_seeded")
        h = res.cpu().numpy()
        st = h[m0 * rho + max_iter + 1:m0 * rho + max_iter + 5].view(np.int64)
        seeds_h = sidx
        if qe_dev is not None:  # the queued exact pass saw the first run's centroids
            qe_dev = exact_assignment_async(points, res, m0, ws)
    iters = int(st[0])
    return DeviceKMeans(centroids=h[:m0 * rho].reshape(m0, rho).copy(),
                        quant_error=None if qe_p is None else float(h[m0 * rho + max_iter]),
                        errors=tuple(h[m0 * rho:m0 * rho + iters].tolist()), iterations=iters,
                        seed_indices=seeds_h, assignment=asg, centroids_dev=res, workspace=ws,
                        quant_error_dev=qe_dev)


def _points_planar(points) -> torch.Tensor:
    """(m, dim) host/device points -> planar (dim, m) float32 device tensor."""
    if isinstance(points, torch.Tensor):
        t = points
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(points, dtype=np.float64)))
    if t.dim() != 2:
        raise ValueError("points must be an (m, dim) matrix")
    return to_device_f32(t.t())


def kmeans_landmarks(points, m0: int, seed: int = 0, max_iter: int = DEFAULT_MAX_ITER) -> LandmarkSet:
    """Cluster ``points`` (m, dim) into ``m0`` groups (landmarks.py:76-129)."""
    pts = np.asarray(points) if not isinstance(points, torch.Tensor) else points
    m = int(pts.shape[0])
    if m0 < 1 or m0 > m:
        raise ValueError(f"m0 must be in [1, {m}], got {m0}")
    if max_iter < 1:
        raise ValueError("max_iter must be >= 1")
    res = kmeans_device(_points_planar(points), m0, seed=seed, max_iter=max_iter, want_assignment=True)
    return LandmarkSet(centroids=res.centroids, assignment=res.assignment.cpu().numpy(),
                       quant_error=res.quant_error, errors=res.errors)


def exact_assignment_async(points_planar: torch.Tensor, centroids_dev: torch.Tensor, m0: int,
                           ws: torch.Tensor | None = None, out_ptr: int | None = None) -> torch.Tensor | None:
    """Launch the exact pass (landmarks.py:121-129) against device centroids
    (the first m0 * rho doubles of ``centroids_dev``) and return quant_error as
    a 1-element device tensor, without synchronising.  ``out_ptr``: write the
    double there instead (a device address, e.g. of mapped pinned memory) and
    return None."""
    rho, m = int(points_planar.shape[0]), int(points_planar.shape[1])
    lib = _native.lib()
    dev = points_planar.device
    wsb = int(lib.nys_kmeans_workspace_bytes(m, rho, m0))
    if ws is None or ws.numel() < wsb:
        ws = workspace(wsb)
    Cd = centroids_dev
    qe = torch.empty(1, dtype=torch.float64, device=dev) if out_ptr is None else None
    _native.check(lib.nys_kmeans_exact(ptr(points_planar), int(points_planar.stride(0)), m, rho, ptr(Cd), m0,
                                       None, ptr(qe) if qe is not None else out_ptr, ptr(ws), wsb, stream_ptr()),
                  "nys_kmeans_exact")
    return qe


def exact_assignment(points_planar: torch.Tensor, centroids: np.ndarray, want_assignment: bool = True):
    """Final exact assignment + quant_error on the device (landmarks.py:121-129)."""
    rho, m = int(points_planar.shape[0]), int(points_planar.shape[1])
    m0 = int(centroids.shape[0])
    lib = _native.lib()
    dev = points_planar.device
    wsb = int(lib.nys_kmeans_workspace_bytes(m, rho, m0))
    ws = workspace(wsb)
    Cd = torch.from_numpy(np.ascontiguousarray(centroids, dtype=np.float64)).to(dev)
    asg = torch.empty(m, dtype=torch.int64, device=dev) if want_assignment else None
    qe = torch.zeros(1, dtype=torch.float64, device=dev)
    _native.check(lib.nys_kmeans_exact(ptr(points_planar), int(points_planar.stride(0)), m, rho, ptr(Cd), m0,
                                       ptr(asg), ptr(qe), ptr(ws), wsb, stream_ptr()), "nys_kmeans_exact")
    return asg, float(qe.cpu().numpy()[0])


def uniform_landmarks(points, m0: int, seed: int = 0) -> LandmarkSet:
    """``m0`` rows uniformly without replacement (landmarks.py:132-148)."""
    pts = np.asarray(points, dtype=np.float64) if not isinstance(points, torch.Tensor) else points
    m = int(pts.shape[0])
    if m0 < 1 or m0 > m:
        raise ValueError(f"m0 must be in [1, {m}], got {m0}")
    rng = np.random.default_rng(seed)
    idx = rng.choice(m, size=m0, replace=False)
    host = pts.cpu().numpy() if isinstance(pts, torch.Tensor) else pts
    centroids = np.asarray(host, dtype=np.float64)[idx].copy()
    asg, e = exact_assignment(_points_planar(points), centroids)
    return LandmarkSet(centroids=centroids, assignment=asg.cpu().numpy(), quant_error=e, errors=(e,))
