"""Row-band sharding of one image across ranks.

One process per GPU (torchrun); ``torch.distributed`` carries the plumbing
(NCCL on B200s, gloo in the CPU tests).  Rank g owns image rows
[g*H/G, (g+1)*H/G) (``bands.shard_rows``):

* **halo exchange**: each rank receives R (+1 for the 3x3 NLM patches) input
  rows from each neighbour -- input rows, not filtered planes (a plane row is
  (m0+1)(n+1) times larger);
* **k-means** keeps the reference's *global* semantics (landmarks.py:60-129)
  on the concatenation of the bands in rank order, which is the image's linear
  pixel order:
    - k-means++: every rank draws the same ``default_rng(seed)`` stream; per
      draw the ranks all-gather their local D^2 totals, every rank finds the
      owner of u * total from the rank prefixes, the owner searches its band
      and broadcasts the point;
    - Lloyd: per-rank cluster sums/counts/objective/changed are all-gathered
      and summed in rank order (deterministic), every rank applies the same
      update; empty clusters take the global farthest point (value desc,
      global index asc) exactly like the single-device repair;
* the **filter** bands are then independent: K2/K3 run on the rank's rows
  with the global image height, the halo rows standing in for the
  neighbours' rows (edge replication only at the true image border).

``KMeansOps`` isolates the per-rank device work so the orchestration can be
exercised with gloo on CPU (tests/test_distributed.py).
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _native
from .bands import halo_rows, shard_rows


# ---------------------------------------------------------------------------
# communication adapter (small host arrays; tensors for the halo exchange)
# ---------------------------------------------------------------------------
class Comm:
    """Thin wrapper over an initialised torch.distributed process group."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.backend = dist.get_backend(group)
        self.device = (torch.device("cuda", torch.cuda.current_device())
                       if self.backend == "nccl" else torch.device("cpu"))

    def _t(self, a: np.ndarray) -> torch.Tensor:
        return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).to(self.device)

    def allgather(self, a) -> np.ndarray:
        """(world, *a.shape) float64, rank order."""
        t = self._t(np.atleast_1d(np.asarray(a, dtype=np.float64)))
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t, group=self.group)
        return np.stack([o.cpu().numpy() for o in out])

    def sum_ordered(self, a) -> np.ndarray:
        """Element-wise sum over ranks, accumulated in rank order (deterministic)."""
        g = self.allgather(a)
        s = np.zeros_like(g[0])
        for r in range(self.world):
            s = s + g[r]
        return s

    def bcast(self, a, src: int) -> np.ndarray:
        t = self._t(np.atleast_1d(np.asarray(a, dtype=np.float64)))
        dist.broadcast(t, src, group=self.group)
        return t.cpu().numpy()

    def exchange_halos(self, ext: torch.Tensor, lo: int, hi: int, H: int, halo: int) -> int:
        """Fill the halo rows of this rank's extended band in place.

        ``ext`` (c, ehi - elo, W) with (elo, ehi) = halo_rows(lo, hi, H, halo) already holds
        the rank's own rows at [lo - elo, hi - elo); the rows above / below are received from
        the neighbours (each sends the same count of its edge rows back).  Only halo rows
        move: the own rows stay where the caller put them.  Returns elo."""
        r, w = self.rank, self.world
        elo, ehi = halo_rows(lo, hi, H, halo)
        need_top, need_bot = lo - elo, ehi - hi
        if need_top > (hi - lo) or need_bot > (hi - lo):
            raise ValueError("each shard must own at least `halo` rows")
        c, rows, W = ext.shape
        if rows != ehi - elo:
            raise ValueError(f"extended band must have {ehi - elo} rows, got {rows}")
        nccl = self.backend == "nccl"
        xfer = (lambda t: t.contiguous()) if nccl else (lambda t: t.cpu().contiguous())
        top, own = need_top, hi - lo
        ops, recv = [], []
        if r > 0:
            buf = xfer(torch.empty((c, top, W), dtype=ext.dtype, device=ext.device))
            ops.append(dist.P2POp(dist.isend, xfer(ext[:, top:2 * top]), r - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, buf, r - 1, self.group))
            recv.append((buf, 0))
        if r < w - 1:
            buf = xfer(torch.empty((c, need_bot, W), dtype=ext.dtype, device=ext.device))
            ops.append(dist.P2POp(dist.isend, xfer(ext[:, top + own - need_bot:top + own]), r + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, buf, r + 1, self.group))
            recv.append((buf, top + own))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for buf, row0 in recv:
            ext[:, row0:row0 + buf.shape[1]].copy_(buf, non_blocking=nccl)
        return elo

    def exchange_rows(self, local: torch.Tensor, lo: int, hi: int, H: int, halo: int):
        """Extend ``local`` (c, hi-lo, W) with up to ``halo`` rows from each
        neighbour; returns (extended tensor, first global row).  Allocates the
        band and copies the own rows once; repeated calls should keep the band
        (``extended_band``) and call exchange_halos."""
        ext, top = extended_band(local.shape[0], lo, hi, H, halo, local.shape[2], local.dtype, local.device)
        ext[:, top:top + (hi - lo)].copy_(local)
        return ext, self.exchange_halos(ext, lo, hi, H, halo)


def extended_band(c: int, lo: int, hi: int, H: int, halo: int, W: int, dtype, device) -> tuple[torch.Tensor, int]:
    """An uninitialised (c, rows + halos, W) band for the rows [lo, hi) and the row offset of
    the own rows inside it."""
    elo, ehi = halo_rows(lo, hi, H, halo)
    return torch.empty((c, ehi - elo, W), dtype=dtype, device=device), lo - elo


# ---------------------------------------------------------------------------
# per-rank k-means operations
# ---------------------------------------------------------------------------
class KMeansOps:
    """Per-rank reductions over the local points (rho, m_local); the device
    implementation below calls the step-wise C ABI."""

    m: int
    rho: int

    def pp_update(self, c: np.ndarray, init: bool) -> float: ...
    def pp_pick(self, target: float) -> int: ...
    def point(self, idx: int) -> np.ndarray: ...
    def assign(self, C_: np.ndarray, first: bool) -> np.ndarray: ...
    def farthest(self, C_: np.ndarray, excl: list) -> tuple[float, int]: ...
    def exact(self, C_: np.ndarray) -> float: ...


class DeviceKMeansOps(KMeansOps):
    """C-ABI step-wise kernels (nys_kmeanspp_update / _pick / nys_kmeans_assign /
    _farthest / _exact / nys_gather_point) on a CUDA tensor of local points."""

    def __init__(self, points: torch.Tensor, m0: int):
        from ._device import ptr, stream_ptr, workspace

        self._ptr, self._stream = ptr, stream_ptr
        self.pts = points
        self.rho, self.m = int(points.shape[0]), int(points.shape[1])
        self.ps = int(points.stride(0))
        self.m0 = m0
        lib = _native.lib()
        self.lib = lib
        self.wsb = int(lib.nys_kmeans_workspace_bytes(self.m, self.rho, max(m0, 1)))
        self.ws = workspace(self.wsb)
        dev = points.device
        self.d2 = torch.empty(self.m, dtype=torch.float64, device=dev)
        self.labels = torch.zeros(self.m, dtype=torch.int32, device=dev)
        self.scalar = torch.zeros(4, dtype=torch.float64, device=dev)
        self.idx = torch.zeros(1, dtype=torch.int64, device=dev)
        self.acc = torch.zeros(m0 * (self.rho + 1) + 2, dtype=torch.float64, device=dev)

    def _c(self, C_: np.ndarray) -> torch.Tensor:
        return torch.from_numpy(np.ascontiguousarray(C_, dtype=np.float64)).to(self.pts.device)

    def pp_update(self, c, init):
        p = self._ptr
        ct = self._c(c)
        _native.check(self.lib.nys_kmeanspp_update(p(self.pts), self.ps, self.m, self.rho, p(ct), int(init),
                                                   p(self.d2), p(self.scalar), p(self.ws), self.wsb, self._stream()),
                      "nys_kmeanspp_update")
        return float(self.scalar[0].item())

    def pp_pick(self, target):
        p = self._ptr
        _native.check(self.lib.nys_kmeanspp_pick(p(self.d2), self.m, float(target), p(self.idx), p(self.ws),
                                                 self.wsb, self._stream()), "nys_kmeanspp_pick")
        return int(self.idx.item())

    def point(self, idx):
        return self.pts[:, int(idx)].double().cpu().numpy()

    def assign(self, C_, first):
        p = self._ptr
        ct = self._c(C_)
        _native.check(self.lib.nys_kmeans_assign(p(self.pts), self.ps, self.m, self.rho, p(ct), C_.shape[0],
                                                 p(self.labels), int(first), p(self.acc), p(self.ws), self.wsb,
                                                 self._stream()), "nys_kmeans_assign")
        return self.acc.cpu().numpy().copy()

    def farthest(self, C_, excl):
        p = self._ptr
        ct = self._c(C_)
        ex = torch.tensor(list(excl) or [0], dtype=torch.int64, device=self.pts.device)
        _native.check(self.lib.nys_kmeans_farthest(p(self.pts), self.ps, self.m, self.rho, p(ct), C_.shape[0],
                                                   p(self.labels), p(ex), len(excl), p(self.scalar), p(self.ws),
                                                   self.wsb, self._stream()), "nys_kmeans_farthest")
        v = self.scalar[:2].cpu().numpy()
        return float(v[0]), int(v[1])

    def exact(self, C_):
        p = self._ptr
        ct = self._c(C_)
        _native.check(self.lib.nys_kmeans_exact(p(self.pts), self.ps, self.m, self.rho, p(ct), C_.shape[0], None,
                                                p(self.scalar), p(self.ws), self.wsb, self._stream()),
                      "nys_kmeans_exact")
        return float(self.scalar[0].item())


@dataclass
class ShardedKMeans:
    centroids: np.ndarray
    quant_error: float
    errors: tuple
    seed_indices: np.ndarray


def distributed_kmeans(ops: KMeansOps, comm: Comm, m0: int, seed: int = 0, max_iter: int = 50) -> ShardedKMeans:
    """Global k-means over the rank-ordered concatenation of the local points
    (landmarks.py:60-129 semantics)."""
    counts = comm.allgather(float(ops.m))[:, 0].astype(np.int64)
    offs = np.concatenate([[0], np.cumsum(counts)])
    m = int(offs[-1])
    rho = ops.rho
    if m0 < 1 or m0 > m:
        raise ValueError(f"m0 must be in [1, {m}], got {m0}")
    if max_iter < 1:
        raise ValueError("max_iter must be >= 1")
    me = comm.rank

    def owner_of(gidx: int) -> int:
        return int(np.searchsorted(offs, gidx, side="right") - 1)

    def fetch(gidx: int) -> np.ndarray:
        r = owner_of(gidx)
        pt = ops.point(gidx - offs[r]) if r == me else np.zeros(rho)
        return comm.bcast(pt, r)

    rng = np.random.default_rng(seed)
    C_ = np.empty((m0, rho))
    seeds = np.empty(m0, dtype=np.int64)
    seeds[0] = int(rng.integers(m))
    C_[0] = fetch(seeds[0])
    zero = False
    for j in range(1, m0):
        if not zero:
            local = ops.pp_update(C_[j - 1], init=(j == 1))
            totals = comm.allgather(local)[:, 0]
            total = 0.0
            for t in totals:
                total += t
            zero = not total > 0.0
        if zero:  # sum(D^2) == 0: rng.integers(m) from here on (landmarks.py:69-70)
            gidx = int(rng.integers(m))
        else:
            target = rng.random() * total
            pre = 0.0
            r_star, last_pos, pre_last = None, None, 0.0
            for r, t in enumerate(totals):
                if t > 0.0:
                    last_pos, pre_last = r, pre
                if pre + t > target:
                    r_star = r
                    break
                pre += t
            if r_star is None:  # rounding pushed target past the end
                r_star, pre = last_pos, pre_last
                target = pre + totals[r_star] * (1.0 - 1e-16)
            li = ops.pp_pick(target - pre) if me == r_star else 0
            gidx = int(comm.bcast(float(offs[r_star] + max(li, 0)), r_star)[0])
        seeds[j] = gidx
        C_[j] = fetch(gidx)

    errors = []
    slots = m0 * (rho + 1)
    for it in range(max_iter):
        acc = comm.sum_ordered(ops.assign(C_, first=(it == 0)))
        errors.append(float(acc[slots]))
        if it > 0 and acc[slots + 1] == 0:
            break
        prev = C_.copy()
        sums = acc[:slots].reshape(m0, rho + 1)
        occ = sums[:, rho] > 0
        C_[occ] = sums[occ, :rho] / sums[occ, rho:rho + 1]
        excl_local: list[int] = []
        for j in np.flatnonzero(~occ):  # empty-cluster repair (landmarks.py:114-119)
            v, li = ops.farthest(prev, excl_local)
            g = comm.allgather(np.array([v, float(offs[me] + li)]))
            best_v, best_i = -np.inf, m
            for r in range(comm.world):
                if g[r, 0] > best_v or (g[r, 0] == best_v and g[r, 1] < best_i):
                    best_v, best_i = g[r, 0], int(g[r, 1])
            C_[j] = fetch(best_i)
            if owner_of(best_i) == me:
                excl_local.append(best_i - int(offs[me]))
    qe = float(comm.sum_ordered(ops.exact(C_))[0])
    return ShardedKMeans(centroids=C_, quant_error=qe, errors=tuple(errors), seed_indices=seeds)


def device_distributed_kmeans(points: torch.Tensor, comm: Comm, m0: int, seed: int = 0,
                              max_iter: int = 50) -> ShardedKMeans | None:
    """distributed_kmeans with every decision taken on the device: per k-means++ draw an
    all-gather of the ranks' D^2 totals and an all-reduce of the owner's candidate point,
    per Lloyd iteration one all-reduce of the cluster sums / counts / objective / changed
    count (the reference's update and break rule then run on the device,
    landmarks.py:60-129); the host waits once, at the end.  Returns None when the run
    needs the host-orchestrated path (a zero D^2 total -- the reference then draws with
    integers(m) -- or an empty cluster, whose repair needs the global farthest point)."""
    from ._device import ptr, stream_ptr, workspace

    lib = _native.lib()
    dev = points.device
    rho, m_loc = int(points.shape[0]), int(points.shape[1])
    ps = int(points.stride(0))
    counts = comm.allgather(float(m_loc))[:, 0].astype(np.int64)
    offs = np.concatenate([[0], np.cumsum(counts)])
    m = int(offs[-1])
    if m0 < 1 or m0 > m:
        raise ValueError(f"m0 must be in [1, {m}], got {m0}")
    if max_iter < 1:
        raise ValueError("max_iter must be >= 1")
    me, world = comm.rank, comm.world
    wsb = int(lib.nys_kmeans_workspace_bytes(m_loc, rho, m0))
    ws = workspace(wsb)
    s = stream_ptr()
    # cands[j] = (landmark j, its global index): the owner of draw j writes its row, the others
    # zeros, and an all-reduce(sum) hands it to every rank; the next draw's D^2 update reads it
    # in place (a one-member group needs no collective at all)
    cands = torch.zeros((m0, rho + 1), dtype=torch.float64, device=dev)
    C_ = torch.zeros((m0, rho), dtype=torch.float64, device=dev)
    reduce = (lambda t: dist.all_reduce(t, group=comm.group)) if world > 1 else (lambda t: None)
    d2 = torch.empty(m_loc, dtype=torch.float64, device=dev)
    mytot = torch.zeros(1, dtype=torch.float64, device=dev)
    totals = torch.zeros(world, dtype=torch.float64, device=dev)
    tot = torch.zeros(m0 * rho + m0 + 1, dtype=torch.int64, device=dev)  # fixed-point sums, counts, changed
    obj = torch.zeros(1, dtype=torch.float64, device=dev)
    # the single-device kernel's fixed-point scale over the global points: 2^sexp,
    # sexp = 61 - ilogb(max|x| * m) - 1 (nys_kmeans_coop.cu)
    mx = points.abs().max().reshape(1).double() if m_loc > 0 else torch.zeros(1, dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=comm.group)
    maxabs = float(np.float32(mx.item()))
    sexp = 61 - int(np.frexp(maxabs * float(m))[1] - 1) - 1 if maxabs > 0 else 0
    errors = torch.zeros(max_iter, dtype=torch.float64, device=dev)
    stats = torch.zeros(4, dtype=torch.int64, device=dev)
    qe = torch.zeros(1, dtype=torch.float64, device=dev)
    chk = _native.check
    chk(lib.nys_kmeans_state_init(ptr(ws), wsb, m_loc, rho, m0, s), "nys_kmeans_state_init")
    rng = np.random.default_rng(seed)
    first = int(rng.integers(m))
    owner0 = int(np.searchsorted(offs, first, side="right") - 1)
    if owner0 == me:
        chk(lib.nys_gather_point(ptr(points), ps, rho, first - int(offs[me]), ptr(cands[0]), s), "nys_gather_point")
        cands[0, rho] = float(first)
    reduce(cands[0])
    for j in range(1, m0):
        u = float(rng.random())  # one random() per draw, as Generator.choice consumes it
        chk(lib.nys_kmeanspp_update(ptr(points), ps, m_loc, rho, ptr(cands[j - 1]), int(j == 1), ptr(d2),
                                    ptr(mytot if world > 1 else totals), ptr(ws), wsb, s), "nys_kmeanspp_update")
        if world > 1:
            dist.all_gather_into_tensor(totals, mytot, group=comm.group)
        chk(lib.nys_kmeanspp_owner_pick(ptr(points), ps, m_loc, rho, m0, ptr(d2), ptr(totals), world, me,
                                        int(offs[me]), u, j, ptr(cands[j]), ptr(ws), wsb, s), "nys_kmeanspp_owner_pick")
        reduce(cands[j])
    C_.copy_(cands[:, :rho])
    seeds = cands[:, rho]
    for it in range(max_iter):
        chk(lib.nys_kmeans_lloyd_local(ptr(points), ps, m_loc, rho, ptr(C_), m0, it, sexp, ptr(tot), ptr(obj),
                                       ptr(ws), wsb, s), "nys_kmeans_lloyd_local")
        reduce(tot)
        reduce(obj)
        chk(lib.nys_kmeans_lloyd_update(m_loc, rho, m0, it, sexp, ptr(tot), ptr(obj), ptr(C_), ptr(errors), ptr(ws),
                                        wsb, s), "nys_kmeans_lloyd_update")
    chk(lib.nys_kmeans_exact(ptr(points), ps, m_loc, rho, ptr(C_), m0, None, ptr(qe), ptr(ws), wsb, s),
        "nys_kmeans_exact")
    reduce(qe)
    chk(lib.nys_kmeans_state_read(ptr(ws), m_loc, rho, m0, ptr(stats), s), "nys_kmeans_state_read")
    st = stats.cpu().numpy()  # the one host wait
    if st[1] >= 0 or st[3] < 0:
        return None
    iters = int(st[0])
    return ShardedKMeans(centroids=C_.cpu().numpy(), quant_error=float(qe.cpu()[0]),
                         errors=tuple(errors[:iters].cpu().numpy().tolist()),
                         seed_indices=seeds.cpu().numpy().astype(np.int64))


# ---------------------------------------------------------------------------
# sharded filter
# ---------------------------------------------------------------------------
def sharded_fast_filter(f_local: torch.Tensor | None, H: int, params, comm: Comm, nlm: bool = False,
                        f_ext: torch.Tensor | None = None):
    """Filter this rank's rows of a row-sharded image.

    ``f_local`` (n, rows, W) holds image rows shard_rows(H, world, rank); or pass
    ``f_ext``, the rank's extended band (parallel.extended_band) with the own rows already
    in place, which is then reused across calls (only the halo rows move).
    Returns (out_local (n, rows, W), report dict)."""
    from .filters import _Inputs, run_filter
    from ._device import ptr, stream_ptr

    lo, hi = shard_rows(H, comm.world, comm.rank)
    R = params.spatial.effective_radius()
    halo = R + (1 if nlm else 0)
    if f_ext is None:
        if f_local.shape[1] != hi - lo:
            raise ValueError("f_local rows do not match this rank's shard")
        ext, elo = comm.exchange_rows(f_local, lo, hi, H, halo)
    else:
        ext = f_ext
        elo = comm.exchange_halos(ext, lo, hi, H, halo)
        f_local = ext[:, lo - elo:hi - elo]
    n, _, W = ext.shape
    if nlm:
        # raw 3x3xn patches of the own rows, gathered from the extended band
        from .filters import PatchGuide  # noqa: F401  (same gather as the single-device path)
        rho = n * 9
        er = ext.shape[1]
        pl = torch.empty((rho, er, W), dtype=torch.float32, device=ext.device)
        _native.call("nys_patch_guide", ptr(ext), er * W, n, er, W, 1, ptr(pl), er * W, stream_ptr())
        # rows of the extended band that are interior to the image are exact; the
        # own rows never touch the band's artificial top/bottom edge (halo >= 1)
        points = pl[:, lo - elo:hi - elo].reshape(rho, -1).contiguous()
        inp = _Inputs(f=ext, guide=ext, gkind=1, points=points, rho=rho)
    else:
        # the own rows of the band, planar (rho, m_local) with the band's plane stride: k-means
        # reads them in place (plane stride = band rows x W)
        points = ext.reshape(n, -1)[:, (lo - elo) * W:(hi - elo) * W]
        inp = _Inputs(f=ext, guide=ext, gkind=0, points=points, rho=n)
    km = None
    if comm.world == 1 and os.environ.get("NYS_SHARD_STEPWISE", "0") != "1":
        # one rank holds every point: the single-device cooperative k-means (no collective to make)
        from .landmarks import kmeans_device

        r = kmeans_device(points, params.m0, seed=params.seed, max_iter=params.kmeans_max_iter)
        km = ShardedKMeans(centroids=r.centroids, quant_error=float(r.quant_error), errors=tuple(r.errors),
                           seed_indices=np.asarray(getattr(r, "seed_indices", np.zeros(0)), np.int64))
    elif comm.backend == "nccl":  # device-resident collectives (gloo keeps the host-orchestrated path)
        km = device_distributed_kmeans(points, comm, params.m0, params.seed, params.kmeans_max_iter)
    if km is None:
        km = distributed_kmeans(DeviceKMeansOps(points, params.m0), comm, params.m0, params.seed,
                                params.kmeans_max_iter)
    out, plan, stats = run_filter(inp, km.centroids, params, rows=(lo, hi), row_origin=elo, H_global=H)
    st = stats.cpu()
    min_den = float(comm.allgather(float(st[0]))[:, 0].min())
    guarded = int(round(comm.sum_ordered(float(st[1:].view(torch.int64)[0]))[0]))
    return out, dict(centroids=km.centroids, quant_error=km.quant_error, errors=km.errors,
                     retained_rank=plan.rank, min_denominator=min_den, guarded_pixels=guarded)


def bench_sharded(args, wl, rank: int, world: int):
    """bench.py --gpus N: one image row-sharded over N ranks (strong scaling).

    ``value`` times the sharded step with every rank's rows resident in HBM;
    ``e2e`` adds, per step, each rank's pinned-host -> device copy of its rows
    and the device -> pinned-host copy of its output rows.  Both are the max
    over ranks of CUDA-event times between barriers."""
    import time

    from bench import ClockSampler
    from paper_1901_06112_b200 import FilterParams, SpatialKernel, _native

    dev = torch.device("cuda", torch.cuda.current_device())
    comm = Comm()
    H, W = wl.H, wl.W
    lo, hi = shard_rows(H, world, rank)
    f_full = wl.image(seed=0)
    f_host = torch.from_numpy(np.ascontiguousarray(f_full[:, lo:hi])).pin_memory()
    del f_full
    sk = SpatialKernel.box(wl.radius) if wl.spatial == "box" else SpatialKernel.gaussian(wl.sigma, wl.radius)
    params = FilterParams(spatial=sk, theta=float(wl.theta), m0=wl.m0, seed=0, kmeans_max_iter=wl.max_iter)
    nlm = wl.mode == "nlm"
    # the rank's rows live in its extended band for the whole run: a step moves only halo rows
    halo = params.spatial.effective_radius() + (1 if nlm else 0)
    f_ext, top = extended_band(f_host.shape[0], lo, hi, H, halo, W, torch.float32, dev)
    f_ext[:, top:top + (hi - lo)].copy_(f_host)
    for _ in range(args.warmup):
        sharded_fast_filter(None, H, params, comm, nlm, f_ext=f_ext)
    torch.cuda.synchronize()
    dist.barrier()

    def timed(step):
        ms = []
        for _ in range(args.steps):
            dist.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            res = step()
            e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1)], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms.append(float(t.item()))
        return sum(ms) / len(ms), res

    lib = _native.lib()
    l0 = int(lib.nys_kernel_launches())
    with ClockSampler(torch.cuda.current_device()) as clk:
        ms, (out, rep) = timed(lambda: sharded_fast_filter(None, H, params, comm, nlm, f_ext=f_ext))
    launches = (int(lib.nys_kernel_launches()) - l0) // max(1, args.steps)
    out_host = torch.empty(out.shape, dtype=torch.float32, pin_memory=True)

    def e2e_step():
        f_ext[:, top:top + (hi - lo)].copy_(f_host, non_blocking=True)  # the own rows, into the band
        o, r = sharded_fast_filter(None, H, params, comm, nlm, f_ext=f_ext)
        out_host.copy_(o, non_blocking=True)
        return o, r

    e2e_ms, _ = timed(e2e_step)
    if rank != 0:
        return None
    return {"metric": "filtered megapixels/sec (d-channel, m landmarks)", "value": round(H * W / (ms * 1e-3) / 1e6, 2),
            "unit": "Mpix/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (seeded random-polygon scene, SURVEY §8d)",
            "config": {"workload": wl.name, "H": H, "W": W, "m0": wl.m0, "parallelism": f"row-band x{world}",
                       "halo_rows": params.spatial.effective_radius() + (1 if nlm else 0),
                       "l2": "not flushed: every rank streams planes far larger than L2"},
            "e2e": {"value": round(H * W / (e2e_ms * 1e-3) / 1e6, 2), "unit": "Mpix/s", "ms_per_step": round(e2e_ms, 3),
                    "h2d_bytes_per_step": int(f_host.numel() * 4), "d2h_bytes_per_step": int(out_host.numel() * 4),
                    "path": "per rank: pinned rows -> device, sharded_fast_filter, output rows -> pinned host (rank 0's bytes)"},
            "gpu_launches": launches, "clocks": clk.summary(),
            "time": time.time(), "report": {"quant_error": rep["quant_error"], "guarded": rep["guarded_pixels"]}}
