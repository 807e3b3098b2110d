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

    def exchange_rows(self, local: torch.Tensor, lo: int, hi: int, H: int, halo: int):
        """Extend ``local`` (c, hi-lo, W) with up to ``halo`` rows from each
        neighbour; returns (extended tensor, first global row)."""
        r, w = self.rank, self.world
        elo, ehi = halo_rows(lo, hi, H, halo)
        need_top, need_bot = lo - elo, ehi - hi
        if need_top > (hi - lo) or need_bot > (hi - lo):
            raise ValueError("each shard must own at least `halo` rows")
        dev = local.device
        xfer = (lambda t: t.contiguous()) if self.backend == "nccl" else (lambda t: t.cpu().contiguous())
        ops, bufs = [], {}
        c, _, W = local.shape
        # counts are symmetric once every shard owns >= halo rows: rank r needs
        # min(lo, halo) rows from r-1 and sends it the same number of its top rows
        if r > 0:
            k = need_top
            bufs["top"] = xfer(torch.empty((c, k, W), dtype=local.dtype, device=dev))
            ops.append(dist.P2POp(dist.isend, xfer(local[:, :k]), r - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, bufs["top"], r - 1, self.group))
        if r < w - 1:
            k = need_bot
            bufs["bot"] = xfer(torch.empty((c, k, W), dtype=local.dtype, device=dev))
            ops.append(dist.P2POp(dist.isend, xfer(local[:, local.shape[1] - k:]), r + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, bufs["bot"], r + 1, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        parts = []
        if "top" in bufs:
            parts.append(bufs["top"].to(dev))
        parts.append(local)
        if "bot" in bufs:
            parts.append(bufs["bot"].to(dev))
        return torch.cat(parts, dim=1).contiguous(), elo


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


# ---------------------------------------------------------------------------
# sharded filter
# ---------------------------------------------------------------------------
def sharded_fast_filter(f_local: torch.Tensor, H: int, params, comm: Comm, nlm: bool = False):
    """Filter this rank's rows of a row-sharded image.

    ``f_local`` (n, rows, W) holds image rows shard_rows(H, world, rank).
    Returns (out_local (n, rows, W), report dict)."""
    from .filters import _Inputs, run_filter
    from ._device import ptr, stream_ptr

    lo, hi = shard_rows(H, comm.world, comm.rank)
    if f_local.shape[1] != hi - lo:
        raise ValueError("f_local rows do not match this rank's shard")
    n, _, W = f_local.shape
    R = params.spatial.effective_radius()
    halo = R + (1 if nlm else 0)
    ext, elo = comm.exchange_rows(f_local, lo, hi, H, halo)
    ext = ext.to(f_local.device).contiguous()
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
        points = f_local.reshape(n, -1)
        inp = _Inputs(f=ext, guide=ext, gkind=0, points=points, rho=n)
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
    f_local = f_host.to(dev)
    del f_full
    sk = SpatialKernel.box(wl.radius) if wl.spatial == "box" else SpatialKernel.gaussian(wl.sigma, wl.radius)
    params = FilterParams(spatial=sk, theta=float(wl.theta), m0=wl.m0, seed=0, kmeans_max_iter=wl.max_iter)
    nlm = wl.mode == "nlm"
    for _ in range(args.warmup):
        sharded_fast_filter(f_local, H, params, comm, nlm)
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
        ms, (out, rep) = timed(lambda: sharded_fast_filter(f_local, H, params, comm, nlm))
    launches = (int(lib.nys_kernel_launches()) - l0) // max(1, args.steps)
    out_host = torch.empty(out.shape, dtype=torch.float32, pin_memory=True)

    def e2e_step():
        fd = f_host.to(dev, non_blocking=True)
        o, r = sharded_fast_filter(fd, H, params, comm, nlm)
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
