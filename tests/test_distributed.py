"""Multi-rank host logic of the row-band-sharded path (parallel.py) on CPU:
world_size 2 over gloo, with NumPy stand-ins for the per-rank device
reductions.  The sharded k-means must reproduce the single-process reference
k-means (oracle) on the concatenated points, and the halo exchange must
reconstruct each rank's extended band exactly."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import nys_oracle as O
from paper_1901_06112_b200.bands import halo_rows, shard_rows
from paper_1901_06112_b200.parallel import Comm, KMeansOps, distributed_kmeans


class NumpyOps(KMeansOps):
    """Reference-order FP64 reductions over this rank's points (m, rho)."""

    def __init__(self, X):
        self.X = np.ascontiguousarray(X, dtype=np.float64)
        self.m, self.rho = self.X.shape
        self.d2 = None
        self.nearest = None
        self.labels = None

    def pp_update(self, c, init):
        v = ((self.X - c) ** 2).sum(axis=1)
        self.d2 = v if init else np.minimum(self.d2, v)
        return float(self.d2.sum())

    def pp_pick(self, target):
        cs = np.cumsum(self.d2)
        idx = int(np.searchsorted(cs, target, side="right"))
        if idx >= self.m:
            idx = int(np.flatnonzero(self.d2 > 0)[-1])
        return idx

    def point(self, idx):
        return self.X[int(idx)].copy()

    def assign(self, C, first):
        lab, nearest = O.assign(self.X, C)
        changed = self.m if (first or self.labels is None) else int((lab != self.labels).sum())
        self.labels, self.nearest = lab, nearest
        m0 = C.shape[0]
        acc = np.zeros(m0 * (self.rho + 1) + 2)
        sums = acc[: m0 * (self.rho + 1)].reshape(m0, self.rho + 1)
        for d in range(self.rho):
            sums[:, d] = np.bincount(lab, weights=self.X[:, d], minlength=m0)
        sums[:, self.rho] = np.bincount(lab, minlength=m0)
        acc[-2] = nearest.sum()
        acc[-1] = changed
        return acc

    def farthest(self, C, excl):
        taken = self.nearest.copy()
        taken[list(excl)] = -1.0
        k = int(np.argmax(taken))
        return float(taken[k]), k

    def exact(self, C):
        _, nearest = O.assign(self.X, C, exact=True)
        return float(nearest.sum())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, args, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(Comm(), *args)))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _run(world, fn, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, args, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    return [out[r] for r in range(world)]


def _kmeans_rank(comm, X, m0, seed, it):
    lo, hi = shard_rows(X.shape[0], comm.world, comm.rank)
    res = distributed_kmeans(NumpyOps(X[lo:hi]), comm, m0, seed, it)
    return res.centroids, res.quant_error, res.errors


def _halo_rank(comm, img, halo):
    H = img.shape[1]
    lo, hi = shard_rows(H, comm.world, comm.rank)
    ext, elo = comm.exchange_rows(torch.from_numpy(img[:, lo:hi].copy()), lo, hi, H, halo)
    return ext.numpy(), elo


def _scene(H, W, seed):
    rng = np.random.default_rng(seed)
    lab = (np.arange(H)[:, None] // 7 + np.arange(W)[None, :] // 9) % 5
    cols = rng.uniform(0, 1, (5, 3))
    return (np.moveaxis(cols[lab], 2, 0) + 0.03 * rng.standard_normal((3, H, W))).astype(np.float32)


@pytest.mark.parametrize("world", [2])
def test_sharded_kmeans_matches_single_process(world):
    img = _scene(24, 20, 3).astype(np.float64)
    X = O.range_vectors(img)
    C_ref, _, qe_ref, err_ref = O.kmeans(X, 6, seed=5, max_iter=10)
    outs = _run(world, _kmeans_rank, X, 6, 5, 10)
    for r in outs:
        assert not isinstance(r, str), r
        C, qe, errs = r
        np.testing.assert_allclose(C, C_ref, rtol=0, atol=1e-12)
        assert qe == pytest.approx(qe_ref, rel=1e-12)
        np.testing.assert_allclose(errs, err_ref, rtol=1e-12)


def test_sharded_kmeans_empty_cluster_repair_and_zero_total():
    # many duplicates: empty clusters during Lloyd; all-equal points: sum(D^2) == 0
    X = np.array([[0.0], [0.0], [0.0], [100.0], [100.0], [0.1], [0.0], [100.0]])
    C_ref, _, qe_ref, _ = O.kmeans(X, 4, seed=0, max_iter=20)
    for r in _run(2, _kmeans_rank, X, 4, 0, 20):
        assert not isinstance(r, str), r
        np.testing.assert_allclose(r[0], C_ref, atol=1e-12)
        assert r[1] == pytest.approx(qe_ref, abs=1e-12)
    X = np.ones((10, 2))
    C_ref, _, qe_ref, _ = O.kmeans(X, 3, seed=2, max_iter=5)
    for r in _run(2, _kmeans_rank, X, 3, 2, 5):
        assert not isinstance(r, str), r
        np.testing.assert_array_equal(r[0], C_ref)


def test_halo_exchange_reconstructs_bands():
    img = np.random.default_rng(1).random((2, 30, 7)).astype(np.float32)
    halo = 4
    outs = _run(3, _halo_rank, img, halo)
    for rank, r in enumerate(outs):
        assert not isinstance(r, str), r
        ext, elo = r
        lo, hi = shard_rows(30, 3, rank)
        e0, e1 = halo_rows(lo, hi, 30, halo)
        assert elo == e0
        np.testing.assert_array_equal(ext, img[:, e0:e1])
