"""Row-band sharded path on the GPU: two ranks (gloo for the host-side
collectives, both computing on cuda:0 -- their kernels never wait on each
other) must reproduce the single-device fast_filter on the whole image."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, img, spatial, theta, m0, iters, nlm, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1901_06112_b200 import FilterParams, SpatialKernel
        from paper_1901_06112_b200.bands import shard_rows
        from paper_1901_06112_b200.parallel import Comm, sharded_fast_filter

        sk = SpatialKernel.box(spatial[1]) if spatial[0] == "box" else SpatialKernel.gaussian(spatial[1], spatial[2])
        params = FilterParams(spatial=sk, theta=theta, m0=m0, kmeans_max_iter=iters)
        H = img.shape[1]
        lo, hi = shard_rows(H, world, rank)
        f_local = torch.from_numpy(np.ascontiguousarray(img[:, lo:hi])).cuda()
        out, rep = sharded_fast_filter(f_local, H, params, Comm(), nlm=nlm)
        q.put((rank, (lo, out.double().cpu().numpy(), rep["quant_error"], rep["guarded_pixels"], rep["centroids"])))
    except Exception as e:  # surfaced by the parent
        import traceback

        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["blf", "nlm"])
def test_two_rank_sharded_filter_matches_single_device(case):
    from paper_1901_06112_b200 import FilterParams, Image, PatchGuide, SpatialKernel, fast_filter
    from paper_1901_06112_b200.synthetic import color_scene

    if case == "blf":
        img = color_scene(70, 64, 8, 0.05, seed=21)
        spatial, theta, m0, iters, nlm = ("gaussian", 3.0, 9), 0.15, 12, 8, False
        sk = SpatialKernel.gaussian(3.0, 9)
    else:
        img = color_scene(64, 48, 6, 0.08, seed=22, lo=0.1, hi=0.9, shading=0.1)
        spatial, theta, m0, iters, nlm = ("box", 10), 0.3 * np.sqrt(27.0) * 0.08, 10, 8, True
        sk = SpatialKernel.box(10)
    f = Image(data=torch.from_numpy(img).cuda(), range_max=1.0)
    ref = fast_filter(f, PatchGuide(f, 1) if nlm else f, FilterParams(spatial=sk, theta=theta, m0=m0,
                                                                       kmeans_max_iter=iters))
    ref_out = ref.output.data.double().cpu().numpy()

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, img, spatial, theta, m0, iters, nlm, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    guarded = 0
    for r in range(2):
        assert not isinstance(res[r], str), res[r]
        lo, out, qe, g, C = res[r]
        np.testing.assert_allclose(C, ref.centroids, rtol=0, atol=1e-9)
        assert qe == pytest.approx(ref.quant_error, rel=1e-9)
        assert np.abs(out - ref_out[:, lo:lo + out.shape[1]]).max() <= 1e-6
        guarded = g
    assert guarded == ref.guarded_pixels


def _nccl_one_rank(port, img, m0, iters, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        from paper_1901_06112_b200 import FilterParams, SpatialKernel
        from paper_1901_06112_b200.parallel import Comm, device_distributed_kmeans, sharded_fast_filter

        f_local = torch.from_numpy(img).cuda()
        n = img.shape[0]
        km = device_distributed_kmeans(f_local.reshape(n, -1), Comm(), m0, 0, iters)
        params = FilterParams(spatial=SpatialKernel.gaussian(3.0, 9), theta=0.15, m0=m0, kmeans_max_iter=iters)
        out, rep = sharded_fast_filter(f_local, img.shape[1], params, Comm())
        q.put(("ok", km.centroids, km.quant_error, km.errors, out.double().cpu().numpy(), rep["quant_error"]))
    except Exception:  # surfaced by the parent
        import traceback

        q.put(("err", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_device_resident_sharded_kmeans_one_rank_nccl():
    """The NCCL path's device-resident k-means (collectives on device buffers, one host
    wait) reproduces the single-device k-means; the sharded filter reproduces fast_filter."""
    from paper_1901_06112_b200 import FilterParams, Image, SpatialKernel, fast_filter, kmeans_landmarks
    from paper_1901_06112_b200.synthetic import color_scene

    img = color_scene(96, 80, 10, 0.05, seed=31)
    m0, iters = 16, 10
    ref = kmeans_landmarks(img.reshape(3, -1).T.astype(np.float64), m0, seed=0, max_iter=iters)
    f = Image(data=torch.from_numpy(img).cuda(), range_max=1.0)
    ref_f = fast_filter(f, f, FilterParams(spatial=SpatialKernel.gaussian(3.0, 9), theta=0.15, m0=m0,
                                           kmeans_max_iter=iters))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_one_rank, args=(_free_port(), img, m0, iters, q))
    p.start()
    res = q.get(timeout=600)
    p.join(timeout=60)
    assert res[0] == "ok", res[1]
    _, C, qe, errs, out, qe2 = res
    np.testing.assert_allclose(C, ref.centroids, rtol=0, atol=1e-9)
    assert qe == pytest.approx(ref.quant_error, rel=1e-9)
    assert len(errs) == len(ref.errors)
    np.testing.assert_allclose(errs, ref.errors, rtol=1e-9)
    assert np.abs(out - ref_f.output.data.double().cpu().numpy()).max() <= 1e-6
