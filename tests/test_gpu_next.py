"""GPU parity for the §8 "next" rows beyond the recursive Gaussian (which
lives in test_gpu_parity.py): f1 brute_force_filter, f4 quality metrics.

Reference fixtures: tests/golden/brute.npz, metrics.npz (written by the
reference itself, tools/make_golden.py)."""

import numpy as np
import pytest
import torch

from conftest import group, load_golden
from oracle import nys_oracle as O
from paper_1901_06112_b200 import (
    FilterParams,
    Image,
    PatchGuide,
    SpatialKernel,
    brute_force_filter,
    mse,
    psnr,
    quality,
    ssim,
)
from paper_1901_06112_b200.synthetic import color_scene

pytestmark = pytest.mark.gpu

TOL = 1e-4
KINDS = {0: "box", 1: "gaussian_fir", 2: "gaussian_recursive"}


def _kernel(kind, sigma, radius):
    if kind == 0:
        return SpatialKernel.box(int(radius))
    if kind == 2:
        return SpatialKernel.recursive(float(sigma))
    return SpatialKernel.gaussian(float(sigma), int(radius))


@pytest.mark.parametrize("name", ["fir", "box", "rec", "hyper", "joint", "nlm"])
def test_brute_force_matches_reference(name):
    c = group(load_golden("brute"), "")[name]
    kind, sigma, radius, theta = c["meta"]
    params = FilterParams(spatial=_kernel(int(kind), sigma, radius), theta=float(theta), m0=4)
    f = Image(data=c["f"].astype(np.float64), range_max=1.0)
    same = np.array_equal(c["guide"], c["f"])
    p = f if same else Image(data=c["guide"].astype(np.float64), range_max=1.0)
    out = brute_force_filter(f, p, params)
    assert isinstance(out.data, np.ndarray) and out.data.dtype == np.float64
    err = np.abs(out.data - c["output"]).max()
    assert err <= 2e-6, err


def test_brute_force_patch_guide_and_device_io():
    c = group(load_golden("brute"), "")["nlm"]
    kind, sigma, radius, theta = c["meta"]
    params = FilterParams(spatial=SpatialKernel.box(int(radius)), theta=float(theta), m0=4)
    f = Image(data=torch.from_numpy(c["f"]).cuda(), range_max=1.0)
    out = brute_force_filter(f, PatchGuide(f, 1), params)
    assert out.data.is_cuda
    assert np.abs(out.data.double().cpu().numpy() - c["output"]).max() <= 2e-6


def test_brute_force_large_radius_and_edges():
    # general (non-SMEM, many-channel) instantiation + 1-row / 1-column images
    for (H, W), sk in (((1, 40), SpatialKernel.gaussian(3.0, 9)), ((37, 1), SpatialKernel.box(6)),
                       ((24, 30), SpatialKernel.gaussian(12.0, 40))):
        f32 = color_scene(H, W, 3, 0.05, seed=H * 7 + W)
        f64 = f32.astype(np.float64)
        kind = {"box": "box", "gaussian_fir": "gaussian_fir"}[sk.kind]
        ref = O.brute_force_filter(f64, f64, 0.15, kind, sk.sigma, sk.radius)
        out = brute_force_filter(Image(data=f64, range_max=1.0), Image(data=f64, range_max=1.0),
                                 FilterParams(spatial=sk, theta=0.15, m0=1))
        assert np.abs(out.data - ref).max() <= 2e-6, (H, W)


def test_fast_filter_approaches_brute_force_at_full_rank():
    # SPEC acceptance #1 on the GPU: m0 = m, eps_drop = 0 -> fast == brute
    g = load_golden("full_rank")
    f = Image(data=g["f"].astype(np.float64), range_max=1.0)
    from paper_1901_06112_b200 import filter_with_landmarks

    params = FilterParams(spatial=SpatialKernel.gaussian(1.0, 3), theta=0.3, m0=144, eps_drop=0.0,
                          kmeans_max_iter=5)
    brute = brute_force_filter(f, f, params)
    assert np.abs(brute.data - g["brute"]).max() <= 2e-6


@pytest.mark.parametrize("name", ["rgb", "u8", "small", "hyper"])
def test_metrics_match_reference(name):
    c = group({k: v for k, v in load_golden("metrics").items() if not k.startswith("same")}, "")[name]
    R = float(c["R"])
    a, b = Image(data=c["a"], range_max=R), Image(data=c["b"], range_max=R)
    assert mse(a, b) == pytest.approx(float(c["mse"]), rel=1e-12)
    assert psnr(a, b) == pytest.approx(float(c["psnr"]), abs=1e-9)
    assert psnr(a, b, per_band=True) == pytest.approx(float(c["psnr_band"]), abs=1e-9)
    assert ssim(a, b) == pytest.approx(float(c["ssim"]), abs=1e-10)
    q = quality(a, b, per_band=True)
    assert q.mse == pytest.approx(float(c["mse"]), rel=1e-12) and q.ssim == pytest.approx(float(c["ssim"]), abs=1e-10)
    # float32 device tensors: same metric from rounded samples
    ta = Image(data=torch.from_numpy(c["a"]).float().cuda(), range_max=R)
    tb = Image(data=torch.from_numpy(c["b"]).float().cuda(), range_max=R)
    assert ssim(ta, tb) == pytest.approx(O.ssim(c["a"].astype(np.float32), c["b"].astype(np.float32), R), abs=1e-10)


def test_metrics_identical_and_shape_errors():
    a = Image(data=np.random.default_rng(0).uniform(0, 1, (3, 16, 16)), range_max=1.0)
    assert psnr(a, a) == 99.0 and mse(a, a) == 0.0 and ssim(a, a) == pytest.approx(1.0, abs=1e-12)
    with pytest.raises(ValueError):
        mse(a, Image(data=np.zeros((3, 16, 15)), range_max=1.0))


# --------------------------------------------------------------------------
# §8 row f3: PCA patch guides (csrc/nys_pca.cu) and NLM filters on them
# --------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["r1k10", "r2k25", "r3k25", "gray_r3k6"])
def test_pca_guide_matches_reference(name):
    from paper_1901_06112_b200 import pca_patch_guide

    c = group(load_golden("pca_guide"), "")[name]
    r, k = (int(v) for v in c["meta"])
    g = pca_patch_guide(Image(data=c["f"].astype(np.float64), range_max=1.0), r, k)
    assert g.data.shape == c["guide"].shape
    assert np.abs(g.data - c["guide"]).max() <= 2e-5 * max(1.0, np.abs(c["guide"]).max())


@pytest.mark.parametrize("case", ["nlm_pca_r2k12", "nlm_pca_r3k25"])
def test_nlm_pca_filter_two_stage(case):
    from paper_1901_06112_b200 import build_guide, fast_filter, filter_with_landmarks

    g = load_golden(case)
    f = Image(data=torch.from_numpy(g["f"]).cuda(), range_max=1.0)
    params = FilterParams(spatial=SpatialKernel.box(int(g["radius"])), theta=float(g["theta"]), m0=int(g["m0"]),
                          mode="nlm", patch_radius=int(g["patch_radius"]), pca_dim=int(g["pca_dim"]),
                          kmeans_max_iter=15)
    p = build_guide(f, "nlm", None, int(g["patch_radius"]), int(g["pca_dim"]))
    assert p.data.is_cuda and p.data.shape[0] == int(g["pca_dim"])
    # stage 1: the reference's landmarks on our guide
    rep = filter_with_landmarks(f, p, g["centroids"], params)
    out = rep.output.data.double().cpu().numpy()
    assert np.abs(out - g["output"]).max() <= TOL
    assert rep.guarded_pixels == int(g["guarded_pixels"])
    # stage 2: our k-means on our guide
    full = fast_filter(f, p, params)
    assert abs(full.quant_error - float(g["quant_error"])) <= 1e-3 * float(g["quant_error"])


def test_pca_guide_large_patch_dimension():
    # 31 bands x 3x3 patches = 279 dims (> the 256 of the first version): moments, the chunked Gram
    # and the narrower projection blocks against a NumPy restatement (filters.py:161-187)
    from paper_1901_06112_b200 import pca_patch_guide
    from paper_1901_06112_b200.synthetic import spectral_scene

    f32 = spectral_scene(24, 28, 31, 4, 0.03, seed=5)
    f64 = f32.astype(np.float64)
    P = O.patch_stack(f64, 1)
    X = P.reshape(P.shape[0], -1).T
    Xc = X - X.mean(axis=0)
    vals, vecs = np.linalg.eigh(Xc.T @ Xc / X.shape[0])
    o = np.argsort(-vals, kind="stable")
    vecs = vecs[:, o]
    idx = np.argmax(np.abs(vecs), axis=0)
    vecs = vecs * np.where(vecs[idx, np.arange(vecs.shape[1])] < 0, -1.0, 1.0)[None, :]
    ref = (Xc @ vecs[:, :8]).T.reshape(8, 24, 28)
    g = pca_patch_guide(Image(data=f64, range_max=1.0), 1, 8)
    assert np.abs(g.data - ref).max() <= 2e-5 * max(1.0, np.abs(ref).max())


def test_standalone_spatial_filters_match_reference():
    # spatial.py public helpers on the device (FP64) vs the reference's own outputs
    from paper_1901_06112_b200 import apply_planes, box_filter, gaussian_fir, gaussian_recursive

    g = load_golden("spatial")
    np.testing.assert_allclose(gaussian_fir(g["plane"], 1.3, 3), g["fir_1.3_3"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(box_filter(g["plane"], 2), g["box_2"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(box_filter(g["plane"], 0), g["box_0"], rtol=0, atol=0)
    r = load_golden("recursive")
    for s in (0.7, 1.0, 2.5, 4.0):
        np.testing.assert_allclose(gaussian_recursive(r["plane"], s), r[f"rec_{s}"], rtol=1e-12, atol=1e-12)
    # pkg/tests/test_spatial.py-style known answers: box of a constant, box of an impulse
    for S in (0, 1, 3):
        assert np.array_equal(box_filter(np.full((6, 5), 2.5), S), np.full((6, 5), 2.5 * (2 * S + 1) ** 2))
    imp = np.zeros((7, 7))
    imp[3, 3] = 1
    exp = np.zeros((7, 7))
    exp[2:5, 2:5] = 1
    assert np.array_equal(box_filter(imp, 1), exp)
    stack = np.random.default_rng(0).random((3, 9, 11))
    t = apply_planes(torch.from_numpy(stack).cuda(), SpatialKernel.recursive(2.0))
    assert t.is_cuda
    np.testing.assert_allclose(t.cpu().numpy(), O.spatial_conv(stack, "gaussian_recursive", 2.0, 0), rtol=1e-12,
                               atol=1e-12)
