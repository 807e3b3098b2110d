"""GPU parity: the CUDA path (through the C ABI) vs the reference's golden
outputs and the pinned CPU oracle.

Tolerances (BASELINE.json north_star): filter output max-abs <= 1e-4 on
[0, 1] data given the reference's landmarks; k-means objective within 1e-3
relative; guarded-pixel counts and retained ranks exact.
"""

import numpy as np
import pytest
import torch

from conftest import FILTER_CASES, group, load_golden, spatial_kernel
from oracle import nys_oracle as O
from paper_1901_06112_b200 import (
    FilterParams,
    Image,
    PatchGuide,
    SpatialKernel,
    fast_filter,
    filter_with_landmarks,
    kmeans_landmarks,
)
from paper_1901_06112_b200.filters import _prepare_inputs, run_filter
from paper_1901_06112_b200.synthetic import CONFIGS, color_scene, spectral_scene

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _params(g, m0=None):
    return FilterParams(spatial=spatial_kernel(g), theta=float(g["theta"]), m0=int(g["m0"] if m0 is None else m0), seed=0,
                        kmeans_max_iter=int(g["max_iter"]), eps_drop=float(g["eps_drop"]))


def _images(g):
    f = Image(data=g["f"].astype(np.float64), range_max=1.0)
    p = f if bool(g["guide_is_f"]) else Image(data=g["guide"].astype(np.float64), range_max=1.0)
    return f, p


@pytest.mark.parametrize("case", FILTER_CASES)
def test_filter_with_reference_landmarks(case):
    g = load_golden(case)
    f, p = _images(g)
    rep = filter_with_landmarks(f, p, g["centroids"], _params(g))
    err = np.abs(rep.output.data - g["output"]).max()
    assert err <= TOL, err
    assert rep.retained_rank == int(g["retained_rank"])
    assert rep.guarded_pixels == int(g["guarded_pixels"])


@pytest.mark.parametrize("case", FILTER_CASES)
def test_fast_filter_end_to_end(case):
    g = load_golden(case)
    f, p = _images(g)
    rep = fast_filter(f, p, _params(g))
    assert abs(rep.quant_error - float(g["quant_error"])) <= 1e-3 * float(g["quant_error"])
    np.testing.assert_allclose(rep.centroids, g["centroids"], rtol=0, atol=1e-5)
    err = np.abs(rep.output.data - g["output"]).max()
    assert err <= TOL, err
    assert rep.guarded_pixels == int(g["guarded_pixels"])
    assert set(rep.timings) >= {"clustering", "eigendecomposition", "extrapolation", "convolutions",
                                "normalization", "total"}


def test_nlm_patch_guide_on_the_fly_equals_materialised():
    g = load_golden("nlm_patch_box10")
    f = Image(data=g["f"].astype(np.float64), range_max=1.0)
    pg = PatchGuide(f, 1)
    params = _params(g)
    a = filter_with_landmarks(f, pg, g["centroids"], params)   # guide_kind 1: gathered in-kernel
    b = filter_with_landmarks(f, Image(data=g["guide"].astype(np.float64), range_max=1.0), g["centroids"], params)
    assert np.abs(a.output.data - b.output.data).max() <= 1e-6
    assert np.abs(a.output.data - g["output"]).max() <= TOL
    assert a.guarded_pixels == b.guarded_pixels == int(g["guarded_pixels"])


def test_kmeans_known_answers():
    for name, c in group(load_golden("kmeans_kat"), "").items():
        m0, seed, it = (int(v) for v in c["meta"])
        lm = kmeans_landmarks(c["points"], m0, seed=seed, max_iter=it)
        # device points are float32: FP64 KAT inputs such as 0.1 round to 0.1f (1.5e-9 away)
        np.testing.assert_allclose(lm.centroids, c["centroids"], rtol=1e-7, atol=1e-9, err_msg=name)
        np.testing.assert_array_equal(lm.assignment, c["assignment"], err_msg=name)
        assert lm.quant_error == pytest.approx(float(c["quant_error"]), rel=1e-6, abs=1e-12), name
        assert len(lm.errors) == len(c["errors"]), name
    lm = kmeans_landmarks(np.array([[0.0], [10.0]]), 2, seed=0)
    assert sorted(lm.centroids.ravel().tolist()) == [0.0, 10.0] and lm.quant_error == 0.0


def test_kmeans_errors_and_validation():
    with pytest.raises(ValueError):
        kmeans_landmarks(np.zeros((4, 2)), 5)
    with pytest.raises(ValueError):
        kmeans_landmarks(np.zeros((4, 2)), 0)
    # all points identical: sum(D^2) == 0 at the first draw -> integers() path
    lm = kmeans_landmarks(np.ones((50, 3)), 4, seed=1, max_iter=5)
    O_C, O_lab, O_qe, _ = O.kmeans(np.ones((50, 3)), 4, 1, 5)
    np.testing.assert_array_equal(lm.centroids, O_C)
    assert lm.quant_error == O_qe == 0.0


def test_kmeans_monotone_and_reproducible():
    rng = np.random.default_rng(7)
    centers = rng.uniform(0, 50, (5, 3))
    pts = np.concatenate([c + 2.0 * rng.standard_normal((60, 3)) for c in centers]).astype(np.float32)
    a = kmeans_landmarks(pts.astype(np.float64), 5, seed=2)
    b = kmeans_landmarks(pts.astype(np.float64), 5, seed=2)
    assert np.array_equal(a.centroids, b.centroids) and a.quant_error == b.quant_error
    e = np.array(a.errors)
    assert np.all(np.diff(e) <= 1e-6 * e[0])
    C, lab, qe, _ = O.kmeans(pts.astype(np.float64), 5, 2, 50)
    assert a.quant_error == pytest.approx(qe, rel=1e-6)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_config_crops_vs_oracle(cfg):
    """Each BASELINE config's kernel on a seeded crop: stage 1 (filter given
    the oracle's landmarks) and stage 2 (GPU k-means objective)."""
    wl = CONFIGS[cfg]
    H, W = {1: (96, 112), 2: (72, 128), 3: (64, 72), 4: (40, 48), 5: (48, 56)}[cfg]
    f32 = wl.image(seed=cfg, H=H, W=W)
    f64 = f32.astype(np.float64)
    p64 = O.patch_stack(f64, 1) if wl.mode == "nlm" else f64
    m0 = min(wl.m0, 24)
    C, _lab, qe, _ = O.kmeans(O.range_vectors(p64), m0, 0, wl.max_iter)
    ref = O.fast_filter_with_landmarks(f64, p64, C, wl.theta, wl.spatial, wl.sigma, wl.radius)
    sk = SpatialKernel.box(wl.radius) if wl.spatial == "box" else SpatialKernel.gaussian(wl.sigma, wl.radius)
    params = FilterParams(spatial=sk, theta=wl.theta, m0=m0, kmeans_max_iter=wl.max_iter)
    f = Image(data=f64, range_max=1.0)
    p = PatchGuide(f, 1) if wl.mode == "nlm" else f
    rep = filter_with_landmarks(f, p, C, params)
    assert np.abs(rep.output.data - ref["output"]).max() <= TOL
    assert rep.guarded_pixels == ref["guarded_pixels"]
    full = fast_filter(f, p, params)
    assert abs(full.quant_error - qe) <= 1e-3 * qe
    assert np.abs(full.output.data - ref["output"]).max() <= TOL


def test_banded_equals_single_band_bitwise():
    f32 = spectral_scene(96, 80, 8, 6, 0.03, seed=3)
    f = Image(data=torch.from_numpy(f32).cuda(), range_max=1.0)
    params = FilterParams(spatial=SpatialKernel.gaussian(3.0, 9), theta=0.25, m0=12)
    inp = _prepare_inputs(f, f)
    C = kmeans_landmarks(f32.reshape(8, -1).T.astype(np.float64), 12, max_iter=10).centroids
    one, _, s1 = run_filter(inp, C, params)
    row_bytes = (12 + 1) * (8 + 1) * 96 * 4  # row stride: W padded to 32 x planes
    many, _, s2 = run_filter(inp, C, params, plane_budget=row_bytes * 30)  # 30-row bands incl. halo
    torch.cuda.synchronize()
    assert torch.equal(one, many)
    assert torch.equal(s1, s2)


def test_device_tensor_roundtrip_and_edge_sizes():
    # 1-row, 1-column and tiny images; device-resident input returns a device tensor
    for H, W in ((1, 37), (29, 1), (3, 3), (17, 300)):
        f32 = color_scene(H, W, 3, 0.05, seed=H * 31 + W)
        f = Image(data=torch.from_numpy(f32).cuda(), range_max=1.0)
        m0 = min(4, H * W)
        params = FilterParams(spatial=SpatialKernel.gaussian(1.5, 4), theta=0.2, m0=m0, kmeans_max_iter=5)
        rep = fast_filter(f, f, params)
        assert isinstance(rep.output.data, torch.Tensor) and rep.output.data.is_cuda
        C, _, qe, _ = O.kmeans(O.range_vectors(f32.astype(np.float64)), m0, 0, 5)
        ref = O.fast_filter_with_landmarks(f32.astype(np.float64), f32.astype(np.float64), C, 0.2,
                                           "gaussian_fir", 1.5, 4)
        out = rep.output.data.double().cpu().numpy()
        assert np.abs(out - ref["output"]).max() <= TOL, (H, W)


def test_constant_image_is_fixed_point():
    f = Image(data=np.full((3, 20, 24), 0.375), range_max=1.0)
    rep = fast_filter(f, f, FilterParams(spatial=SpatialKernel.box(2), theta=0.1, m0=1, kmeans_max_iter=3))
    assert np.abs(rep.output.data - 0.375).max() <= 1e-6
    assert rep.retained_rank == 1


@pytest.mark.parametrize("n", [1, 2, 5, 7])
def test_channel_counts_with_partial_plane_chunks(n):
    # (n+1) planes per landmark group not a multiple of 4: K3's tail TMA box
    f32 = spectral_scene(40, 72, n, 5, 0.03, seed=40 + n) if n >= 4 else \
        np.ascontiguousarray(color_scene(40, 72, 5, 0.03, seed=40 + n)[:n])
    f = Image(data=torch.from_numpy(f32).cuda(), range_max=1.0)
    C, _, _, _ = O.kmeans(O.range_vectors(f32.astype(np.float64)), 6, 0, 6)
    params = FilterParams(spatial=SpatialKernel.gaussian(2.0, 6), theta=0.3, m0=6)
    rep = filter_with_landmarks(f, f, C, params)
    ref = O.fast_filter_with_landmarks(f32.astype(np.float64), f32.astype(np.float64), C, 0.3, "gaussian_fir", 2.0, 6)
    out = rep.output.data.double().cpu().numpy()
    assert np.abs(out - ref["output"]).max() <= TOL
    assert rep.guarded_pixels == ref["guarded_pixels"]


@pytest.mark.parametrize("rho,m0,radius", [(2, 7, 9), (3, 13, 9), (4, 11, 5), (3, 33, 15), (16, 21, 12), (9, 10, 9)])
def test_guide_dimensions_and_odd_landmark_counts(rho, m0, radius):
    """K2's feature loops against the oracle where their padding shows: colour-guide loop (two
    landmarks per packed operation, pair-interleaved centroids) with odd landmark counts and
    rho = 2 .. 4 (zero-padded dimensions); wide-guide loop (two dimensions per packed operation)
    with rho not a multiple of four; compiled radii and the generic one."""
    f32 = spectral_scene(56, 88, rho, 6, 0.03, seed=rho * 10 + m0) if rho > 3 else \
        np.ascontiguousarray(color_scene(56, 88, 6, 0.04, seed=rho * 10 + m0)[:rho])
    f64 = f32.astype(np.float64)
    f = Image(data=torch.from_numpy(f32).cuda(), range_max=1.0)
    C, _, _, _ = O.kmeans(O.range_vectors(f64), m0, 0, 6)
    theta = 0.2 if rho <= 4 else 0.3
    params = FilterParams(spatial=SpatialKernel.gaussian(radius / 3.0, radius), theta=theta, m0=m0)
    rep = filter_with_landmarks(f, f, C, params)
    ref = O.fast_filter_with_landmarks(f64, f64, C, theta, "gaussian_fir", radius / 3.0, radius)
    out = rep.output.data.double().cpu().numpy()
    assert np.abs(out - ref["output"]).max() <= TOL
    assert rep.guarded_pixels == ref["guarded_pixels"]
    assert rep.retained_rank == ref["retained_rank"]


@pytest.mark.parametrize("rho", [1, 2, 3, 16, 27])
def test_lloyd_bounds_are_exact(rho, monkeypatch):
    # Hamerly-style skipping (and, for rho <= 3, the cell-pruned candidate search) must not
    # change a single label or centroid bit against searching every centroid for every point
    rng = np.random.default_rng(100 + rho)
    centers = rng.uniform(0, 1, (40, rho))
    pts = (centers[rng.integers(0, 40, 60000)] + 0.08 * rng.standard_normal((60000, rho))).astype(np.float32)
    a = kmeans_landmarks(pts.astype(np.float64), 32, seed=3, max_iter=40)
    monkeypatch.setenv("NYS_KM_NOBOUNDS", "1")
    b = kmeans_landmarks(pts.astype(np.float64), 32, seed=3, max_iter=40)
    assert np.array_equal(a.centroids, b.centroids)
    assert np.array_equal(a.assignment, b.assignment)
    assert len(a.errors) == len(b.errors)
    np.testing.assert_allclose(a.errors, b.errors, rtol=1e-12)
    assert a.quant_error == b.quant_error
    if rho <= 3:  # the Hamerly-bounds kernel the wider guides use, on the same points
        monkeypatch.delenv("NYS_KM_NOBOUNDS")
        monkeypatch.setenv("NYS_KM_NOGRID", "1")
        c = kmeans_landmarks(pts.astype(np.float64), 32, seed=3, max_iter=40)
        assert np.array_equal(c.centroids, b.centroids) and np.array_equal(c.assignment, b.assignment)


@pytest.mark.parametrize("rho,m0", [(16, 64), (31, 48), (32, 40), (40, 24), (17, 100)])
def test_tensor_core_lloyd_equals_fp32_search(rho, m0, monkeypatch):
    """Wide guides: the cooperative Lloyd kernel's tcgen05 3xTF32 search ((x, 1) . (-2c, |c|^2)
    in TMEM, exact FP32 re-check of the candidates within the error bound) against the FP32 search
    of every centroid: identical labels, centroids and objectives.  Shapes cover K and N padding
    (rho + 1 = 17 .. 41, m0 = 24 .. 100), near-duplicate points and far-off outliers."""
    rng = np.random.default_rng(rho * 100 + m0)
    centers = rng.uniform(0, 1, (m0 + 5, rho))
    pts = centers[rng.integers(0, m0 + 5, 40000)] + 0.05 * rng.standard_normal((40000, rho))
    pts[:200] = pts[200:400] + 1e-6 * rng.standard_normal((200, rho))  # near-ties between neighbours
    pts[400:420] *= 30.0  # outliers: large |x|^2 against small centroid gaps
    pts = pts.astype(np.float32)
    monkeypatch.setenv("NYS_KM_TC_COOP", "1")  # opt-in variant of k_lloyd_coop
    a = kmeans_landmarks(pts.astype(np.float64), m0, seed=2, max_iter=20)
    monkeypatch.setenv("NYS_KM_NOBOUNDS", "1")
    b = kmeans_landmarks(pts.astype(np.float64), m0, seed=2, max_iter=20)
    assert np.array_equal(a.centroids, b.centroids)
    assert np.array_equal(a.assignment, b.assignment)
    np.testing.assert_allclose(a.errors, b.errors, rtol=1e-12)


@pytest.mark.parametrize("rho,m,m0", [(3, 4_500_000, 24), (16, 300_000, 20), (27, 200_000, 12)])
def test_seeding_owner_publication_matches_all_blocks_resolution(rho, m, m0, monkeypatch):
    """k-means++: the owning block resolves a draw from its own run sums and stored D^2 and
    publishes the point (default) vs. every block resolving it from remote run sums and a
    recomputed run (NYS_SEED_MODE=0).  4.5 M points keep D^2 in global memory; the wide guides
    sweep their runs backwards on odd draws."""
    from paper_1901_06112_b200.landmarks import kmeans_device

    rng = np.random.default_rng(rho)
    pts = torch.from_numpy(rng.random((rho, m), dtype=np.float32)).cuda()
    a = kmeans_device(pts, m0, seed=3, max_iter=2)
    monkeypatch.setenv("NYS_SEED_MODE", "0")
    b = kmeans_device(pts, m0, seed=3, max_iter=2)
    assert np.array_equal(np.asarray(a.centroids), np.asarray(b.centroids))
    assert a.quant_error == b.quant_error


@pytest.mark.parametrize("case", ["quantised", "constant_dim", "negative_wide", "m64_duplicates"])
def test_cell_pruned_assignment_edge_cases(case, monkeypatch):
    """rho <= 3 Lloyd (candidate masks per cell of the points' bounding box) against the full
    search: exact ties from quantised colours, a dimension with zero range, negative / wide
    ranges, duplicated seeds with m0 = 64 (empty-cluster repairs)."""
    rng = np.random.default_rng(7)
    if case == "quantised":
        pts = (rng.integers(0, 8, (50000, 3)) / 7.0).astype(np.float32)
        m0 = 48
    elif case == "constant_dim":
        pts = rng.uniform(0, 1, (40000, 3)).astype(np.float32)
        pts[:, 1] = 0.25
        m0 = 24
    elif case == "negative_wide":
        pts = (rng.standard_normal((40000, 2)) * np.array([1000.0, 1e-3]) + np.array([-500.0, 2.0])).astype(np.float32)
        m0 = 40
    else:
        base = rng.uniform(0, 1, (20, 3))
        pts = np.repeat(base, 2000, axis=0).astype(np.float32)  # 20 distinct points, 64 landmarks
        m0 = 64
    a = kmeans_landmarks(pts.astype(np.float64), m0, seed=1, max_iter=25)
    monkeypatch.setenv("NYS_KM_NOBOUNDS", "1")
    b = kmeans_landmarks(pts.astype(np.float64), m0, seed=1, max_iter=25)
    assert np.array_equal(a.centroids, b.centroids)
    assert np.array_equal(a.assignment, b.assignment)
    np.testing.assert_allclose(a.errors, b.errors, rtol=1e-12)


def test_pinned_host_io_and_out_buffer():
    # pinned host in -> K3 writes the pinned host output in place; out= reuses a caller buffer
    f32 = color_scene(45, 70, 6, 0.05, seed=77)
    params = FilterParams(spatial=SpatialKernel.gaussian(2.0, 6), theta=0.15, m0=8, kmeans_max_iter=6)
    dev = fast_filter(Image(data=torch.from_numpy(f32).cuda(), range_max=1.0),
                      Image(data=torch.from_numpy(f32).cuda(), range_max=1.0), params)
    ref = dev.output.data.cpu()
    h = Image(data=torch.from_numpy(f32).pin_memory(), range_max=1.0)
    rep = fast_filter(h, h, params)
    assert not rep.output.data.is_cuda and rep.output.data.is_pinned()
    assert torch.equal(rep.output.data, ref)
    buf = torch.full(f32.shape, -1.0).pin_memory()
    rep2 = fast_filter(h, h, params, out=buf)
    assert rep2.output.data.data_ptr() == buf.data_ptr() and torch.equal(buf, ref)
    dbuf = torch.empty(f32.shape, device="cuda")
    rep3 = fast_filter(h, h, params, out=dbuf)
    assert rep3.output.data.is_cuda and torch.equal(dbuf.cpu(), ref)
    with pytest.raises(ValueError):
        fast_filter(h, h, params, out=torch.empty(3, 45, 71).pin_memory())


# --------------------------------------------------------------------------
# §8 row f2: recursive Gaussian (csrc/nys_recursive.cu)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("shape,sigma,m0", [((72, 128), 5.0, 24), ((1, 37), 2.0, 4), ((29, 1), 1.5, 4),
                                            ((3, 3), 1.0, 3), ((33, 300), 12.0, 16)])
def test_recursive_gaussian_vs_oracle(shape, sigma, m0):
    H, W = shape
    f32 = color_scene(H, W, 5, 0.05, seed=H + 7 * W)
    f64 = f32.astype(np.float64)
    C, _, qe, _ = O.kmeans(O.range_vectors(f64), m0, 0, 8)
    ref = O.fast_filter_with_landmarks(f64, f64, C, 0.12, "gaussian_recursive", sigma, 0)
    params = FilterParams(spatial=SpatialKernel.recursive(sigma), theta=0.12, m0=m0, kmeans_max_iter=8)
    f = Image(data=torch.from_numpy(f32).cuda(), range_max=1.0)
    rep = filter_with_landmarks(f, f, C, params)
    out = rep.output.data.double().cpu().numpy()
    assert np.abs(out - ref["output"]).max() <= TOL
    assert rep.guarded_pixels == ref["guarded_pixels"]
    assert rep.min_denominator == pytest.approx(ref["min_denominator"], rel=1e-4)
    full = fast_filter(f, f, params)
    assert abs(full.quant_error - qe) <= 1e-3 * qe
    assert np.abs(full.output.data.double().cpu().numpy() - ref["output"]).max() <= TOL


def test_recursive_landmark_bands_match_single_band():
    # a small plane budget forces several landmark bands (Z accumulates across bands)
    f32 = spectral_scene(40, 52, 7, 5, 0.03, seed=91)
    f = Image(data=torch.from_numpy(f32).cuda(), range_max=1.0)
    C, _, _, _ = O.kmeans(O.range_vectors(f32.astype(np.float64)), 20, 0, 6)
    params = FilterParams(spatial=SpatialKernel.recursive(2.5), theta=0.25, m0=20)
    inp = _prepare_inputs(f, f)
    one, _, s1 = run_filter(inp, C, params)
    per_group = 40 * 52 * 8 * 4
    fixed = 40 * 52 * 4 * (21 + 20 + 16) + 4096
    many, _, s2 = run_filter(inp, C, params, plane_budget=fixed + 4 * per_group)
    torch.cuda.synchronize()
    assert (one - many).abs().max().item() <= 1e-6
    ref = O.fast_filter_with_landmarks(f32.astype(np.float64), f32.astype(np.float64), C, 0.25,
                                       "gaussian_recursive", 2.5, 0)
    assert np.abs(many.double().cpu().numpy() - ref["output"]).max() <= TOL


@pytest.mark.parametrize("rho,m,m0", [(3, 200000, 64), (16, 50000, 40), (27, 30000, 33), (5, 700, 9), (3, 1, 1)])
def test_seeding_runs_match_owner_handoff(rho, m, m0, monkeypatch):
    # the one-barrier thread-run seeding (k_seed_runs) draws the same k-means++
    # picks as the owner-handoff kernel (NYS_SEED_V1=1) and the FP64 oracle
    from paper_1901_06112_b200.landmarks import kmeans_device

    rng = np.random.default_rng(rho * 1000 + m0)
    pts = rng.uniform(0, 1, (rho, m)).astype(np.float32)
    t = torch.from_numpy(pts).cuda()
    a = kmeans_device(t, m0, seed=4, max_iter=2)
    monkeypatch.setenv("NYS_SEED_V1", "1")
    b = kmeans_device(t, m0, seed=4, max_iter=2)
    assert np.array_equal(a.seed_indices, b.seed_indices)
    assert np.array_equal(a.centroids, b.centroids)
    if m <= 1000:
        rs = np.random.default_rng(4)
        seeds = O.plus_plus_seeds(pts.T.astype(np.float64), m0, rs)
        assert np.array_equal(pts.T.astype(np.float64)[a.seed_indices], seeds)


@pytest.mark.parametrize("shape,m0,theta", [((130, 9), 5, 0.35), ((64, 64), 5, 0.35), ((48, 56), 12, 0.2)])
@pytest.mark.parametrize("kind", ["gaussian_fir", "gaussian_recursive", "box"])
def test_ill_conditioned_kernels_use_phi_form(shape, m0, theta, kind):
    # 1-D guides with several landmarks: cond(A) 6e6 .. 1e8+, where the FP32 y-form missed 1e-4 by
    # up to 400x; the phi-form (nys_filter_desc.phi_form) keeps the reference's accuracy
    from paper_1901_06112_b200.nystrom import mixing_plan

    H, W = shape
    f32 = np.ascontiguousarray(color_scene(H, W, 5, 0.05, seed=H + 1)[:1])
    f64 = f32.astype(np.float64)
    C, _, _, _ = O.kmeans(O.range_vectors(f64), m0, 0, 6)
    sk = {"gaussian_fir": SpatialKernel.gaussian(2.5, 8), "gaussian_recursive": SpatialKernel.recursive(2.5),
          "box": SpatialKernel.box(4)}[kind]
    assert mixing_plan(C, theta, 1e-8, sk.effective_radius()).phi_form
    f = Image(data=torch.from_numpy(f32).cuda(), range_max=1.0)
    rep = filter_with_landmarks(f, f, C, FilterParams(spatial=sk, theta=theta, m0=m0))
    ref = O.fast_filter_with_landmarks(f64, f64, C, theta, kind, 2.5, 8 if kind != "box" else 4)
    out = rep.output.data.double().cpu().numpy()
    assert np.abs(out - ref["output"]).max() <= TOL
    assert rep.guarded_pixels == ref["guarded_pixels"]
    assert rep.retained_rank == ref["retained_rank"]


@pytest.mark.parametrize("m0,rho,theta", [(64, 3, 0.1), (60, 5, 0.3), (13, 4, 0.2), (8, 3, 0.2), (41, 31, 0.4)])
def test_device_inverse_from_cholesky_matches_host_M(m0, rho, theta):
    # nys_filter_desc.M_is_cholesky: the device forms M = L^{-T} L^{-1} (k_inverse_cholesky, blocked
    # 8-row substitution, n padded to a multiple of 8); the prepared workspace must equal the one
    # prepared from the host's M up to FP32 rounding of M, everything else bit-identical
    import ctypes as C

    from paper_1901_06112_b200 import _native
    from paper_1901_06112_b200._device import ptr, stream_ptr
    from paper_1901_06112_b200.filters import _desc
    from paper_1901_06112_b200.nystrom import mixing_plan

    cen = np.random.default_rng(m0 + rho).random((m0, rho))
    host = mixing_plan(cen, theta, 1e-8, 15)
    dev = mixing_plan(cen, theta, 1e-8, 15, lite=True, device_inverse=True)
    assert dev.M_is_cholesky and not host.M_is_cholesky and not host.phi_form
    lib = _native.lib()
    wss, m64s = [], []
    for plan in (host, dev):
        keep: list = []
        d = _desc(3, rho, 64, 64, 0, SpatialKernel.gaussian(5.0, 15), theta, cen, plan, keep)
        wsb = int(lib.nys_filter_workspace_bytes(C.byref(d)))
        ws = torch.zeros((wsb // 4,), dtype=torch.float32, device="cuda")
        _native.check(lib.nys_filter_prepare(C.byref(d), ptr(ws), wsb, stream_ptr()), "nys_filter_prepare")
        lay = np.zeros(8, np.int64)
        _native.check(lib.nys_filter_workspace_layout(C.byref(d), lay.ctypes.data), "layout")
        stats_floats, m64_off = int(lay[1]) // 4, int(lay[3]) // 4
        wss.append(ws[:stats_floats].cpu().numpy().view(np.uint32))
        m64s.append(ws[m64_off:m64_off + 2 * m0 * m0].cpu().numpy().view(np.float64).reshape(m0, m0))
    # float block (filter_layout: C, MT, U0, SC) then the FP64 block (C64, U064, SC64)
    off_d = int(lay[0]) // 4
    dblk = [w[off_d:off_d + 2 * (m0 * rho + m0 + 4)].view(np.float64) for w in wss]
    np.testing.assert_array_equal(dblk[0][:m0 * rho], dblk[1][:m0 * rho])  # landmarks
    # u0, 1/alpha_1, eps_den, alpha_1: full eigensystem vs the lite plan's inverse iteration
    np.testing.assert_allclose(dblk[0][m0 * rho:], dblk[1][m0 * rho:], rtol=1e-9, atol=1e-12)
    a, b = (w[:off_d] for w in wss)
    # the FP64 M of the near-guard refinement: host M vs the device's FP64 inverse
    np.testing.assert_allclose(m64s[1], host.M, rtol=0, atol=1e-9 * np.abs(host.M).max())
    np.testing.assert_array_equal(m64s[0], host.M)
    differ = a != b  # bit patterns (the FP64 block would read as NaN floats)
    af, bf = a.view(np.float32), b.view(np.float32)
    scale = np.abs(host.M).max()
    assert np.abs(af[differ] - bf[differ]).max(initial=0.0) <= 1e-6 * scale
    assert differ.sum() <= m0 * m0  # only the M block may differ


@pytest.mark.parametrize("cfg,H", [(2, 96), (3, 64), (4, 48), (1, None)])
def test_pipelined_plan_equals_synchronous_plan(cfg, H, monkeypatch):
    # fast_filter queues the whole step (in-stream plan on a side stream, nys_filter_plan_async);
    # it must give exactly the synchronous path's results
    from bench import _guide, _params

    wl = CONFIGS[cfg]
    img = wl.image(seed=1, H=H)
    params = _params(wl)
    f = Image(data=torch.from_numpy(img).cuda(), range_max=1.0)
    p = _guide(f, wl)
    a = fast_filter(f, p, params)
    monkeypatch.setenv("NYS_PIPELINED", "0")
    b = fast_filter(f, p, params)
    assert torch.equal(a.output.data, b.output.data)
    assert a.guarded_pixels == b.guarded_pixels and a.retained_rank == b.retained_rank
    assert a.quant_error == b.quant_error and a.min_denominator == b.min_denominator
    assert np.array_equal(a.centroids, b.centroids)


def test_pipelined_plan_falls_back_when_speculation_misses():
    # an ill-conditioned landmark kernel (1-D guide): the in-stream plan reports NYS_EUNSUPPORTED
    # and fast_filter reruns the step with the full plan (phi-form) -- still within 1e-4 of the oracle
    f32 = np.ascontiguousarray(color_scene(130, 9, 5, 0.05, seed=131)[:1])
    f = Image(data=torch.from_numpy(f32).cuda(), range_max=1.0)
    params = FilterParams(spatial=SpatialKernel.gaussian(2.5, 8), theta=0.35, m0=5, kmeans_max_iter=6)
    rep = fast_filter(f, f, params)
    C, _, _, _ = O.kmeans(O.range_vectors(f32.astype(np.float64)), 5, 0, 6)
    np.testing.assert_allclose(rep.centroids, C, rtol=0, atol=1e-9)
    ref = O.fast_filter_with_landmarks(f32.astype(np.float64), f32.astype(np.float64), C, 0.35, "gaussian_fir", 2.5, 8)
    assert np.abs(rep.output.data.double().cpu().numpy() - ref["output"]).max() <= TOL
    assert rep.retained_rank == ref["retained_rank"]


@pytest.mark.parametrize("rho,m0", [(1, 5), (3, 64), (16, 48), (27, 64), (31, 40)])
def test_exact_assignment_filter_equals_fp64_brute_force(rho, m0):
    # k_exact evaluates FP64 only for the centroids its FP32 error bound cannot exclude; labels
    # (first index on ties) and the FP64 minima must equal numpy's brute force, including exact
    # ties (duplicated centroids, points on bisectors) and ~1e-12 near-ties
    from paper_1901_06112_b200.landmarks import exact_assignment

    rng = np.random.default_rng(rho * 100 + m0)
    C = rng.random((m0, rho))
    C[m0 // 2] = C[1]                                  # duplicate centroid: exact ties for its points
    P = rng.random((6000, rho)).astype(np.float32).astype(np.float64)
    P[:200] = ((C[0] + C[2]) / 2).astype(np.float32)   # on (close to) the bisector of 0 and 2
    P[200:400] = C[1].astype(np.float32)               # nearest is the duplicated pair
    C[3] = C[4] + 1e-12                                # near-tie pair
    P[400:600] = C[4].astype(np.float32)
    d2 = ((P[:, None, :] - C[None, :, :]) ** 2).sum(axis=2)
    ref_lab = np.argmin(d2, axis=1)
    ref_qe = float(np.min(d2, axis=1).sum())
    pts = torch.from_numpy(np.ascontiguousarray(P.T.astype(np.float32))).cuda()
    asg, qe = exact_assignment(pts, C)
    np.testing.assert_array_equal(asg.cpu().numpy(), ref_lab)
    assert qe == pytest.approx(ref_qe, rel=1e-12)


@pytest.mark.parametrize("m0,theta", [(80, 0.12), (128, 0.04), (96, 0.06)])
def test_pipelined_plan_with_host_formed_M(m0, theta, monkeypatch):
    # above 64 landmarks the in-stream plan carries M formed by the worker (no device inverse);
    # still exactly the synchronous path's results, and the plan reports rank m0 and alpha_1
    from paper_1901_06112_b200.filters import plan_staging_buffers
    from paper_1901_06112_b200.nystrom import mixing_plan

    img = color_scene(72, 96, 30, 0.05, seed=m0)
    f = Image(data=torch.from_numpy(img).cuda(), range_max=1.0)
    params = FilterParams(spatial=SpatialKernel.gaussian(2.0, 6), theta=theta, m0=m0, kmeans_max_iter=8)
    a = fast_filter(f, f, params)
    plan = mixing_plan(a.centroids, theta, params.eps_drop, 6)
    if plan.phi_form or plan.rank < m0:
        pytest.skip("landmark kernel outside the speculation (the fallback test covers it)")
    import ctypes as C

    from paper_1901_06112_b200 import _native

    r = _native.PlanResult()
    bufs = plan_staging_buffers()
    assert any(_native.lib().nys_filter_plan_result(b.data_ptr(), C.byref(r)) == 0 and r.rank == m0
               and r.alpha0 == pytest.approx(plan.alpha0, rel=1e-13) for b in bufs)
    monkeypatch.setenv("NYS_PIPELINED", "0")
    b = fast_filter(f, f, params)
    assert torch.equal(a.output.data, b.output.data)
    assert a.guarded_pixels == b.guarded_pixels and a.retained_rank == b.retained_rank == m0


def test_pipelined_calls_from_two_host_threads():
    # each host thread gets its own staging / result buffers; the plan worker serves both
    import threading

    imgs = [color_scene(64, 80, 12, 0.05, seed=s) for s in (5, 6)]
    params = FilterParams(spatial=SpatialKernel.gaussian(2.0, 6), theta=0.15, m0=16, kmeans_max_iter=6)
    ref = []
    for im in imgs:
        f = Image(data=torch.from_numpy(im).cuda(), range_max=1.0)
        ref.append(fast_filter(f, f, params).output.data.clone())
    out = [None, None]
    errs = []

    def work(k):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                f = Image(data=torch.from_numpy(imgs[k]).cuda(), range_max=1.0)
                for _ in range(5):
                    r = fast_filter(f, f, params)
                out[k] = r.output.data.clone()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=work, args=(k,)) for k in (0, 1)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not errs, errs
    torch.cuda.synchronize()
    for k in (0, 1):
        assert torch.equal(out[k], ref[k])


def test_pipelined_calls_from_two_host_threads_full_size():
    # at full size the seeding / Lloyd launches are cooperative (a CTA on every SM)
    # while another stream's device gate (k_inverse_cholesky) may be spinning on an SM for its
    # plan; the plan worker must never block one job behind another, or the two streams wait on
    # each other until the 60 s timeouts.  Two threads, own streams, 1080p cfg 2 calls.
    import threading
    import time

    from bench import _params
    from paper_1901_06112_b200.synthetic import CONFIGS

    wl = CONFIGS[2]
    params = _params(wl)
    imgs = [wl.image(seed=s) for s in (0, 1)]
    ref = []
    for im in imgs:
        f = Image(data=torch.from_numpy(im).cuda(), range_max=1.0)
        ref.append(fast_filter(f, f, params).output.data.clone())
    out = [None, None]
    errs = []

    def work(k):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                f = Image(data=torch.from_numpy(imgs[k]).cuda(), range_max=1.0)
                for _ in range(6):
                    r = fast_filter(f, f, params)
                out[k] = r.output.data.clone()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    t0 = time.monotonic()
    th = [threading.Thread(target=work, args=(k,)) for k in (0, 1)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not errs, errs
    torch.cuda.synchronize()
    assert time.monotonic() - t0 < 30, "the two streams waited on each other"
    for k in (0, 1):
        assert torch.equal(out[k], ref[k])


def test_pipelined_call_after_an_interrupted_one():
    # a call that dies between the plan's fork and its final wait leaves its staging buffer
    # pending; the next call on the thread waits for that plan instead of failing
    import paper_1901_06112_b200.filters as F

    img = color_scene(48, 64, 8, 0.05, seed=9)
    f = Image(data=torch.from_numpy(img).cuda(), range_max=1.0)
    params = FilterParams(spatial=SpatialKernel.gaussian(2.0, 6), theta=0.15, m0=12, kmeans_max_iter=5)
    ref = fast_filter(f, f, params).output.data.clone()
    orig = F.exact_assignment_async

    def boom(*a, **k):
        raise RuntimeError("interrupted")

    F.exact_assignment_async = boom
    try:
        with pytest.raises(RuntimeError, match="interrupted"):
            fast_filter(f, f, params)
    finally:
        F.exact_assignment_async = orig
    assert torch.equal(fast_filter(f, f, params).output.data, ref)
