"""Pin the CPU oracle (oracle/nys_oracle.py) to the reference's own outputs.

tests/golden/*.npz were produced by running the reference package itself
(tools/make_golden.py).  The oracle is only trusted as a checker for the
CUDA path because these pass.
"""

import numpy as np
import pytest

from conftest import FILTER_CASES, group, load_golden, oracle_kind
from oracle import nys_oracle as O


@pytest.mark.parametrize("case", FILTER_CASES)
def test_oracle_filter_matches_reference(case):
    g = load_golden(case)
    res = O.fast_filter_with_landmarks(g["f"], g["guide"], g["centroids"], float(g["theta"]), oracle_kind(g),
                                       float(g["sigma"]), int(g["radius"]), float(g["eps_drop"]))
    assert res["retained_rank"] == int(g["retained_rank"])
    assert res["guarded_pixels"] == int(g["guarded_pixels"])
    np.testing.assert_allclose(res["output"], g["output"], rtol=0, atol=1e-9)
    assert res["min_denominator"] == pytest.approx(float(g["min_denominator"]), rel=1e-6, abs=1e-300)


@pytest.mark.parametrize("case", FILTER_CASES)
def test_oracle_kmeans_matches_reference(case):
    g = load_golden(case)
    C, lab, qe, errors = O.kmeans(O.range_vectors(g["guide"]), int(g["m0"]), 0, int(g["max_iter"]))
    np.testing.assert_array_equal(C, g["centroids"])
    np.testing.assert_array_equal(lab, g["assignment"])
    assert qe == float(g["quant_error"])
    np.testing.assert_array_equal(np.array(errors), g["errors"])


def test_oracle_kmeans_known_answers():
    cases = group(load_golden("kmeans_kat"), "")
    for name, c in cases.items():
        m0, seed, it = (int(v) for v in c["meta"])
        C, lab, qe, errors = O.kmeans(c["points"], m0, seed, it)
        np.testing.assert_array_equal(C, c["centroids"], err_msg=name)
        np.testing.assert_array_equal(lab, c["assignment"], err_msg=name)
        assert qe == float(c["quant_error"]), name
    # analytic answers from pkg/tests/test_landmarks.py:12-29
    C, _, qe, _ = O.kmeans(np.array([[0.0], [2.0], [10.0], [12.0]]), 2, 0)
    assert sorted(C.ravel().tolist()) == [1.0, 11.0] and qe == pytest.approx(4.0)
    C, _, qe, _ = O.kmeans(np.array([[0.0], [2.0], [10.0], [12.0]]), 1, 3)
    assert C.ravel().tolist() == [6.0] and qe == pytest.approx(104.0)


def test_oracle_jacobi_matches_reference():
    for name, c in group(load_golden("jacobi"), "").items():
        vals, vecs = O.jacobi_eig(c["a"])
        np.testing.assert_allclose(vals, c["values"], rtol=0, atol=1e-12, err_msg=name)
        np.testing.assert_allclose(vecs, c["vectors"], rtol=0, atol=1e-10, err_msg=name)


def test_oracle_spatial_known_answers():
    g = load_golden("spatial")
    np.testing.assert_allclose(O.spatial_conv(g["plane"][None], "gaussian_fir", 1.3, 3)[0], g["fir_1.3_3"],
                               rtol=0, atol=1e-13)
    np.testing.assert_allclose(O.spatial_conv(g["plane"][None], "box", 0, 2)[0], g["box_2"], rtol=0, atol=1e-13)
    np.testing.assert_array_equal(O.spatial_conv(g["plane"][None], "box", 0, 0)[0], g["box_0"])
    # pkg/tests/test_spatial.py:40-52 box constant / impulse
    for S in (0, 1, 3):
        out = O.spatial_conv(np.full((1, 6, 5), 2.5), "box", 0, S)[0]
        assert np.array_equal(out, np.full((6, 5), 2.5 * (2 * S + 1) ** 2))
    imp = np.zeros((1, 7, 7))
    imp[0, 3, 3] = 1
    exp = np.zeros((7, 7))
    exp[2:5, 2:5] = 1
    assert np.array_equal(O.spatial_conv(imp, "box", 0, 1)[0], exp)
    # FIR impulse ratio e^-1/2 (test_spatial.py:79-84)
    imp = np.zeros((1, 9, 9))
    imp[0, 4, 4] = 1
    out = O.spatial_conv(imp, "gaussian_fir", 1.0, 3)[0]
    assert out[4, 4] == pytest.approx(1.0) and out[4, 5] / out[4, 4] == pytest.approx(np.exp(-0.5))


def test_oracle_recursive_known_answers():
    """§8 f2: coefficients, the scan and the sigma < 1 FIR fallback vs the
    reference's gaussian_recursive (spatial.py:114-191, 206-208)."""
    g = load_golden("recursive")
    for s, c in zip(g["sigmas"], g["coeffs"]):
        np.testing.assert_allclose(O.vyv_coeffs(float(s)), c, rtol=1e-14, atol=1e-15)
    for s in (0.7, 1.0, 2.5, 4.0):
        out = O.spatial_conv(g["plane"][None], "gaussian_recursive", s, 0)[0]
        np.testing.assert_allclose(out, g[f"rec_{s}"], rtol=1e-12, atol=1e-12)
    # constants are preserved up to the mass^2 rescale (spatial.py:10-13)
    out = O.spatial_conv(np.full((1, 9, 12), 0.75), "gaussian_recursive", 2.0, 0)[0]
    np.testing.assert_allclose(out, 0.75 * O.fir_mass(2.0) ** 2, rtol=1e-12)


def test_native_vyv_coeffs_match_reference():
    """Host C++ nys_vyv_coeffs (no GPU needed) vs the reference's _vyv_coeffs."""
    import ctypes as C

    from paper_1901_06112_b200 import _native

    g = load_golden("recursive")
    for s, c in zip(g["sigmas"], g["coeffs"]):
        out = (C.c_double * 6)()
        _native.check(_native.lib().nys_vyv_coeffs(float(s), out), "nys_vyv_coeffs")
        np.testing.assert_allclose(np.array(out[:]), c, rtol=1e-14, atol=1e-15)
    out = (C.c_double * 6)()
    assert _native.lib().nys_vyv_coeffs(0.0, out) == _native.NYS_EINVAL


def test_oracle_full_rank_exactness():
    g = load_golden("full_rank")
    f = g["f"].astype(np.float64)
    res = O.fast_filter(f, f, 0.3, "gaussian_fir", 1.0, 3, m0=144, seed=0, max_iter=5, eps_drop=0.0)
    np.testing.assert_allclose(res["output"], g["fast"], atol=1e-9)
    brute = O.brute_force_filter(f, f, 0.3, "gaussian_fir", 1.0, 3)
    np.testing.assert_allclose(brute, g["brute"], atol=1e-12)
    assert np.abs(res["output"] - brute).max() < 1e-8


def test_choice_is_cumsum_searchsorted():
    """The k-means++ draw the GPU reproduces (landmarks.py:68)."""
    for seed in range(3):
        r1 = np.random.default_rng(seed)
        r2 = np.random.default_rng(seed)
        d2 = np.random.default_rng(100 + seed).random(5000) ** 3
        d2[::5] = 0.0
        for _ in range(10):
            a = r1.choice(d2.size, p=d2 / d2.sum())
            p = d2 / d2.sum()
            cdf = p.cumsum()
            cdf /= cdf[-1]
            assert a == np.searchsorted(cdf, r2.random(), side="right")


def test_vector_uniforms_equal_scalar_stream():
    r1 = np.random.default_rng(7)
    r2 = np.random.default_rng(7)
    assert r1.integers(1000) == r2.integers(1000)
    v = r1.random(50)
    assert np.array_equal(v, np.array([r2.random() for _ in range(50)]))


def test_patch_stack_order():
    f = np.arange(2 * 4 * 5, dtype=np.float64).reshape(2, 4, 5)
    P = O.patch_stack(f, 1)
    assert P.shape == (18, 4, 5)
    # channel-major, then dy, then dx, edge replicate (filters.py:176-181)
    assert P[4, 2, 3] == f[0, 2, 3]
    assert P[9 + 0, 0, 0] == f[1, 0, 0]
    assert P[9 + 8, 3, 4] == f[1, 3, 4]
    assert P[2, 1, 1] == f[0, 0, 2]


BRUTE_KIND = {0: "box", 1: "gaussian_fir", 2: "gaussian_recursive"}


def test_oracle_brute_force_matches_reference():
    """§8 f1 fixtures: Eq. (1) over box / FIR / recursive (as FIR) / joint /
    NLM-patch / 9-band guides (filters.py:116-138)."""
    for name, c in group(load_golden("brute"), "").items():
        kind, sigma, radius, theta = c["meta"]
        out = O.brute_force_filter(c["f"], c["guide"], float(theta), BRUTE_KIND[int(kind)], float(sigma),
                                   int(radius))
        np.testing.assert_allclose(out, c["output"], rtol=0, atol=1e-12, err_msg=name)


def test_oracle_metrics_match_reference():
    """§8 f4 fixtures: mse / psnr (global and per band) / ssim incl. the
    below-window global-statistics branch (metrics.py:37-122)."""
    g = load_golden("metrics")
    for name, c in group({k: v for k, v in g.items() if not k.startswith("same")}, "").items():
        R = float(c["R"])
        assert O.mse(c["a"], c["b"]) == pytest.approx(float(c["mse"]), rel=1e-13), name
        assert O.psnr(c["a"], c["b"], R) == pytest.approx(float(c["psnr"]), abs=1e-10), name
        assert O.psnr(c["a"], c["b"], R, per_band=True) == pytest.approx(float(c["psnr_band"]), abs=1e-10), name
        assert O.ssim(c["a"], c["b"], R) == pytest.approx(float(c["ssim"]), abs=1e-12), name
    a = g["rgb__a"]
    assert O.psnr(a, a, 1.0) == float(g["same__psnr"]) == 99.0


def test_oracle_pca_guide_matches_reference():
    """§8 f3 fixtures: truncated PCA patch guides (filters.py:161-187)."""
    for name, c in group(load_golden("pca_guide"), "").items():
        r, k = (int(v) for v in c["meta"])
        g = O.pca_patch_guide(c["f"].astype(np.float64), r, k)
        np.testing.assert_allclose(g, c["guide"], rtol=0, atol=1e-10, err_msg=name)


@pytest.mark.parametrize("case", ["nlm_pca_r2k12", "nlm_pca_r3k25"])
def test_oracle_nlm_pca_filter_matches_reference(case):
    g = load_golden(case)
    f = g["f"].astype(np.float64)
    p = O.pca_patch_guide(f, int(g["patch_radius"]), int(g["pca_dim"]))
    np.testing.assert_allclose(p, g["guide"], rtol=0, atol=1e-10)
    res = O.fast_filter_with_landmarks(f, p, g["centroids"], float(g["theta"]), "box", 0.0, int(g["radius"]))
    assert res["guarded_pixels"] == int(g["guarded_pixels"])
    np.testing.assert_allclose(res["output"], g["output"], rtol=0, atol=1e-9)
