"""CPU-side checks: the C-ABI library loads and exports every declared entry
point, the host FP64 pieces (Jacobi, mixing plan), the band planner, and the
drop-in API's validation behaviour.  No device compute."""

import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, group, load_golden
from oracle import nys_oracle as O
from paper_1901_06112_b200 import (
    FilterParams,
    Image,
    SpatialKernel,
    SymMatrix,
    _native,
    build_guide,
    jacobi_eig,
)
from paper_1901_06112_b200.bands import halo_rows, plan_bands, shard_rows
from paper_1901_06112_b200.nystrom import DegenerateKernelError, _retain, mixing_plan


def _declared_symbols():
    text = (ROOT / "include" / "nysfilter_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|uint64_t|int64_t)\s+(nys_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    declared = _declared_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_native.exported_symbols()) == declared
    assert lib.nys_abi_version() == 100


def test_native_jacobi_matches_reference_bitwise():
    for name, c in group(load_golden("jacobi"), "").items():
        es = jacobi_eig(SymMatrix(c["a"]))
        np.testing.assert_array_equal(es.values, c["values"], err_msg=name)
        np.testing.assert_allclose(es.vectors, c["vectors"], rtol=0, atol=1e-15, err_msg=name)


def test_jacobi_known_answers():
    es = jacobi_eig(SymMatrix(np.eye(3)))
    np.testing.assert_array_equal(es.values, np.ones(3))
    es = jacobi_eig(SymMatrix(np.array([[2.0, 1.0], [1.0, 2.0]])))
    np.testing.assert_allclose(es.values, [3.0, 1.0], atol=1e-14)
    with pytest.raises(ValueError):
        SymMatrix(np.array([[1.0, np.nan], [0.0, 1.0]]))


def test_mixing_plan_matches_oracle_algebra():
    g = load_golden("blf_rgb_fir9")
    C = g["centroids"]
    plan = mixing_plan(C, float(g["theta"]), 1e-8, int(g["radius"]))
    vals, vecs = O.jacobi_eig(O.gram(C, C, float(g["theta"])))
    al, Wk = O.retain(vals, vecs, 1e-8)
    M = (Wk / al) @ Wk.T  # LAPACK vs Jacobi: agree to ~1e-10 of max|M| (cond(A) ~ 7e4 here)
    assert plan.phi_form  # cond(A) ~ 7e4 > PHI_FORM_COND: M holds P, P^T P = A^+
    np.testing.assert_allclose(plan.M.T @ plan.M, M, rtol=0, atol=1e-9 * np.abs(M).max())
    assert plan.alpha0 == pytest.approx(al[0], rel=1e-13)
    assert plan.eps_den == pytest.approx(1e-12 * (2 * 9 + 1) ** 2 * np.abs(al).max())


def test_drop_rule_and_degenerate():
    v, w = _retain(np.array([2.0, 1e-9, 1e-7]), np.eye(3), 1e-8)
    assert v.tolist() == [2.0, 1e-7]
    with pytest.raises(DegenerateKernelError):
        _retain(np.array([0.0, -1.0]), np.eye(2), 1e-8)


def test_filter_params_validation_matches_reference():
    sk = SpatialKernel.gaussian(2.0)
    assert sk.radius == 6
    with pytest.raises(ValueError):
        FilterParams(spatial=sk, theta=0.0)
    with pytest.raises(ValueError):
        FilterParams(spatial=sk, theta=1.0, m0=0)
    with pytest.raises(ValueError):
        FilterParams(spatial=sk, theta=1.0, mode="other")
    with pytest.raises(ValueError):
        FilterParams(spatial=sk, theta=1.0, eps_drop=1.0)
    with pytest.raises(ValueError):
        SpatialKernel.box(-1)
    with pytest.raises(ValueError):
        SpatialKernel(kind="gaussian_fir", sigma=1.0, radius=0)
    assert SpatialKernel.recursive(2.5).effective_radius() == 8


def test_image_contract():
    img = Image(data=np.arange(24.0).reshape(2, 3, 4))
    assert (img.channels, img.height, img.width) == (2, 3, 4)
    assert img.samples[1 * 12 + 2 * 4 + 3] == img.data[1, 2, 3]
    with pytest.raises(ValueError):
        Image(data=np.array([[np.inf]]))
    with pytest.raises(ValueError):
        Image(data=np.zeros((0, 3)))
    with pytest.raises(ValueError):
        build_guide(img, "joint")
    with pytest.raises(ValueError):
        build_guide(img, "joint", Image(data=np.zeros((1, 2, 2))))
    assert build_guide(img, "bilateral") is img


def test_plan_bands_cover_rows_with_halo():
    H, R = 1000, 18
    for budget_rows in (60, 100, 333, 2000):
        bands = plan_bands(H, R, row_bytes=7, budget_bytes=7 * budget_rows)
        assert bands[0].out0 == 0 and sum(b.out_rows for b in bands) == H
        for a, b in zip(bands, bands[1:]):
            assert a.out0 + a.out_rows == b.out0
        for b in bands:
            assert b.hp0 == b.out0 - R
            assert b.hp_rows == b.out_rows + 2 * R
            assert b.hp_rows <= budget_rows
    with pytest.raises(MemoryError):
        plan_bands(H, R, row_bytes=7, budget_bytes=7 * (2 * R))


def test_shard_rows_partition():
    for H in (1, 7, 1080, 8192):
        for G in (1, 2, 3, 8):
            if G > H:
                continue
            spans = [shard_rows(H, G, g) for g in range(G)]
            assert spans[0][0] == 0 and spans[-1][1] == H
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0 and a1 > a0
    assert halo_rows(0, 10, 100, 18) == (0, 28)
    assert halo_rows(50, 60, 100, 18) == (32, 78)
    assert halo_rows(90, 100, 100, 18) == (72, 100)


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1901_06112_b200 import fast_filter

    f = Image(data=np.random.default_rng(0).random((3, 8, 8)), range_max=1.0)
    with pytest.raises(RuntimeError):
        fast_filter(f, f, FilterParams(spatial=SpatialKernel.gaussian(1.0), theta=0.2, m0=4))


def test_public_names_are_native():
    import paper_1901_06112_b200 as P

    for name in ("brute_force_filter", "psnr", "ssim", "mse", "quality", "load_image", "save_image",
                 "gaussian_recursive", "box_filter", "gaussian_fir", "apply_planes"):
        assert callable(getattr(P, name)) and getattr(P, name).__name__ != "_f"


def test_header_cites_reference():
    text = (ROOT / "include" / "nysfilter_b200.h").read_text()
    for cite in ("landmarks.py:76-129", "filters.py:214-257", "symeig.py:58-125"):
        assert cite in text


@pytest.mark.parametrize("k,rho,theta", [(64, 3, 0.1), (64, 27, 1.3), (48, 31, 0.25), (6, 1, 0.3), (32, 3, 2.0),
                                         (64, 3, 0.5), (1, 3, 0.2)])
def test_native_mixing_plan_matches_eigh(k, rho, theta):
    # nys_mixing_plan (Cholesky fast path when nothing is dropped, full eigensystem otherwise)
    # against numpy's eigh + the reference drop rule
    from paper_1901_06112_b200.nystrom import PHI_FORM_COND, RangeKernel, _retain, build_A, mixing_plan

    C = np.random.default_rng(k * 100 + rho).random((k, rho))
    p = mixing_plan(C, theta, 1e-8, 15)
    A = build_A(C, RangeKernel(theta)).entries
    vals, vecs = np.linalg.eigh(A)
    o = np.argsort(vals)[::-1]
    al, Wr = _retain(vals[o], vecs[:, o], 1e-8)
    M = (Wr / al) @ Wr.T
    assert len(p.alphas) == len(al)
    np.testing.assert_allclose(p.alphas, al, rtol=0, atol=1e-13 * al[0])
    kappa = al[0] / al[-1]  # both solvers are backward stable: forward error ~ eps * kappa
    Mp = p.M.T @ p.M if p.phi_form else p.M  # phi-form above PHI_FORM_COND: M holds P, P^T P = A^+
    assert p.phi_form == (kappa > PHI_FORM_COND)
    assert np.abs(Mp - M).max() <= max(1e-12, 1e-14 * kappa) * np.abs(M).max()
    if k == 1 or al[0] - al[1] > 1e-6 * al[0]:  # u0 is defined up to sign when alpha_1 is simple
        assert min(np.abs(p.u0 - Wr[:, 0]).max(), np.abs(p.u0 + Wr[:, 0]).max()) <= 1e-9


def test_phi_form_plan_for_ill_conditioned_kernels():
    # cond(A) > PHI_FORM_COND -> phi-form: M holds P = diag(alpha^-1/2) W^T with P^T P = A^+ on the
    # retained eigenpairs, u0 the lead eigenvector (host only, no GPU)
    from paper_1901_06112_b200.nystrom import PHI_FORM_COND, mixing_plan

    C = np.array([[0.40], [0.45], [0.50], [0.55], [0.60], [0.62]])
    p = mixing_plan(C, 0.35, 1e-8, 8)
    assert p.phi_form and p.alphas[0] / p.alphas[-1] > PHI_FORM_COND
    A = np.exp(-((C - C.T) ** 2) / (2 * 0.35 ** 2))
    w, V = np.linalg.eigh(A)
    o = np.argsort(-w)
    w, V = w[o], V[:, o]
    keep = w > 1e-8 * w[0]
    Mref = (V[:, keep] / w[keep]) @ V[:, keep].T
    assert np.abs(p.M.T @ p.M - Mref).max() <= 1e-8 * np.abs(Mref).max()
    assert np.all(p.M[keep.sum():] == 0.0)
    assert min(np.abs(p.u0 - V[:, 0]).max(), np.abs(p.u0 + V[:, 0]).max()) <= 1e-10
    q = mixing_plan(np.random.default_rng(0).random((16, 3)), 0.2, 1e-8, 8)
    assert not q.phi_form


@pytest.mark.parametrize("k,rho,theta", [(64, 3, 0.1), (48, 31, 0.25), (64, 27, 1.3), (32, 3, 0.15), (5, 1, 0.35),
                                         (6, 1, 0.35)])
def test_lite_mixing_plan_matches_full(k, rho, theta):
    # the hot-path plan (alpha_1 by Sturm bisection + two Sturm counts) gives the full plan's
    # M, u0, alpha_1 and rank, or defers to it (drops / phi-form)
    from paper_1901_06112_b200.nystrom import mixing_plan

    C = np.random.default_rng(k + rho).random((k, rho))
    if k == 6:
        C = np.array([[0.40], [0.45], [0.50], [0.55], [0.60], [0.62]])  # cond 1e8: phi-form via the full plan
    a = mixing_plan(C, theta, 1e-8, 15)
    b = mixing_plan(C, theta, 1e-8, 15, lite=True)
    assert a.phi_form == b.phi_form and a.rank == b.rank
    assert b.alpha0 == pytest.approx(a.alpha0, rel=1e-14)
    assert b.eps_den == pytest.approx(a.eps_den, rel=1e-14)
    np.testing.assert_allclose(b.M, a.M, rtol=0, atol=1e-12 * np.abs(a.M).max())
    assert min(np.abs(a.u0 - b.u0).max(), np.abs(a.u0 + b.u0).max()) <= 1e-9


@pytest.mark.parametrize("k,rho,theta", [(64, 3, 0.1), (48, 31, 0.25), (32, 3, 0.15), (4, 2, 0.5)])
def test_lite_plan_cholesky_factor(k, rho, theta):
    # device_inverse=True hands the device the Cholesky factor L of A (A = L L^T) instead of M;
    # (L^{-1})^T L^{-1} must be the full plan's M, with the same u0 / alpha_1 / rank, and the
    # lite plan must not defer to the full one for a well-conditioned A
    from paper_1901_06112_b200.nystrom import mixing_plan

    C = np.random.default_rng(k + rho).random((k, rho))
    a = mixing_plan(C, theta, 1e-8, 15)
    b = mixing_plan(C, theta, 1e-8, 15, lite=True, device_inverse=True)
    assert b.M_is_cholesky and not b.phi_form and b.rank == a.rank == k
    L = np.tril(b.M)
    assert np.all(b.M[np.triu_indices(k, 1)] == 0.0)
    Li = np.linalg.inv(L)
    np.testing.assert_allclose(Li.T @ Li, a.M, rtol=0, atol=1e-10 * np.abs(a.M).max())
    assert b.alpha0 == pytest.approx(a.alpha0, rel=1e-14)
    assert min(np.abs(a.u0 - b.u0).max(), np.abs(a.u0 + b.u0).max()) <= 1e-9
