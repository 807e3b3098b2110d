"""Generate tests/golden/*.npz by running the REFERENCE package itself.

Run in the build container only (the reference lives at /root/reference and
does not travel to the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba python tools/make_golden.py

Each fixture stores the inputs (float32, exactly representable in the
reference's float64), the reference's outputs, and the parameters.  The
oracle (oracle/nys_oracle.py) is pinned against these in
tests/test_oracle_golden.py and the CUDA path in tests/test_gpu_*.py.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
REF = Path("/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))

import nysfilter as ref  # noqa: E402  (the reference, imported read-only)
from nysfilter.landmarks import kmeans_landmarks as ref_kmeans  # noqa: E402

from paper_1901_06112_b200.synthetic import color_scene, spectral_scene  # noqa: E402
from oracle.nys_oracle import patch_stack  # noqa: E402

OUT = ROOT / "tests" / "golden"


def _filter_case(name, f32, guide32, spatial, theta, m0, max_iter, mode="bilateral", eps_drop=1e-8):
    f = ref.Image(data=f32.astype(np.float64), range_max=1.0)
    p = f if guide32 is None else ref.Image(data=guide32.astype(np.float64), range_max=1.0)
    if spatial[0] == "box":
        sk = ref.SpatialKernel.box(spatial[1])
    elif spatial[0] == "recursive":
        sk = ref.SpatialKernel.recursive(spatial[1])
        spatial = ("gaussian_recursive", spatial[1], sk.effective_radius())
    else:
        sk = ref.SpatialKernel.gaussian(spatial[1], spatial[2])
    params = ref.FilterParams(spatial=sk, theta=theta, m0=m0, seed=0, mode=mode, kmeans_max_iter=max_iter,
                              eps_drop=eps_drop)
    rep = ref.fast_filter(f, p, params)
    rl = ref.extract_range_list(p)
    lm = ref_kmeans(rl.vectors, m0, seed=0, max_iter=max_iter)
    np.savez_compressed(
        OUT / f"{name}.npz", f=f32, guide=(f32 if guide32 is None else guide32),
        guide_is_f=guide32 is None, spatial_kind=spatial[0],
        sigma=(0.0 if spatial[0] == "box" else spatial[1]), radius=(spatial[1] if spatial[0] == "box" else spatial[2]),
        theta=theta, m0=m0, max_iter=max_iter, eps_drop=eps_drop,
        output=rep.output.data, retained_rank=rep.retained_rank, quant_error=rep.quant_error,
        min_denominator=rep.min_denominator, guarded_pixels=rep.guarded_pixels,
        centroids=lm.centroids, assignment=lm.assignment, errors=np.array(lm.errors))
    print(name, "rank", rep.retained_rank, "guarded", rep.guarded_pixels, "qe", rep.quant_error)


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    # BLF colour, FIR radius 9 (the cfg-1 kernel: sigma 3, R 9, theta 0.15, m0 32, 10 it)
    f = color_scene(64, 72, 8, 0.04, seed=11)
    _filter_case("blf_rgb_fir9", f, None, ("gaussian", 3.0, 9), 0.15, 32, 10)
    # BLF colour, small generic radius (runtime-radius kernels)
    f = color_scene(40, 48, 6, 0.05, seed=12)
    _filter_case("blf_rgb_fir4", f, None, ("gaussian", 1.5, 4), 0.1, 8, 15)
    # joint BLF with an external 2-channel guide
    g = color_scene(40, 48, 5, 0.05, seed=13)[:2].copy()
    _filter_case("joint_rgb_g2", f, g, ("gaussian", 2.0, 5), 0.2, 6, 10, mode="joint")
    # NLM: raw 3x3x3 patch guide, box(10) -> cfg-3 semantics at small size
    f = color_scene(48, 40, 6, 0.08, seed=14, lo=0.1, hi=0.9, shading=0.1)
    P = patch_stack(f.astype(np.float64), 1).astype(np.float32)
    _filter_case("nlm_patch_box10", f, P, ("box", 10), 0.3 * np.sqrt(27.0) * 0.08, 16, 15, mode="joint")
    # NLM with a small box (edge-heavy)
    _filter_case("nlm_patch_box3", f, P, ("box", 3), 0.3 * np.sqrt(27.0) * 0.08, 8, 15, mode="joint")
    # hyperspectral: 31 bands, FIR radius 12 (cfg-4 kernel), m0 12
    h = spectral_scene(32, 40, 31, 6, 0.03, seed=15)
    _filter_case("hyper31_fir12", h, None, ("gaussian", 4.0, 12), 0.25, 12, 15)
    # hyperspectral: 16 bands, FIR radius 18 (cfg-5 kernel), m0 10
    h = spectral_scene(40, 44, 16, 6, 0.03, seed=16)
    _filter_case("hyper16_fir18", h, None, ("gaussian", 6.0, 18), 0.2, 10, 15)
    # FIR radius 15 (cfg-2 kernel)
    f = color_scene(48, 56, 10, 0.05, seed=17)
    _filter_case("blf_rgb_fir15", f, None, ("gaussian", 5.0, 15), 0.1, 16, 15)

    # k-means known answers (reference test inputs + seeded blobs)
    km = {}
    cases = {
        "two_points": (np.array([[0.0], [10.0]]), 2, 0, 50),
        "two_cluster": (np.array([[0.0], [2.0], [10.0], [12.0]]), 2, 0, 50),
        "single": (np.array([[0.0], [2.0], [10.0], [12.0]]), 1, 3, 50),
        "ties": (np.array([[0.0], [1.0], [2.0]]), 2, 9, 50),
        "empty_repair": (np.array([[0.0], [0.0], [0.0], [100.0], [100.0], [0.1]]), 3, 0, 50),
    }
    rng = np.random.default_rng(6)
    cases["rgb200"] = (np.round(rng.uniform(0, 255, (200, 3))).astype(np.float64), 8, 11, 50)
    rng = np.random.default_rng(8)
    centers = rng.uniform(0, 50, (3, 2))
    cases["blobs"] = (np.concatenate([c + rng.standard_normal((50, 2)).astype(np.float32) for c in centers]
                                     ).astype(np.float64), 3, 4, 200)
    for k, (pts, m0, seed, it) in cases.items():
        lm = ref_kmeans(pts, m0, seed=seed, max_iter=it)
        km[f"{k}__points"] = pts
        km[f"{k}__meta"] = np.array([m0, seed, it])
        km[f"{k}__centroids"] = lm.centroids
        km[f"{k}__assignment"] = lm.assignment
        km[f"{k}__quant_error"] = np.array(lm.quant_error)
        km[f"{k}__errors"] = np.array(lm.errors)
    np.savez_compressed(OUT / "kmeans_kat.npz", **km)

    # Jacobi eigensystems (symeig.py) on landmark kernels and random symmetric matrices
    ev = {}
    rng = np.random.default_rng(0)
    for i, k in enumerate((1, 2, 5, 16, 33)):
        A = rng.standard_normal((k, k))
        A = A + A.T
        es = ref.jacobi_eig(ref.SymMatrix(A))
        ev[f"m{i}__a"] = A
        ev[f"m{i}__values"] = es.values
        ev[f"m{i}__vectors"] = es.vectors
    lms = rng.uniform(0, 1, (24, 3))
    A = ref.build_A(lms, ref.RangeKernel(theta=0.2)).entries
    es = ref.jacobi_eig(ref.SymMatrix(A))
    ev["kern__a"], ev["kern__values"], ev["kern__vectors"] = A, es.values, es.vectors
    np.savez_compressed(OUT / "jacobi.npz", **ev)

    # separable convolution known answers (spatial.py)
    sp = {}
    rng = np.random.default_rng(4)
    plane = rng.uniform(0, 1, (11, 13))
    sp["plane"] = plane
    sp["fir_1.3_3"] = ref.gaussian_fir(plane, 1.3, 3)
    sp["box_2"] = ref.box_filter(plane, 2)
    sp["box_0"] = ref.box_filter(plane, 0)
    np.savez_compressed(OUT / "spatial.npz", **sp)

    # full-rank exactness (SPEC.md acceptance #1): fast == brute at m0 = m, eps_drop = 0
    f = color_scene(12, 12, 4, 0.05, seed=18)
    fi = ref.Image(data=f.astype(np.float64), range_max=1.0)
    params = ref.FilterParams(spatial=ref.SpatialKernel.gaussian(1.0, 3), theta=0.3, m0=144, seed=0,
                              eps_drop=0.0, kmeans_max_iter=5)
    rep = ref.fast_filter(fi, fi, params)
    brute = ref.brute_force_filter(fi, fi, params)
    np.savez_compressed(OUT / "full_rank.npz", f=f, fast=rep.output.data, brute=brute.data,
                        retained_rank=rep.retained_rank)
    print("full rank: max|fast-brute|", np.abs(rep.output.data - brute.data).max(), "rank", rep.retained_rank)


def main_recursive():
    """§8 row f2: recursive Gaussian (spatial.py:114-191) known answers."""
    from nysfilter.spatial import _vyv_coeffs

    sig = np.array([1.0, 1.3, 2.5, 3.0, 5.0, 6.0, 12.7, 40.0])
    rec = {"sigmas": sig, "coeffs": np.array([_vyv_coeffs(float(s)) for s in sig])}
    rng = np.random.default_rng(21)
    plane = rng.uniform(0, 1, (19, 23))
    rec["plane"] = plane
    for s in (0.7, 1.0, 2.5, 4.0):
        rec[f"rec_{s}"] = ref.gaussian_recursive(plane, s)
    np.savez_compressed(OUT / "recursive.npz", **rec)
    f = color_scene(48, 56, 8, 0.05, seed=22)
    _filter_case("blf_rgb_rec3", f, None, ("recursive", 3.0), 0.15, 16, 10)
    f = color_scene(40, 44, 6, 0.05, seed=23)
    _filter_case("blf_rgb_rec07", f, None, ("recursive", 0.7), 0.12, 8, 10)
    g = color_scene(40, 44, 5, 0.05, seed=24)[:2].copy()
    _filter_case("joint_rgb_rec15", f, g, ("recursive", 1.5), 0.2, 6, 10, mode="joint")
    h = spectral_scene(32, 36, 16, 6, 0.03, seed=25)
    _filter_case("hyper16_rec2", h, None, ("recursive", 2.0), 0.2, 10, 15)


def main_brute_metrics_io():
    """§8 rows f1 (brute_force_filter) and f4 (metrics, KFC1/PNM I/O)."""
    out = {}
    cases = {
        "fir": (color_scene(30, 34, 5, 0.05, seed=31), None, ref.SpatialKernel.gaussian(2.0, 6), 0.15),
        "box": (color_scene(26, 30, 5, 0.05, seed=32), None, ref.SpatialKernel.box(4), 0.2),
        "rec": (color_scene(28, 24, 5, 0.05, seed=33), None, ref.SpatialKernel.recursive(1.7), 0.12),
        "hyper": (spectral_scene(20, 22, 9, 5, 0.03, seed=34), None, ref.SpatialKernel.gaussian(1.5, 4), 0.25),
    }
    g = color_scene(24, 26, 5, 0.05, seed=35)
    cases["joint"] = (g, g[:2].copy() * 0.5 + 0.25, ref.SpatialKernel.gaussian(1.5, 5), 0.2)
    fn = color_scene(22, 20, 4, 0.08, seed=36, lo=0.1, hi=0.9, shading=0.1)
    cases["nlm"] = (fn, patch_stack(fn.astype(np.float64), 1).astype(np.float32), ref.SpatialKernel.box(5),
                    0.3 * np.sqrt(27.0) * 0.08)
    for k, (f32, g32, sk, theta) in cases.items():
        fi = ref.Image(data=f32.astype(np.float64), range_max=1.0)
        gi = fi if g32 is None else ref.Image(data=g32.astype(np.float64), range_max=1.0)
        params = ref.FilterParams(spatial=sk, theta=theta, m0=4)
        out[f"{k}__f"] = f32
        out[f"{k}__guide"] = f32 if g32 is None else g32
        out[f"{k}__meta"] = np.array([{"box": 0, "gaussian_fir": 1, "gaussian_recursive": 2}[sk.kind],
                                      sk.sigma, sk.radius, theta])
        out[f"{k}__output"] = ref.brute_force_filter(fi, gi, params).data
    np.savez_compressed(OUT / "brute.npz", **out)

    from nysfilter import metrics as M

    mt = {}
    rng = np.random.default_rng(37)
    pairs = {
        "rgb": (rng.uniform(0, 1, (3, 40, 52)), 1.0),
        "u8": (np.round(rng.uniform(0, 255, (1, 33, 29))), 255.0),
        "small": (rng.uniform(0, 1, (2, 7, 30)), 1.0),        # below the 11x11 window
        "hyper": (rng.uniform(0, 1, (6, 24, 20)), 1.0),
    }
    for k, (a, R) in pairs.items():
        b = np.clip(a + rng.normal(0, 0.05 * R, a.shape), 0, R)
        ia, ib = ref.Image(data=a, range_max=R), ref.Image(data=b, range_max=R)
        mt[f"{k}__a"], mt[f"{k}__b"], mt[f"{k}__R"] = a, b, np.array(R)
        mt[f"{k}__mse"] = np.array(M.mse(ia, ib))
        mt[f"{k}__psnr"] = np.array(M.psnr(ia, ib))
        mt[f"{k}__psnr_band"] = np.array(M.psnr(ia, ib, per_band=True))
        mt[f"{k}__ssim"] = np.array(M.ssim(ia, ib))
    mt["same__psnr"] = np.array(M.psnr(ref.Image(data=pairs["rgb"][0], range_max=1.0),
                                       ref.Image(data=pairs["rgb"][0], range_max=1.0)))
    np.savez_compressed(OUT / "metrics.npz", **mt)

    import tempfile

    io = {}
    with tempfile.TemporaryDirectory() as td:
        cube = rng.uniform(0, 1, (5, 6, 7))
        for dt in ("float32", "float64"):
            pth = Path(td) / f"c_{dt}.kfc"
            ref.save_image(ref.Image(data=cube, range_max=1.0), pth, cube_dtype=dt)
            io[f"cube_{dt}"] = np.frombuffer(pth.read_bytes(), dtype=np.uint8)
        rgb = rng.uniform(-10, 265, (3, 5, 4))
        gray = rng.uniform(0, 255, (1, 4, 6))
        for nm, img in (("ppm", rgb), ("pgm", gray)):
            pth = Path(td) / f"x.{nm}"
            ref.save_image(ref.Image(data=img, range_max=255.0), pth)
            io[f"pnm_{nm}"] = np.frombuffer(pth.read_bytes(), dtype=np.uint8)
        io["cube"], io["rgb"], io["gray"] = cube, rgb, gray
    np.savez_compressed(OUT / "image_io.npz", **io)
    print("brute / metrics / io fixtures written")


def main_pca():
    """§8 row f3: PCA patch guides with pca_dim < full (filters.py:161-187)
    and NLM-mode filters on them."""
    from nysfilter.filters import pca_patch_guide as ref_pca

    out = {}
    for name, (f32, r, k) in {
        "r1k10": (color_scene(30, 34, 5, 0.08, seed=41, lo=0.1, hi=0.9, shading=0.1), 1, 10),
        "r2k25": (color_scene(36, 40, 5, 0.08, seed=42, lo=0.1, hi=0.9, shading=0.1), 2, 25),
        "r3k25": (color_scene(40, 44, 6, 0.08, seed=43, lo=0.1, hi=0.9, shading=0.1), 3, 25),
        "gray_r3k6": (color_scene(32, 30, 5, 0.08, seed=44)[:1].copy(), 3, 6),
    }.items():
        g = ref_pca(ref.Image(data=f32.astype(np.float64), range_max=1.0), r, k).data
        out[f"{name}__f"], out[f"{name}__meta"], out[f"{name}__guide"] = f32, np.array([r, k]), g
    np.savez_compressed(OUT / "pca_guide.npz", **out)
    # NLM-mode filters (the CLI's nlm path at small size): guide = PCA(r, k) of f
    for name, (f32, r, k, S, m0) in {
        "nlm_pca_r2k12": (color_scene(36, 40, 5, 0.08, seed=45, lo=0.1, hi=0.9, shading=0.1), 2, 12, 5, 12),
        "nlm_pca_r3k25": (color_scene(32, 36, 5, 0.08, seed=46, lo=0.1, hi=0.9, shading=0.1), 3, 25, 4, 10),
    }.items():
        fi = ref.Image(data=f32.astype(np.float64), range_max=1.0)
        theta = 0.3 * np.sqrt(3 * (2 * r + 1) ** 2) * 0.08  # cfg-3 rule on the raw patch dimension
        params = ref.FilterParams(spatial=ref.SpatialKernel.box(S), theta=theta, m0=m0, seed=0, mode="nlm",
                                  patch_radius=r, pca_dim=k, kmeans_max_iter=15)
        p = ref.build_guide(fi, "nlm", None, r, k)
        rep = ref.fast_filter(fi, p, params)
        lm = ref_kmeans(ref.extract_range_list(p).vectors, m0, seed=0, max_iter=15)
        np.savez_compressed(OUT / f"{name}.npz", f=f32, guide=p.data, patch_radius=r, pca_dim=k, radius=S,
                            theta=theta, m0=m0, output=rep.output.data, retained_rank=rep.retained_rank,
                            quant_error=rep.quant_error, guarded_pixels=rep.guarded_pixels,
                            min_denominator=rep.min_denominator, centroids=lm.centroids)
        print(name, "rank", rep.retained_rank, "guarded", rep.guarded_pixels, "qe", rep.quant_error)


if __name__ == "__main__":
    which = sys.argv[1:] or ["base", "recursive", "f1f4", "pca"]
    if "pca" in which:
        main_pca()
    if "f1f4" in which:
        main_brute_metrics_io()
    if "base" in which:
        main()
    if "recursive" in which:
        main_recursive()
