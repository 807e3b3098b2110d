"""CPU oracle for the Nystrom kernel-filter hot path (TEST INFRASTRUCTURE ONLY).

This module is a from-scratch NumPy restatement of the reference package
``nysfilter`` 0.1.0 (``/root/reference/pkg/src/nysfilter``), used ONLY as the
checker in ``tests/``, by ``__graft_entry__.smoke()`` and by ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs.  The product path
(``paper_1901_06112_b200``) never imports it and has no CPU fallback.

Everything is float64, exactly like the reference (``image.py:41``).  Each
function cites the reference file:line whose semantics it restates.

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
``tests/golden/*.npz``, which ``tools/make_golden.py`` produced by running the
reference itself in the build container (the reference cannot travel to the
GPU box), plus the reference test suite's own known-answer cases
(``pkg/tests/test_spatial.py``, ``test_landmarks.py``, ``test_nystrom.py``,
``test_symeig.py``).
"""

from __future__ import annotations

import math
import time

import numpy as np

DEFAULT_EPS_DROP = 1e-8          # nystrom.py:24
DENOMINATOR_EPS_SCALE = 1e-12    # filters.py:54
JACOBI_MAX_SWEEPS = 100          # symeig.py:18
JACOBI_OFFDIAG_TOL = 1e-12       # symeig.py:19


# --------------------------------------------------------------------------
# range list (image.py:108-112): pixel-major (m, rho) copy of a planar guide
# --------------------------------------------------------------------------
def range_vectors(guide: np.ndarray) -> np.ndarray:
    rho = guide.shape[0]
    return np.ascontiguousarray(np.asarray(guide, np.float64).reshape(rho, -1).T)


# --------------------------------------------------------------------------
# k-means landmarks (landmarks.py:37-129)
# --------------------------------------------------------------------------
def assign(points: np.ndarray, centroids: np.ndarray, exact: bool = False):
    """Nearest centroid, first index on ties (landmarks.py:37-57).

    exact=False is the expansion form |x|^2 - 2 x.c + |c|^2 used inside the
    Lloyd loop; exact=True is the differenced form used for the final report.
    """
    if exact:
        d2 = np.stack([((points - c) ** 2).sum(axis=1) for c in centroids], axis=1)
    else:
        pn = (points * points).sum(axis=1)
        cn = (centroids * centroids).sum(axis=1)
        d2 = pn[:, None] - 2.0 * (points @ centroids.T) + cn[None, :]
    lab = np.argmin(d2, axis=1)
    nearest = np.maximum(d2[np.arange(points.shape[0]), lab], 0.0)
    return lab.astype(np.int64), nearest


def plus_plus_seeds(points: np.ndarray, m0: int, rng: np.random.Generator) -> np.ndarray:
    """k-means++ seeding (landmarks.py:60-73).

    The D^2 draw is ``Generator.choice(m, p=d2/total)``; its index equals
    searchsorted(cumsum(p)/cumsum(p)[-1], rng.random(), 'right'), one uniform
    per draw (verified against numpy in tests/test_oracle_golden.py).
    """
    m = points.shape[0]
    C = np.empty((m0, points.shape[1]))
    C[0] = points[rng.integers(m)]
    d2 = ((points - C[0]) ** 2).sum(axis=1)
    for j in range(1, m0):
        total = d2.sum()
        idx = rng.choice(m, p=d2 / total) if total > 0.0 else rng.integers(m)
        C[j] = points[idx]
        d2 = np.minimum(d2, ((points - C[j]) ** 2).sum(axis=1))
    return C


def kmeans(points: np.ndarray, m0: int, seed: int = 0, max_iter: int = 50):
    """k-means++ then Lloyd until labels repeat or max_iter (landmarks.py:76-129).

    Returns (centroids, assignment, quant_error, errors).
    """
    X = np.ascontiguousarray(np.asarray(points, np.float64))
    m, dim = X.shape
    if m0 < 1 or m0 > m:
        raise ValueError(f"m0 must be in [1, {m}], got {m0}")
    if max_iter < 1:
        raise ValueError("max_iter must be >= 1")
    rng = np.random.default_rng(seed)
    C = plus_plus_seeds(X, m0, rng)
    errors = []
    prev = None
    for _ in range(max_iter):
        lab, nearest = assign(X, C)
        errors.append(float(nearest.sum()))
        if prev is not None and np.array_equal(lab, prev):
            break
        prev = lab
        counts = np.bincount(lab, minlength=m0)
        sums = np.stack([np.bincount(lab, weights=X[:, d], minlength=m0)
                         for d in range(dim)], axis=1)
        occ = counts > 0
        C[occ] = sums[occ] / counts[occ, None]
        # empty clusters, ascending j: farthest remaining point (landmarks.py:114-119)
        taken = nearest.copy()
        for j in np.flatnonzero(~occ):
            k = int(np.argmax(taken))
            C[j] = X[k]
            taken[k] = -1.0
    lab, nearest = assign(X, C, exact=True)
    return C, lab, float(nearest.sum()), tuple(errors)


# --------------------------------------------------------------------------
# Gaussian range kernel, Nystrom algebra (nystrom.py:33-114)
# --------------------------------------------------------------------------
def gram(left: np.ndarray, right: np.ndarray, theta: float) -> np.ndarray:
    """K(i,j) = exp(-|l_i - r_j|^2 / (2 theta^2)), differenced (nystrom.py:43-54)."""
    L = np.asarray(left, np.float64)
    Rr = np.asarray(right, np.float64)
    inv = 1.0 / (2.0 * theta * theta)
    out = np.empty((L.shape[0], Rr.shape[0]))
    step = 16384
    for s in range(0, Rr.shape[0], step):
        d2 = ((L[:, None, :] - Rr[None, s:s + step, :]) ** 2).sum(axis=2)
        out[:, s:s + step] = np.exp(-d2 * inv)
    return out


def symmetrize(a: np.ndarray) -> np.ndarray:
    """SymMatrix construction (symeig.py:21-39)."""
    a = np.asarray(a, np.float64)
    return (a + a.T) / 2.0


def jacobi_eig(a: np.ndarray):
    """Cyclic Jacobi, descending eigenvalues, sign convention (symeig.py:58-125).

    Row-vector rotation bookkeeping as in the reference; returns
    (values (k,), vectors (k,k) with column j paired to values[j]).
    """
    A = symmetrize(a).copy()
    k = A.shape[0]
    V = np.eye(k)
    tol = JACOBI_OFFDIAG_TOL * np.abs(A).max()
    for _sweep in range(JACOBI_MAX_SWEEPS):
        off = np.abs(np.triu(A, 1)).max() if k > 1 else 0.0
        if off <= tol:
            break
        for p in range(k - 1):
            for q in range(p + 1, k):
                apq = A[p, q]
                if abs(apq) <= tol:
                    continue
                app, aqq = A[p, p], A[q, q]
                tau = (aqq - app) / (2.0 * apq)
                if tau >= 0.0:
                    t = 1.0 / (tau + math.sqrt(1.0 + tau * tau))
                else:
                    t = -1.0 / (-tau + math.sqrt(1.0 + tau * tau))
                c = 1.0 / math.sqrt(1.0 + t * t)
                s = t * c
                rp = A[p].copy()
                rq = A[q].copy()
                A[p] = c * rp - s * rq
                A[q] = s * rp + c * rq
                A[p, p] = app - t * apq
                A[q, q] = aqq + t * apq
                A[p, q] = A[q, p] = 0.0
                mask = np.ones(k, bool)
                mask[[p, q]] = False
                A[mask, p] = A[p, mask]
                A[mask, q] = A[q, mask]
                vp = V[p].copy()
                vq = V[q].copy()
                V[p] = c * vp - s * vq
                V[q] = s * vp + c * vq
    vals = np.diag(A).copy()
    order = np.argsort(-vals, kind="stable")
    vals = vals[order]
    vecs = V.T[:, order]
    lead = vecs[np.argmax(np.abs(vecs), axis=0), np.arange(k)]
    vecs = vecs * np.where(lead < 0.0, -1.0, 1.0)
    return vals, vecs


def retain(values: np.ndarray, vectors: np.ndarray, eps_drop: float):
    """Drop rule alpha_k > eps_drop * alpha_1 (nystrom.py:103-109)."""
    if values[0] <= 0.0:
        raise RuntimeError("landmark kernel has no positive eigenvalue")
    keep = values > eps_drop * values[0]
    if not keep.any():
        raise RuntimeError("every eigenpair fell below the drop threshold")
    return values[keep].copy(), vectors[:, keep].copy()


# --------------------------------------------------------------------------
# separable spatial kernels with replicate borders (spatial.py:72-109,194-209)
# --------------------------------------------------------------------------
def gaussian_taps(sigma: float, radius: int) -> np.ndarray:
    """Unnormalised exp(-t^2/(2 sigma^2)), t=-R..R (spatial.py:72-75)."""
    t = np.arange(-radius, radius + 1, dtype=np.float64)
    return np.exp(-(t * t) / (2.0 * sigma * sigma))


def _edge_pad_last(a: np.ndarray, r: int) -> np.ndarray:
    return np.concatenate([np.repeat(a[..., :1], r, -1), a,
                           np.repeat(a[..., -1:], r, -1)], axis=-1)


def box_last(a: np.ndarray, r: int) -> np.ndarray:
    """Sliding (2r+1)-sum via a cumulative sum (spatial.py:91-99)."""
    if r == 0:
        return a.copy()
    n = a.shape[-1]
    cs = np.cumsum(_edge_pad_last(a, r), axis=-1)
    cs = np.concatenate([np.zeros(cs.shape[:-1] + (1,)), cs], axis=-1)
    return cs[..., 2 * r + 1:] - cs[..., :n]


def fir_last(a: np.ndarray, taps: np.ndarray) -> np.ndarray:
    """Shifted-AXPY FIR along the last axis (spatial.py:102-109)."""
    r = (len(taps) - 1) // 2
    n = a.shape[-1]
    pad = _edge_pad_last(a, r)
    out = np.zeros_like(a, dtype=np.float64)
    for t, w in enumerate(taps):
        out += w * pad[..., t:t + n]
    return out


_VYV_POLES = (0.86430 + 1.45389j, 0.86430 - 1.45389j, 1.61433 + 0.83134j, 1.61433 - 0.83134j, 1.87504 + 0.0j)


def vyv_coeffs(sigma: float):
    """(gain, a1..a5) of the fifth-order recursive Gaussian whose cascade
    variance is sigma^2: bisection on the pole scale q, then the monic
    denominator polynomial (spatial.py:114-146)."""
    def variance(q):
        total = 0.0 + 0.0j
        for d in _VYV_POLES:
            z = d ** (1.0 / q)
            total += 2.0 * z / (z - 1.0) ** 2
        return total.real

    lo, hi = 1e-3, 1000.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if variance(mid) < sigma * sigma:
            lo = mid
        else:
            hi = mid
    q = 0.5 * (lo + hi)
    poly = np.array([1.0 + 0.0j])
    for d in _VYV_POLES:
        poly = np.convolve(poly, np.array([1.0, -1.0 / d ** (1.0 / q)]))
    a = poly.real
    return (float(a.sum()),) + tuple(float(v) for v in a[1:6])


def vyv_scan_last(a: np.ndarray, coeffs) -> np.ndarray:
    """Causal then anticausal recursion along the last axis, vectorised over
    the leading axes (spatial.py:149-176): forward state = the edge sample,
    backward state = the forward output's edge sample."""
    g, a1, a2, a3, a4, a5 = coeffs
    x = np.array(a, dtype=np.float64, copy=True)
    n = x.shape[-1]
    w1 = x[..., 0].copy()
    w2, w3, w4, w5 = w1.copy(), w1.copy(), w1.copy(), w1.copy()
    for i in range(n):
        cur = g * x[..., i] - (a1 * w1 + a2 * w2 + a3 * w3 + a4 * w4 + a5 * w5)
        x[..., i] = cur
        w5, w4, w3, w2, w1 = w4, w3, w2, w1, cur
    w1 = x[..., n - 1].copy()
    w2, w3, w4, w5 = w1.copy(), w1.copy(), w1.copy(), w1.copy()
    for i in range(n - 1, -1, -1):
        cur = g * x[..., i] - (a1 * w1 + a2 * w2 + a3 * w3 + a4 * w4 + a5 * w5)
        x[..., i] = cur
        w5, w4, w3, w2, w1 = w4, w3, w2, w1, cur
    return x


def fir_mass(sigma: float) -> float:
    """Sum of the truncated taps at radius ceil(3 sigma) (spatial.py:78-82)."""
    return float(gaussian_taps(sigma, math.ceil(3.0 * sigma)).sum())


def recursive_planes(planes: np.ndarray, sigma: float) -> np.ndarray:
    """Row recursion, column recursion, times fir_mass^2 (spatial.py:179-191)."""
    cf = vyv_coeffs(sigma)
    rows = vyv_scan_last(planes, cf)
    cols = vyv_scan_last(rows.transpose(0, 2, 1), cf).transpose(0, 2, 1)
    m = fir_mass(sigma)
    return np.ascontiguousarray(cols) * (m * m)


def spatial_conv(planes: np.ndarray, kind: str, sigma: float, radius: int) -> np.ndarray:
    """Row pass then column pass over a (P,H,W) stack (spatial.py:194-209)."""
    planes = np.asarray(planes, np.float64)
    if kind == "gaussian_recursive":
        if sigma < 1.0:  # spatial.py:206-208
            return spatial_conv(planes, "gaussian_fir", sigma, math.ceil(3.0 * sigma))
        return recursive_planes(planes, sigma)
    if kind == "box":
        rows = box_last(planes, radius)
        return np.ascontiguousarray(box_last(rows.transpose(0, 2, 1), radius).transpose(0, 2, 1))
    if kind == "gaussian_fir":
        w = gaussian_taps(sigma, radius)
        rows = fir_last(planes, w)
        return np.ascontiguousarray(fir_last(rows.transpose(0, 2, 1), w).transpose(0, 2, 1))
    raise ValueError(f"unknown spatial kernel kind {kind!r}")


# --------------------------------------------------------------------------
# guides (filters.py:141-187)
# --------------------------------------------------------------------------
def patch_stack(f: np.ndarray, r: int) -> np.ndarray:
    """(n*(2r+1)^2, H, W) raw patches, channel-major then dy then dx, edge
    replicated (filters.py:174-181)."""
    n, H, W = f.shape
    side = 2 * r + 1
    pad = np.pad(np.asarray(f, np.float64), ((0, 0), (r, r), (r, r)), mode="edge")
    out = np.empty((n * side * side, H, W))
    k = 0
    for c in range(n):
        for dy in range(side):
            for dx in range(side):
                out[k] = pad[c, dy:dy + H, dx:dx + W]
                k += 1
    return out


def pca_patch_guide(f: np.ndarray, r: int, pca_dim: int) -> np.ndarray:
    """Centred patches projected on the top pca_dim covariance eigenvectors
    (filters.py:161-187)."""
    P = patch_stack(f, r)
    dim, H, W = P.shape
    if not 1 <= pca_dim <= dim:
        raise ValueError(f"pca_dim must lie in [1, {dim}], got {pca_dim}")
    X = P.reshape(dim, -1).T
    Xc = X - X.mean(axis=0)
    _, vecs = jacobi_eig(Xc.T @ Xc / X.shape[0])
    coeffs = Xc @ vecs[:, :pca_dim]
    return np.ascontiguousarray(coeffs.T.reshape(pca_dim, H, W))


# --------------------------------------------------------------------------
# Algorithm 1 (filters.py:199-274)
# --------------------------------------------------------------------------
def effective_radius(kind: str, sigma: float, radius: int) -> int:
    """spatial.py:66-69."""
    if kind == "gaussian_recursive":
        return math.ceil(3.0 * sigma)
    return radius


def fast_filter_with_landmarks(f, p, centroids, theta, kind, sigma, radius,
                               eps_drop: float = DEFAULT_EPS_DROP, threads: int = 1):
    """Nystrom filter given landmarks (filters.py:214-257).

    threads > 1 splits the rank loop (filters.py:227) over a thread pool
    (NumPy releases the GIL in the array kernels); partial sums are combined
    in a fixed order.  Used only by bench.py's CPU baseline.

    Returns dict(output, retained_rank, min_denominator, guarded_pixels,
    eps_den, alphas).
    """
    f = np.asarray(f, np.float64)
    p = np.asarray(p, np.float64)
    n, H, W = f.shape
    C = np.asarray(centroids, np.float64)
    vals, vecs = jacobi_eig(gram(C, C, theta))
    alphas, Wk = retain(vals, vecs, eps_drop)
    B = gram(C, range_vectors(p), theta)             # (m0, m)
    V = (B.T @ Wk) / alphas[None, :]                 # (m, rank)
    rank = alphas.shape[0]

    def terms(k):
        d = V[:, k].reshape(H, W)
        planes = np.concatenate([d[None] * f, d[None]], axis=0)
        conv = spatial_conv(planes, kind, sigma, radius)
        return (alphas[k] * d) * conv[:n], (alphas[k] * d) * conv[n]

    def run(ks):
        z = np.zeros((n, H, W))
        e = np.zeros((H, W))
        lead = None
        for k in ks:
            tn, td = terms(k)
            z += tn
            e += td
            if k == 0:
                lead = (tn.copy(), td.copy())
        return z, e, lead

    if threads > 1 and rank > 1:
        from concurrent.futures import ThreadPoolExecutor
        parts = [list(range(i, rank, threads)) for i in range(min(threads, rank))]
        with ThreadPoolExecutor(len(parts)) as ex:
            results = list(ex.map(run, parts))
        zeta = np.zeros((n, H, W))
        eta = np.zeros((H, W))
        for z, e, lead in results:
            zeta += z
            eta += e
            if lead is not None:
                zl, el = lead
    else:
        zeta, eta, (zl, el) = run(range(rank))
    S = effective_radius(kind, sigma, radius)
    eps_den = DENOMINATOR_EPS_SCALE * (2 * S + 1) ** 2 * float(np.abs(alphas).max())
    aeta = np.abs(eta)
    mask = aeta < eps_den
    out = zeta / np.where(mask, 1.0, eta)
    guarded = int(mask.sum())
    if guarded:
        ok = np.abs(el) >= eps_den
        fb = np.where(ok, zl / np.where(ok, el, 1.0), f)
        out = np.where(mask, fb, out)
    return dict(output=out, retained_rank=int(rank),
                min_denominator=float(aeta.min()), guarded_pixels=guarded,
                eps_den=eps_den, alphas=alphas, eta=eta)


def fast_filter(f, p, theta, kind, sigma, radius, m0, seed=0, max_iter=50,
                eps_drop: float = DEFAULT_EPS_DROP, threads: int = 1):
    """Full Algorithm 1: k-means landmarks then the filter (filters.py:199-274)."""
    t0 = time.perf_counter()
    C, _lab, qe, errors = kmeans(range_vectors(p), m0, seed=seed, max_iter=max_iter)
    t1 = time.perf_counter()
    res = fast_filter_with_landmarks(f, p, C, theta, kind, sigma, radius, eps_drop, threads)
    t2 = time.perf_counter()
    res.update(centroids=C, quant_error=qe, errors=errors,
               timings={"clustering": t1 - t0, "filter": t2 - t1, "total": t2 - t0})
    return res


def brute_force_filter(f, p, theta, kind, sigma, radius):
    """Direct Eq. (1) over the (2S+1)^2 window (filters.py:116-138)."""
    f = np.asarray(f, np.float64)
    p = np.asarray(p, np.float64)
    S = effective_radius(kind, sigma, radius)
    if kind == "box":
        w2 = np.ones((2 * S + 1, 2 * S + 1))
    else:
        w1 = gaussian_taps(sigma, S)
        w2 = np.outer(w1, w1)
    _, H, W = f.shape
    inv = 1.0 / (2.0 * theta * theta)
    pf = np.pad(f, ((0, 0), (S, S), (S, S)), mode="edge")
    pp = np.pad(p, ((0, 0), (S, S), (S, S)), mode="edge")
    num = np.zeros_like(f)
    den = np.zeros((H, W))
    for iy in range(2 * S + 1):
        for ix in range(2 * S + 1):
            dd = pp[:, iy:iy + H, ix:ix + W] - p
            kv = np.exp(-(dd * dd).sum(axis=0) * inv) * w2[iy, ix]
            num += kv * pf[:, iy:iy + H, ix:ix + W]
            den += kv
    return num / den


# --------------------------------------------------------------------------
# quality metrics (metrics.py:37-122)
# --------------------------------------------------------------------------
PSNR_CAP = 99.0


def mse(a, b) -> float:
    """metrics.py:37-40."""
    d = np.asarray(a, np.float64) - np.asarray(b, np.float64)
    return float(np.mean(d * d))


def psnr(a, b, R: float, per_band: bool = False) -> float:
    """metrics.py:43-64 (99 dB cap)."""
    def from_mse(e):
        return PSNR_CAP if e <= 0.0 else float(min(PSNR_CAP, 10.0 * np.log10(R * R / e)))

    if per_band:
        return float(np.mean([from_mse(mse(a[c], b[c])) for c in range(len(a))]))
    return from_mse(mse(a, b))


def ssim(a, b, R: float) -> float:
    """Single-scale SSIM, 11x11 Gaussian window sigma 1.5, valid positions,
    whole-plane statistics below the window (metrics.py:67-115)."""
    c1, c2 = (0.01 * R) ** 2, (0.03 * R) ** 2
    t = np.arange(-5, 6, dtype=np.float64)
    w1 = np.exp(-(t * t) / (2.0 * 1.5 * 1.5))
    w = np.outer(w1, w1)
    w /= w.sum()
    vals = []
    for x, y in zip(np.asarray(a, np.float64), np.asarray(b, np.float64)):
        H, W = x.shape
        if H < 11 or W < 11:
            mx, my = x.mean(), y.mean()
            cov = ((x - mx) * (y - my)).mean()
            vals.append(((2 * mx * my + c1) * (2 * cov + c2)) / ((mx * mx + my * my + c1) * (x.var() + y.var() + c2)))
            continue
        Hv, Wv = H - 10, W - 10
        acc = {k: np.zeros((Hv, Wv)) for k in ("mx", "my", "xx", "yy", "xy")}
        for dy in range(11):
            for dx in range(11):
                xs, ys, wv = x[dy:dy + Hv, dx:dx + Wv], y[dy:dy + Hv, dx:dx + Wv], w[dy, dx]
                acc["mx"] += wv * xs
                acc["my"] += wv * ys
                acc["xx"] += wv * xs * xs
                acc["yy"] += wv * ys * ys
                acc["xy"] += wv * xs * ys
        mx, my = acc["mx"], acc["my"]
        vx, vy, cv = acc["xx"] - mx * mx, acc["yy"] - my * my, acc["xy"] - mx * my
        vals.append(float((((2 * mx * my + c1) * (2 * cv + c2)) / ((mx * mx + my * my + c1) * (vx + vy + c2))).mean()))
    return float(np.mean(vals))
