"""Nystrom algebra (mirror of reference ``nystrom.py:29-114``).

On the B200 path only the m0 x m0 landmark kernel A, its eigensystem, the drop
rule and the mixing matrix M = W_r diag(1/alpha_r) W_r^T are formed (host,
FP64).  The m0 x m cross kernel B and the extrapolated eigenvectors
V = B^T W / alpha are never materialised: the K2/K3 kernels recompute
b(x) = kappa(C, p(x)) per pixel and apply M there.  ``build_B``/``fit`` are
kept as host-side API mirrors for diagnostics at small m (the reference's
``fit`` is likewise a test/diagnostic boundary).
"""

from __future__ import annotations

from dataclasses import dataclass

import ctypes as C

import numpy as np

from . import _native
from .image import RangeList
from .landmarks import LandmarkSet
from .symeig import SymMatrix, jacobi_eig

DEFAULT_EPS_DROP = 1e-8
KERNEL_ERROR_MAX_POINTS = 5000


class DegenerateKernelError(RuntimeError):
    """All eigenpairs of the landmark kernel were dropped (nystrom.py:29-30)."""


@dataclass(frozen=True)
class RangeKernel:
    """Gaussian similarity exp(-|s-t|^2 / (2 theta^2)) (nystrom.py:33-54)."""

    theta: float

    def __post_init__(self) -> None:
        if not self.theta > 0:
            raise ValueError("theta must be positive")

    def gram(self, left: np.ndarray, right: np.ndarray) -> np.ndarray:
        left = np.asarray(left, dtype=np.float64)
        right = np.asarray(right, dtype=np.float64)
        inv = 1.0 / (2.0 * self.theta * self.theta)
        out = np.empty((left.shape[0], right.shape[0]))
        step = 32768
        for s in range(0, right.shape[0], step):
            d2 = ((left[:, None, :] - right[None, s:s + step, :]) ** 2).sum(axis=2)
            np.exp(-d2 * inv, out=out[:, s:s + step])
        return out


@dataclass(frozen=True)
class NystromModel:
    landmarks: LandmarkSet
    alphas: np.ndarray
    extrapolated: np.ndarray
    retained_rank: int


def build_A(landmarks: np.ndarray, kernel: RangeKernel) -> SymMatrix:
    """Landmark kernel, unit diagonal (nystrom.py:67-69)."""
    return SymMatrix(kernel.gram(landmarks, landmarks))


def build_B(landmarks: np.ndarray, range_list: RangeList, kernel: RangeKernel) -> np.ndarray:
    """Cross kernel landmarks x guides (nystrom.py:72-79); diagnostic only."""
    landmarks = np.asarray(landmarks, dtype=np.float64)
    if landmarks.shape[1] != range_list.dim:
        raise ValueError(f"landmark dim {landmarks.shape[1]} != range-list dim {range_list.dim}")
    return kernel.gram(landmarks, range_list.vectors)


def _retain(values: np.ndarray, vectors: np.ndarray, eps_drop: float):
    """Keep alpha_k > eps_drop * alpha_1 (nystrom.py:103-109)."""
    if values[0] <= 0.0:
        raise DegenerateKernelError("landmark kernel has no positive eigenvalue")
    keep = values > eps_drop * values[0]
    if not keep.any():
        raise DegenerateKernelError("every eigenpair fell below the drop threshold")
    return values[keep].copy(), vectors[:, keep].copy()


def extrapolate(B: np.ndarray, alphas: np.ndarray, vectors: np.ndarray) -> np.ndarray:
    """v_k = B^T w_k / alpha_k (nystrom.py:112-114); diagnostic only."""
    return (B.T @ vectors) / alphas[None, :]


def fit(range_list: RangeList, landmarks: LandmarkSet, kernel: RangeKernel,
        eps_drop: float = DEFAULT_EPS_DROP) -> NystromModel:
    if not 0.0 <= eps_drop < 1.0:
        raise ValueError("eps_drop must lie in [0, 1)")
    eig = jacobi_eig(build_A(landmarks.centroids, kernel))
    alphas, vectors = _retain(eig.values, eig.vectors, eps_drop)
    B = build_B(landmarks.centroids, range_list, kernel)
    return NystromModel(landmarks=landmarks, alphas=alphas, extrapolated=extrapolate(B, alphas, vectors),
                        retained_rank=alphas.shape[0])


def kernel_error(model: NystromModel, range_list: RangeList, kernel: RangeKernel,
                 max_points: int = KERNEL_ERROR_MAX_POINTS) -> float:
    """|K - K_hat|_F at test scale (nystrom.py:117-138)."""
    m = range_list.m
    if m > max_points:
        raise ValueError(f"kernel_error materializes an m x m matrix; m={m} exceeds the "
                         f"{max_points}-point diagnostic guard")
    V = model.extrapolated
    K = kernel.gram(range_list.vectors, range_list.vectors) - (V * model.alphas[None, :]) @ V.T
    return float(np.sqrt((K * K).sum()))


@dataclass(frozen=True)
class MixingPlan:
    """Host FP64 products the kernels need (filters.py:214-242)."""

    alphas: np.ndarray   # retained eigenvalues, descending
    M: np.ndarray        # (m0, m0) = W_r diag(1/alpha_r) W_r^T
    u0: np.ndarray       # leading eigenvector w_1
    alpha0: float
    eps_den: float       # 1e-12 (2S+1)^2 max|alpha|
    phi_form: bool = False  # M holds P = diag(alpha_r^-1/2) W_r^T (padded to m0 rows), see nys_filter_desc
    rank: int = -1          # retained eigenpairs (lite plans carry only alpha_1 in `alphas`)
    M_is_cholesky: bool = False  # M holds the Cholesky factor of A; the device forms A^{-1}

    def __post_init__(self):
        if self.rank < 0:
            object.__setattr__(self, "rank", int(self.alphas.shape[0]))


# Above this cond(A) over the retained eigenpairs the FP32 y-form (y = M b with
# M = A^+) loses ~eps * cond of accuracy (1.9e-3 at 6e6 on a 1-D guide,
# tools/dbg_rec.py); the phi-form's FP32 error does not grow with cond(A).
PHI_FORM_COND = 3.0e4


def mixing_plan(centroids: np.ndarray, theta: float, eps_drop: float, S: int, lite: bool = False,
                device_inverse: bool = False) -> MixingPlan:
    """Host FP64 products the kernels consume, in one native call
    (``nys_mixing_plan``: Gram matrix nystrom.py:67-69, eigenvalues + drop
    rule nystrom.py:97-109, M and the lead eigenvector).

    The filter only sees M = sum_k w_k w_k^T / alpha_k (invariant to the
    eigenvector basis and signs) and the lead pair (w_1 enters the guard
    quadratically).  With no eigenpair dropped M = A^{-1}, which the native
    code forms by Cholesky next to a values-only QL and an inverse iteration
    for w_1 (~0.15 ms at m0 = 64 instead of ~0.8 ms for the full eigensystem
    plus numpy products); otherwise it falls back to the full Householder + QL
    eigensystem.  ``jacobi_eig`` remains the bit-faithful API mirror."""
    C_ = np.ascontiguousarray(np.asarray(centroids, np.float64))
    k, rho = C_.shape
    alphas = np.empty(k)
    M = np.empty((k, k))
    u0 = np.empty(k)
    rank = C.c_int(0)
    if lite:
        # hot path: alpha_1 + two Sturm counts (nothing dropped, cond <= PHI_FORM_COND), else the full plan
        chol = bool(device_inverse and k <= 64)  # M = A^{-1} formed on the device from the Cholesky factor
        rc = _native.lib().nys_mixing_plan_lite(C_.ctypes.data, k, rho, float(theta), float(eps_drop), PHI_FORM_COND,
                                                int(chol), alphas.ctypes.data, C.byref(rank), M.ctypes.data,
                                                u0.ctypes.data)
        if rc == _native.NYS_OK:
            a1 = float(alphas[0])
            return MixingPlan(alphas=np.array([a1]), M=M, u0=u0, alpha0=a1,
                              eps_den=1e-12 * (2 * S + 1) ** 2 * a1, rank=k, M_is_cholesky=chol)
        if rc == _native.NYS_EDEGENERATE:
            raise DegenerateKernelError("landmark kernel has no positive eigenvalue")
        if rc != _native.NYS_EUNSUPPORTED:
            _native.check(rc, "nys_mixing_plan_lite")
    rc = _native.lib().nys_mixing_plan(C_.ctypes.data, k, rho, float(theta), float(eps_drop), alphas.ctypes.data,
                                       C.byref(rank), M.ctypes.data, u0.ctypes.data)
    if rc == _native.NYS_EDEGENERATE:
        raise DegenerateKernelError("landmark kernel has no positive eigenvalue")
    _native.check(rc, "nys_mixing_plan")
    alphas = alphas[:rank.value].copy()
    eps_den = 1e-12 * (2 * S + 1) ** 2 * float(np.abs(alphas).max())
    if alphas[0] / alphas[-1] > PHI_FORM_COND:
        # ill-conditioned landmark kernel: phi-form (same quantity, filters.py:227-238)
        A = np.empty((k, k))
        inv = 1.0 / (2.0 * theta * theta)
        d2 = ((C_[:, None, :] - C_[None, :, :]) ** 2).sum(-1)
        A[:] = np.exp(-d2 * inv)
        vals = np.empty(k)
        vecs = np.empty((k, k))
        _native.check(_native.lib().nys_sym_eig(np.ascontiguousarray(A).ctypes.data, k, vals.ctypes.data,
                                                vecs.ctypes.data), "nys_sym_eig")
        order = np.argsort(-vals, kind="stable")
        vals, vecs = vals[order], vecs[:, order]
        r = alphas.shape[0]
        P = np.zeros((k, k))
        P[:r] = (vecs[:, :r] / np.sqrt(vals[:r])[None, :]).T
        return MixingPlan(alphas=alphas, M=P, u0=vecs[:, 0].copy(), alpha0=float(alphas[0]), eps_den=eps_den,
                          phi_form=True)
    return MixingPlan(alphas=alphas, M=M, u0=u0, alpha0=float(alphas[0]), eps_den=eps_den)
