"""PCA patch guide on the B200 (reference filters.py:161-187).

The patch matrix X (m x n(2r+1)^2) is never materialised: ``nys_patch_moments``
gathers patches from the image to form the mean and the centred Gram matrix
in FP64 (csrc/nys_pca.cu), the small dim x dim covariance is diagonalised on
the host (the m0 x m0 landmark eig's tridiagonal QL solver, with the
reference's ordering and sign convention: descending eigenvalues, the
largest-|.| entry of every eigenvector non-negative, symeig.py:115-125), and
``nys_pca_project`` writes the planar (pca_dim, H, W) guide.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native
from ._device import ptr, stream_ptr, to_device_f32
from .image import Image


def _sign_convention(vecs: np.ndarray) -> np.ndarray:
    """Flip each column so its largest-|.| entry (earliest on ties) is >= 0."""
    idx = np.argmax(np.abs(vecs), axis=0)
    sgn = np.where(vecs[idx, np.arange(vecs.shape[1])] < 0, -1.0, 1.0)
    return vecs * sgn[None, :]


def patch_covariance(f_dev: torch.Tensor, r: int):
    """(mean (dim,), covariance (dim, dim)) of the raw patches, FP64 host arrays."""
    n, H, W = f_dev.shape
    dim = n * (2 * r + 1) ** 2
    lib = _native.lib()
    wsb = int(lib.nys_patch_moments_workspace_bytes(n, H, W, r))
    if wsb == 0:
        raise NotImplementedError(f"patch dimension {dim} > 1024 is not supported on the B200 path")
    nt = (dim + 3) // 4
    ntiles = nt * (nt + 1) // 2
    ws = torch.empty(wsb, dtype=torch.uint8, device=f_dev.device)
    res = torch.empty(dim + ntiles * 16, dtype=torch.float64, device=f_dev.device)
    _native.check(lib.nys_patch_moments(ptr(f_dev), H * W, n, H, W, r, ptr(res), ptr(res) + 8 * dim, ptr(ws), wsb,
                                        stream_ptr()), "nys_patch_moments")
    h = res.cpu().numpy()
    mean = h[:dim].copy()
    tiles = h[dim:].reshape(ntiles, 4, 4)
    G = np.zeros((4 * nt, 4 * nt))
    t = 0
    for ti in range(nt):
        for tj in range(ti, nt):
            G[4 * ti:4 * ti + 4, 4 * tj:4 * tj + 4] = tiles[t]
            G[4 * tj:4 * tj + 4, 4 * ti:4 * ti + 4] = tiles[t].T
            t += 1
    cov = G[:dim, :dim] / float(H * W)
    return mean, 0.5 * (cov + cov.T)


def pca_basis(cov: np.ndarray):
    """Descending eigenpairs of the covariance with the reference's sign
    convention (symeig.py:107-125)."""
    k = cov.shape[0]
    a = np.ascontiguousarray(cov, dtype=np.float64)
    vals = np.zeros(k)
    vecs = np.zeros((k, k))
    _native.check(_native.lib().nys_sym_eig(a.ctypes.data, k, vals.ctypes.data, vecs.ctypes.data), "nys_sym_eig")
    order = np.argsort(-vals, kind="stable")
    return vals[order], _sign_convention(vecs[:, order])


def pca_patch_guide_device(f_dev: torch.Tensor, r: int, pca_dim: int) -> torch.Tensor:
    """Planar float32 (pca_dim, H, W) guide on the device."""
    n, H, W = f_dev.shape
    mean, cov = patch_covariance(f_dev, r)
    _, vecs = pca_basis(cov)
    dim = mean.shape[0]
    mu = torch.from_numpy(mean.astype(np.float32)).to(f_dev.device)
    basis = torch.from_numpy(np.ascontiguousarray(vecs[:, :pca_dim], dtype=np.float32)).to(f_dev.device)
    out = torch.empty((pca_dim, H, W), dtype=torch.float32, device=f_dev.device)
    _native.check(_native.lib().nys_pca_project(ptr(f_dev), H * W, n, H, W, r, ptr(mu), ptr(basis), pca_dim,
                                                ptr(out), H * W, stream_ptr()), "nys_pca_project")
    assert dim == n * (2 * r + 1) ** 2
    return out


def pca_patch_guide(f: Image, patch_radius: int, pca_dim: int) -> Image:
    """Truncated PCA guide as an Image: a device tensor when ``f`` is on the
    device, else the reference's float64 ndarray."""
    g = pca_patch_guide_device(to_device_f32(f.data), int(patch_radius), int(pca_dim))
    data = g if f.on_device else g.double().cpu().numpy()
    return Image(data=data, range_max=f.range_max)
