"""Image quality metrics on the B200 (mirror of reference ``metrics.py``).

MSE, PSNR (capped at 99 dB, optionally per band) and single-scale SSIM
(11x11 Gaussian window, sigma 1.5, C1 = (0.01 R)^2, C2 = (0.03 R)^2, valid
positions only, whole-plane statistics below the window size), computed by
``nys_quality_planes`` (csrc/nys_metrics.cu) in FP64 from float32 or float64
planes.  Same names, arguments and errors as metrics.py:26-122.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from ._device import ptr, require_cuda, stream_ptr
from .image import Image

PSNR_CAP = 99.0
SSIM_WINDOW = 11
SSIM_SIGMA = 1.5
SSIM_K1 = 0.01
SSIM_K2 = 0.03


@dataclass(frozen=True)
class QualityScore:
    mse: float
    psnr: float
    ssim: float


def _check(a: Image, b: Image) -> None:  # metrics.py:32-34
    if tuple(a.data.shape) != tuple(b.data.shape):
        raise ValueError(f"image shapes differ: {tuple(a.data.shape)} vs {tuple(b.data.shape)}")


def _planes(img: Image, dtype=None) -> torch.Tensor:
    dev = require_cuda()
    d = img.data
    if isinstance(d, torch.Tensor):
        t = d if d.dtype in (torch.float32, torch.float64) else d.to(torch.float64)
        return t.to(dev, dtype=dtype or t.dtype).contiguous()
    return torch.from_numpy(np.array(d, dtype=np.float64, copy=True)).to(dev, dtype=dtype or torch.float64)


def _per_plane(a: Image, b: Image, want_ssim: bool):
    """(Σ (a-b)^2 per plane, mean SSIM per plane or None) as host float64 arrays."""
    _check(a, b)
    ta = _planes(a)
    tb = _planes(b, dtype=ta.dtype)
    n, H, W = ta.shape
    lib = _native.lib()
    wsb = int(lib.nys_quality_workspace_bytes(n))
    ws = torch.empty(wsb, dtype=torch.uint8, device=ta.device)
    res = torch.empty(2 * n, dtype=torch.float64, device=ta.device)
    _native.check(lib.nys_quality_planes(ptr(ta), H * W, ptr(tb), H * W, ta.element_size(), n, H, W,
                                         float(a.range_max), ptr(res), ptr(res) + 8 * n if want_ssim else None,
                                         ptr(ws), wsb, stream_ptr()), "nys_quality_planes")
    h = res.cpu().numpy()
    return h[:n], (h[n:] if want_ssim else None), H * W


def _psnr_from_mse(err: float, R: float) -> float:  # metrics.py:61-64
    if err <= 0.0:
        return PSNR_CAP
    return float(min(PSNR_CAP, 10.0 * math.log10(R * R / err)))


def mse(a: Image, b: Image) -> float:
    sq, _, px = _per_plane(a, b, False)
    return float(sq.sum() / (sq.size * px))


def psnr(a: Image, b: Image, per_band: bool = False) -> float:
    """10 log10(R^2 / MSE) with R = a.range_max, capped at 99 dB; per_band
    averages the per-band PSNRs (metrics.py:43-58)."""
    sq, _, px = _per_plane(a, b, False)
    R = a.range_max
    if per_band:
        return float(np.mean([_psnr_from_mse(float(s / px), R) for s in sq]))
    return _psnr_from_mse(float(sq.sum() / (sq.size * px)), R)


def ssim(a: Image, b: Image) -> float:
    """Mean single-scale SSIM over channels/bands (metrics.py:111-115)."""
    _, s, _ = _per_plane(a, b, True)
    return float(np.mean(s))


def quality(a: Image, b: Image, per_band: bool = False) -> QualityScore:
    """All three in one device pass (metrics.py:118-122)."""
    sq, s, px = _per_plane(a, b, True)
    R = a.range_max
    m = float(sq.sum() / (sq.size * px))
    p = float(np.mean([_psnr_from_mse(float(v / px), R) for v in sq])) if per_band else _psnr_from_mse(m, R)
    return QualityScore(mse=m, psnr=p, ssim=float(np.mean(s)))
