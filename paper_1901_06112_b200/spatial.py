"""Spatial kernels (mirror of reference ``spatial.py``).

Inside the filter the convolutions run fused into the K2/K3 (box / FIR) and
R1-R4 (recursive) CUDA kernels.  The reference's stand-alone helpers
(``apply_planes``, ``box_filter``, ``gaussian_fir``, ``gaussian_recursive``,
spatial.py:194-234) run on the device too (``nys_spatial_planes``, FP64).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

BOX = "box"
GAUSSIAN_FIR = "gaussian_fir"
GAUSSIAN_RECURSIVE = "gaussian_recursive"


@dataclass(frozen=True)
class SpatialKernel:
    kind: str
    sigma: float = 0.0
    radius: int = 0

    def __post_init__(self) -> None:  # spatial.py:38-49
        if self.kind == BOX:
            if self.radius < 0:
                raise ValueError("box radius must be >= 0")
        elif self.kind == GAUSSIAN_FIR:
            if self.sigma <= 0 or self.radius < 1:
                raise ValueError("gaussian FIR needs sigma > 0 and radius >= 1")
        elif self.kind == GAUSSIAN_RECURSIVE:
            if self.sigma <= 0:
                raise ValueError("recursive gaussian needs sigma > 0")
        else:
            raise ValueError(f"unknown spatial kernel kind {self.kind!r}")

    @classmethod
    def box(cls, radius: int) -> "SpatialKernel":
        return cls(kind=BOX, radius=int(radius))

    @classmethod
    def gaussian(cls, sigma: float, radius: int | None = None) -> "SpatialKernel":
        if radius is None:
            radius = math.ceil(3.0 * sigma)
        return cls(kind=GAUSSIAN_FIR, sigma=float(sigma), radius=int(radius))

    @classmethod
    def recursive(cls, sigma: float) -> "SpatialKernel":
        return cls(kind=GAUSSIAN_RECURSIVE, sigma=float(sigma))

    def effective_radius(self) -> int:
        """Window radius: explicit for box/FIR, ceil(3*sigma) for recursive."""
        if self.kind == GAUSSIAN_RECURSIVE:
            return math.ceil(3.0 * self.sigma)
        return self.radius


def gaussian_weights(sigma: float, radius: int) -> np.ndarray:
    """Unnormalised exp(-t^2 / (2 sigma^2)), t = -radius..radius (spatial.py:72-75)."""
    t = np.arange(-radius, radius + 1, dtype=np.float64)
    return np.exp(-(t * t) / (2.0 * sigma * sigma))


def fir_mass(sigma: float, radius: int | None = None) -> float:
    if radius is None:
        radius = math.ceil(3.0 * sigma)
    return float(gaussian_weights(sigma, radius).sum())


def apply_planes(planes, kernel: SpatialKernel):
    """Filter a (planes, height, width) stack with ``kernel``, batched
    (spatial.py:194-213): row pass then column pass, edge replicate, FP64 on
    the device.  NumPy in -> float64 NumPy out; a torch tensor stays on its
    device (as float64)."""
    import torch

    from . import _native
    from ._device import ptr, require_cuda, stream_ptr

    dev = require_cuda()
    is_t = isinstance(planes, torch.Tensor)
    t = planes if is_t else torch.from_numpy(np.array(planes, dtype=np.float64, copy=True))
    if t.dim() != 3:
        raise ValueError("expected a (planes, height, width) array")
    t = t.to(dev, dtype=torch.float64).contiguous()
    P, H, W = (int(v) for v in t.shape)
    out = torch.empty_like(t)
    kind = {BOX: _native.NYS_SPATIAL_BOX, GAUSSIAN_FIR: _native.NYS_SPATIAL_GAUSSIAN_FIR,
            GAUSSIAN_RECURSIVE: _native.NYS_SPATIAL_GAUSSIAN_RECURSIVE}[kernel.kind]
    scratch = torch.empty_like(t) if (kernel.kind != GAUSSIAN_RECURSIVE or kernel.sigma < 1.0) else None
    _native.check(_native.lib().nys_spatial_planes(ptr(t), ptr(out), P, H, W, kind, float(kernel.sigma),
                                                   int(kernel.radius), ptr(scratch), stream_ptr()),
                  "nys_spatial_planes")
    if is_t:
        return out
    return out.cpu().numpy()


def box_filter(plane, S: int):
    """Sliding-sum box filter: sum of the (2S+1)^2 window, replicate borders (spatial.py:216-219)."""
    return apply_planes(np.asarray(plane, dtype=np.float64)[np.newaxis], SpatialKernel.box(S))[0]


def gaussian_fir(plane, sigma: float, S: int):
    """Separable truncated-Gaussian convolution (spatial.py:222-226)."""
    return apply_planes(np.asarray(plane, dtype=np.float64)[np.newaxis], SpatialKernel.gaussian(sigma, S))[0]


def gaussian_recursive(plane, sigma: float):
    """Recursive Gaussian, O(1) per pixel in sigma; the FIR path below sigma 1 (spatial.py:229-234)."""
    return apply_planes(np.asarray(plane, dtype=np.float64)[np.newaxis], SpatialKernel.recursive(sigma))[0]
