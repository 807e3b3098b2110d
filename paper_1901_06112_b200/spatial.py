"""Spatial kernel description (mirror of reference ``spatial.py:32-75``).

The convolution itself runs inside the K2/K3 CUDA kernels; this module only
carries the parameters and the tap weights.
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
