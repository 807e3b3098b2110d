"""Seeded synthetic inputs standing in for the paper's images.

BASELINE.json's five configs are all synthetic: random-polygon piecewise
constant scenes (colour or hyperspectral) plus Gaussian noise, clipped to
[0, 1], planar (C, H, W) float32.  The same arrays feed the GPU path and the
CPU oracle / reference.  Draw order from ``np.random.default_rng(seed)`` is
fixed: polygons, then region colours / spectra, then (NLM only) shading,
then noise.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def polygon_labels(rng: np.random.Generator, H: int, W: int, regions: int) -> np.ndarray:
    """Label map of ``regions`` random star-shaped polygons painted in order on
    background label 0 (later polygons overwrite earlier ones)."""
    from PIL import Image as _PIL, ImageDraw

    canvas = _PIL.new("I", (W, H), 0)
    draw = ImageDraw.Draw(canvas)
    short = min(H, W)
    for r in range(regions):
        cx = rng.uniform(0, W)
        cy = rng.uniform(0, H)
        k = int(rng.integers(3, 9))
        ang = np.sort(rng.uniform(0.0, 2.0 * np.pi, k))
        rad = rng.uniform(0.05, 0.35) * short * rng.uniform(0.5, 1.0, k)
        pts = [(float(cx + a * np.cos(t)), float(cy + a * np.sin(t))) for t, a in zip(ang, rad)]
        draw.polygon(pts, fill=r + 1)
    return np.asarray(canvas, dtype=np.int32)


def _noise(rng, shape, sigma):
    return (sigma * rng.standard_normal(shape, dtype=np.float32)).astype(np.float32)


def color_scene(H: int, W: int, regions: int, noise: float, seed: int = 0,
                lo: float = 0.0, hi: float = 1.0, shading: float = 0.0) -> np.ndarray:
    """(3, H, W) float32 polygon scene, uniform RGB per region in [lo, hi],
    optional low-frequency sinusoidal shading per channel, Gaussian noise."""
    rng = np.random.default_rng(seed)
    lab = polygon_labels(rng, H, W, regions)
    colours = rng.uniform(lo, hi, (regions + 1, 3)).astype(np.float32)
    img = np.ascontiguousarray(np.moveaxis(colours[lab], 2, 0))
    if shading:
        yy = (np.arange(H, dtype=np.float32) / H)[:, None]
        xx = (np.arange(W, dtype=np.float32) / W)[None, :]
        for c in range(3):
            fx, fy = rng.uniform(0.5, 2.0, 2)
            ph = rng.uniform(0.0, 2.0 * np.pi)
            img[c] += np.float32(shading) * np.sin(
                np.float32(2 * np.pi) * (np.float32(fx) * xx + np.float32(fy) * yy) + np.float32(ph))
    img += _noise(rng, img.shape, noise)
    return np.clip(img, 0.0, 1.0).astype(np.float32)


def spectral_scene(H: int, W: int, bands: int, regions: int, noise: float,
                   seed: int = 0) -> np.ndarray:
    """(bands, H, W) float32 cube: each region gets a smooth spectrum
    sum_{g<3} a_g exp(-(b - mu_g)^2 / (2 s_g^2)), a~U(.1,.5), mu~U(0,bands),
    s~U(2, bands/2); plus Gaussian noise; clipped to [0, 1]."""
    rng = np.random.default_rng(seed)
    lab = polygon_labels(rng, H, W, regions)
    b = np.arange(bands, dtype=np.float64)
    spectra = np.zeros((regions + 1, bands))
    for r in range(regions + 1):
        for _ in range(3):
            a = rng.uniform(0.1, 0.5)
            mu = rng.uniform(0.0, bands)
            s = rng.uniform(2.0, bands / 2.0)
            spectra[r] += a * np.exp(-(b - mu) ** 2 / (2.0 * s * s))
    spectra = spectra.astype(np.float32)
    cube = np.empty((bands, H, W), np.float32)
    for c in range(bands):
        cube[c] = spectra[:, c][lab]
    for c in range(bands):                      # band by band keeps peak RAM low
        cube[c] += _noise(rng, (H, W), noise)
        np.clip(cube[c], 0.0, 1.0, out=cube[c])
    return cube


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json config: inputs recipe plus filter parameters."""

    name: str
    H: int
    W: int
    channels: int
    regions: int
    noise: float
    theta: float
    spatial: str          # "gaussian_fir" | "box"
    sigma: float
    radius: int
    m0: int
    max_iter: int
    mode: str = "bilateral"   # "bilateral" | "nlm"
    patch_radius: int = 0
    kind: str = "color"       # "color" | "shaded" | "spectral"

    def image(self, seed: int = 0, H: int | None = None, W: int | None = None) -> np.ndarray:
        H = self.H if H is None else H
        W = self.W if W is None else W
        if self.kind == "spectral":
            return spectral_scene(H, W, self.channels, self.regions, self.noise, seed)
        if self.kind == "shaded":
            return color_scene(H, W, self.regions, self.noise, seed, lo=0.1, hi=0.9, shading=0.1)
        return color_scene(H, W, self.regions, self.noise, seed)

    @property
    def pixels(self) -> int:
        return self.H * self.W


CONFIGS = {
    1: Workload("cfg1_blf_rgb_512", 512, 512, 3, 40, 0.04, 0.15, "gaussian_fir", 3.0, 9, 32, 10),
    2: Workload("cfg2_blf_rgb_1080p", 1080, 1920, 3, 200, 0.05, 0.1, "gaussian_fir", 5.0, 15, 64, 15),
    3: Workload("cfg3_nlm_rgb_1024", 1024, 1024, 3, 64, 0.08, 0.3 * np.sqrt(27.0) * 0.08, "box",
                0.0, 10, 64, 15, mode="nlm", patch_radius=1, kind="shaded"),
    4: Workload("cfg4_blf_hyper31_1024", 1024, 1024, 31, 64, 0.03, 0.25, "gaussian_fir", 4.0, 12,
                48, 15, kind="spectral"),
    5: Workload("cfg5_blf_hyper16_8192", 8192, 8192, 16, 256, 0.03, 0.2, "gaussian_fir", 6.0, 18,
                64, 15, kind="spectral"),
}
