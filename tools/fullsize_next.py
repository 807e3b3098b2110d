"""Full-size parity of the §8(f) rows against the FP64 oracle, on the GPU box's
host (the oracle is test infrastructure; run it where the GPU is):

    python tools/fullsize_next.py > profiles/r1_fullsize_next.jsonl

  f2  recursive Gaussian on the full cfg-2 image (sigma 5), stage 1 (oracle landmarks)
  f1  brute_force_filter on the full cfg-1 image and on a 256-row cfg-2 band
  f3  PCA patch guide r=3 -> 25 on a 384x384 NLM scene; NLM-PCA filter stage 1 on it
  f4  mse / psnr / ssim on the full cfg-2 image vs its filtered output
One JSON line per case.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import nys_oracle as O  # noqa: E402
from paper_1901_06112_b200 import (  # noqa: E402
    FilterParams,
    Image,
    SpatialKernel,
    brute_force_filter,
    filter_with_landmarks,
    mse,
    pca_patch_guide,
    psnr,
    ssim,
)
from paper_1901_06112_b200.synthetic import CONFIGS, color_scene  # noqa: E402


def emit(d):
    print(json.dumps(d), flush=True)


def main():
    dev = torch.device("cuda", 0)
    # f2: recursive Gaussian, full cfg-2 image
    wl = CONFIGS[2]
    f32 = wl.image(seed=0)
    f64 = f32.astype(np.float64)
    t0 = time.time()
    C, _, _, _ = O.kmeans(O.range_vectors(f64), wl.m0, 0, wl.max_iter)
    ref = O.fast_filter_with_landmarks(f64, f64, C, wl.theta, "gaussian_recursive", 5.0, 0, threads=16)
    t1 = time.time()
    f = Image(data=torch.from_numpy(f32).to(dev), range_max=1.0)
    rep = filter_with_landmarks(f, f, C, FilterParams(spatial=SpatialKernel.recursive(5.0), theta=float(wl.theta),
                                                      m0=wl.m0))
    out = rep.output.data.double().cpu().numpy()
    emit({"row": "f2", "case": "cfg2 1920x1080x3, SpatialKernel.recursive(5.0), oracle landmarks",
          "maxabs": float(np.abs(out - ref["output"]).max()), "n_over_1e4": int((np.abs(out - ref["output"]) > 1e-4).sum()),
          "guarded_gpu": rep.guarded_pixels, "guarded_ref": ref["guarded_pixels"], "rank_gpu": rep.retained_rank,
          "rank_ref": ref["retained_rank"], "oracle_s": round(t1 - t0, 1)})

    # f1: brute force, full cfg 1 and a cfg-2 band
    for cfg, rows in ((1, None), (2, 256)):
        w = CONFIGS[cfg]
        g32 = w.image(seed=0, H=rows)
        g64 = g32.astype(np.float64)
        t0 = time.time()
        refb = O.brute_force_filter(g64, g64, w.theta, "gaussian_fir", w.sigma, w.radius)
        t1 = time.time()
        gi = Image(data=torch.from_numpy(g32).to(dev), range_max=1.0)
        outb = brute_force_filter(gi, gi, FilterParams(spatial=SpatialKernel.gaussian(w.sigma, w.radius),
                                                       theta=float(w.theta), m0=1)).data.double().cpu().numpy()
        emit({"row": "f1", "case": f"{w.name} {g32.shape[1]}x{g32.shape[2]}, window {2 * w.radius + 1}^2",
              "maxabs": float(np.abs(outb - refb).max()), "oracle_s": round(t1 - t0, 1)})

    # f3: PCA guide r=3 -> 25 and the NLM-PCA filter on it
    n32 = color_scene(384, 384, 40, 0.08, seed=3, lo=0.1, hi=0.9, shading=0.1)
    n64 = n32.astype(np.float64)
    t0 = time.time()
    gref = O.pca_patch_guide(n64, 3, 25)
    t1 = time.time()
    ni = Image(data=torch.from_numpy(n32).to(dev), range_max=1.0)
    gg = pca_patch_guide(ni, 3, 25)
    gout = gg.data.double().cpu().numpy()
    emit({"row": "f3", "case": "384x384x3 NLM scene, r=3 (147 dims) -> 25", "guide_maxabs": float(np.abs(gout - gref).max()),
          "guide_max": float(np.abs(gref).max()), "oracle_s": round(t1 - t0, 1)})
    theta = 3 * 0.08 * 3.0
    Cg, _, _, _ = O.kmeans(O.range_vectors(gref), 16, 0, 10)
    refn = O.fast_filter_with_landmarks(n64, gref, Cg, theta, "box", 0.0, 5, threads=16)
    repn = filter_with_landmarks(ni, gg, Cg, FilterParams(spatial=SpatialKernel.box(5), theta=theta, m0=16))
    on = repn.output.data.double().cpu().numpy()
    emit({"row": "f3", "case": "NLM-PCA filter (box 5, m0 16, oracle landmarks on the oracle guide)",
          "maxabs": float(np.abs(on - refn["output"]).max()), "guarded_gpu": repn.guarded_pixels,
          "guarded_ref": refn["guarded_pixels"]})

    # f4: metrics on cfg 2 (input vs its recursive-filtered output)
    a = Image(data=f64, range_max=1.0)
    b = Image(data=ref["output"], range_max=1.0)
    t0 = time.time()
    m_ref, p_ref, s_ref = O.mse(f64, ref["output"]), O.psnr(f64, ref["output"], 1.0), O.ssim(f64, ref["output"], 1.0)
    t1 = time.time()
    emit({"row": "f4", "case": "cfg2 1920x1080x3 pair (FP64)", "mse_rel": abs(mse(a, b) - m_ref) / m_ref,
          "psnr_abs": abs(psnr(a, b) - p_ref), "ssim_abs": abs(ssim(a, b) - s_ref), "oracle_s": round(t1 - t0, 1)})


if __name__ == "__main__":
    main()
