"""Measure the §8(f) rows on one B200: recursive-Gaussian filter (f2),
brute-force filter (f1), PCA patch guide (f3), quality metrics (f4).

    python tools/bench_next.py [--steps 10] [--warmup 3] > profiles/rN_next.jsonl

Device-resident inputs, CUDA events on the launching stream, L2 flushed
(512 MB write) before every timed step; one JSON line per row.  ``bytes_px``
is the algorithmic DRAM traffic per pixel of the design named in ``design``.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1901_06112_b200 import (  # noqa: E402
    FilterParams,
    Image,
    SpatialKernel,
    _native,
    brute_force_filter,
    fast_filter,
    pca_patch_guide,
    quality,
)
from paper_1901_06112_b200.synthetic import CONFIGS, color_scene  # noqa: E402

PEAK = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
HBM = float(PEAK.get("hbm_gbs", 6650.0))


def timed(fn, steps, warmup, flush):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ms = []
    lib = _native.lib()
    l0 = int(lib.nys_kernel_launches())
    for _ in range(steps):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return float(np.median(ms)), (int(lib.nys_kernel_launches()) - l0) // steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    buf = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def flush():
        buf.random_(0, 255)

    out = []
    # f2: cfg 2 workload with the recursive Gaussian (the CLI's default spatial backend) instead of the FIR
    wl = CONFIGS[2]
    f = Image(data=torch.from_numpy(wl.image(seed=0)).to(dev), range_max=1.0)
    n, H, W = f.data.shape
    px = H * W
    for sigma in (5.0, 20.0):
        params = FilterParams(spatial=SpatialKernel.recursive(sigma), theta=float(wl.theta), m0=wl.m0,
                              kmeans_max_iter=wl.max_iter)
        evs = []

        def run():
            evs.clear()
            fast_filter(f, f, params, kernel_events=evs)

        ms, launches = timed(run, args.steps, args.warmup, flush)
        k_ms = evs[0][1].elapsed_time(evs[0][2])
        P = (wl.m0 + 1) * (n + 1)
        # Y, B written once + read once; row pass: fwd write, bwd read + write; column pass: fwd read + write,
        # bwd read (feeds the contraction only); Z / lead planes written + read; f read twice; output written
        bpx = 4 * (2 * (wl.m0 + 1) + 2 * wl.m0) + 4 * 6 * P - 4 * P + 4 * 4 * (n + 1) + 4 * 3 * n
        out.append({"row": "f2 recursive Gaussian", "workload": f"{wl.name} with SpatialKernel.recursive({sigma})",
                    "ms_per_step": round(ms, 3), "mpix_s": round(px / ms / 1e3, 1), "gpu_launches": launches,
                    "filter_ms": round(k_ms, 3), "bytes_px": bpx,
                    "achieved_gbs": round(bpx * px / k_ms / 1e6, 1), "hbm_peak_gbs": HBM,
                    "frac": round(bpx * px / k_ms / 1e6 / HBM, 3),
                    "design": "features -> row IIR (fwd/bwd in place) -> column IIR fused with the contraction"})

    # f1: brute force, cfg 1 kernel (sigma 3, R 9) at 512x512 and the cfg 2 kernel at 1080p
    for cfg in (1, 2):
        w = CONFIGS[cfg]
        fi = Image(data=torch.from_numpy(w.image(seed=0)).to(dev), range_max=1.0)
        params = FilterParams(spatial=SpatialKernel.gaussian(w.sigma, w.radius), theta=float(w.theta), m0=1)
        ms, launches = timed(lambda: brute_force_filter(fi, fi, params), args.steps, args.warmup, flush)
        T = 2 * w.radius + 1
        ops = T * T * (2 * 3 + 3 + 3)  # diff+fma per dim, exp scale, n fma + den
        pxx = w.H * w.W
        out.append({"row": "f1 brute_force_filter", "workload": f"{w.name} window {T}x{T}",
                    "ms_per_step": round(ms, 3), "mpix_s": round(pxx / ms / 1e3, 1), "gpu_launches": launches,
                    "fp32_ops_px": ops, "achieved_tops": round(ops * pxx / ms / 1e9, 2)})

    # f3: PCA patch guide, 1024x1024x3, r = 3 (147 dims) -> 25, and r = 1 -> 10
    f3 = Image(data=torch.from_numpy(color_scene(1024, 1024, 64, 0.08, seed=3, lo=0.1, hi=0.9,
                                                 shading=0.1)).to(dev), range_max=1.0)
    for r, k in ((3, 25), (1, 10)):
        ms, launches = timed(lambda: pca_patch_guide(f3, r, k), args.steps, args.warmup, flush)
        dim = 3 * (2 * r + 1) ** 2
        out.append({"row": "f3 pca_patch_guide", "workload": f"1024x1024x3 r={r} ({dim} dims) -> {k}",
                    "ms_per_step": round(ms, 3), "mpix_s": round(1024 * 1024 / ms / 1e3, 1),
                    "gpu_launches": launches, "fp64_gram_flops": 2 * 1024 * 1024 * dim * (dim + 4) / 2})

    # f4: quality metrics of two 1080p RGB frames
    a = Image(data=f.data, range_max=1.0)
    b = Image(data=(f.data + 0.01).clamp(0, 1), range_max=1.0)
    ms, launches = timed(lambda: quality(a, b), args.steps, args.warmup, flush)
    out.append({"row": "f4 quality (mse/psnr/ssim)", "workload": "1920x1080x3 float32 pair",
                "ms_per_step": round(ms, 3), "mpix_s": round(px / ms / 1e3, 1), "gpu_launches": launches})
    for o in out:
        print(json.dumps(o), flush=True)


if __name__ == "__main__":
    main()
