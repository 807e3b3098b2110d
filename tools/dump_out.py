"""Dump the GPU filter output (stage 1: given the oracle's landmarks) of a config
to gpurun_out/out_cfg{N}_{tag}.npy for host-side error analysis (GPU box).
The landmarks are the oracle's k-means (bit-identical to the reference's).

usage: NYS_REFINE_TAU=.. python tools/dump_out.py CFG TAG [H W]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import nys_oracle as O  # the checker (landmarks)
from paper_1901_06112_b200 import FilterParams, Image, PatchGuide, SpatialKernel, filter_with_landmarks
from paper_1901_06112_b200.synthetic import CONFIGS

cfg, tag = int(sys.argv[1]), sys.argv[2]
H = int(sys.argv[3]) if len(sys.argv) > 3 else None
W = int(sys.argv[4]) if len(sys.argv) > 4 else None
wl = CONFIGS[cfg]
f32 = wl.image(H=H, W=W)
f64 = f32.astype(np.float64)
nlm = wl.mode == "nlm"
p64 = O.patch_stack(f64, 1) if nlm else f64
C, _, qe, _ = O.kmeans(O.range_vectors(p64), wl.m0, 0, wl.max_iter)
sk = SpatialKernel.box(wl.radius) if wl.spatial == "box" else SpatialKernel.gaussian(wl.sigma, wl.radius)
params = FilterParams(spatial=sk, theta=float(wl.theta), m0=wl.m0, kmeans_max_iter=wl.max_iter)
f = Image(data=torch.from_numpy(f32).cuda(), range_max=1.0)
g = PatchGuide(f, 1) if nlm else f
r = filter_with_landmarks(f, g, C, params)
out = r.output.data.cpu().numpy()
np.save(f"gpurun_out/out_cfg{cfg}_{tag}.npy", out)
np.save(f"gpurun_out/centroids_cfg{cfg}.npy", C)
print(tag, r.guarded_pixels, r.min_denominator)
