"""Debug: recursive (global / shared) and FIR paths vs the oracle on small single-channel images."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, '/root/repo')
from oracle import nys_oracle as O  # noqa: E402
from paper_1901_06112_b200 import FilterParams, Image, SpatialKernel, filter_with_landmarks  # noqa: E402
from paper_1901_06112_b200.synthetic import color_scene  # noqa: E402

for (H, W, n, m0, th) in [(130, 9, 1, 5, 0.35), (130, 9, 2, 5, 0.35), (130, 9, 3, 5, 0.35), (9, 130, 1, 5, 0.35),
                          (64, 64, 1, 5, 0.35), (130, 9, 1, 3, 0.5)]:
    f32 = np.ascontiguousarray(color_scene(H, W, 5, 0.05, seed=H + n)[:n])
    f64 = f32.astype(np.float64)
    C, _, _, _ = O.kmeans(O.range_vectors(f64), m0, 0, 6)
    A = O.gram(C, C, th)
    f = Image(data=torch.from_numpy(f32).cuda(), range_max=1.0)
    res = []
    for kind, sk in (("rec", SpatialKernel.recursive(2.5)), ("fir", SpatialKernel.gaussian(2.5, 8))):
        params = FilterParams(spatial=sk, theta=th, m0=m0)
        a = filter_with_landmarks(f, f, C, params).output.data.double().cpu().numpy()
        ref = O.fast_filter_with_landmarks(f64, f64, C, th, sk.kind, 2.5, 8)["output"]
        res.append(f"{kind} {np.abs(a - ref).max():.2e}")
    print(H, W, n, m0, th, "cond", f"{np.linalg.cond(A):.1e}", *res)
