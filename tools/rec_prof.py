"""One recursive-Gaussian filter on the cfg-2 image (for ncu)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1901_06112_b200 import FilterParams, Image, SpatialKernel, fast_filter  # noqa: E402
from paper_1901_06112_b200.synthetic import CONFIGS  # noqa: E402

wl = CONFIGS[2]
f = Image(data=torch.from_numpy(wl.image(seed=0)).cuda(), range_max=1.0)
p = FilterParams(spatial=SpatialKernel.recursive(float(sys.argv[1]) if len(sys.argv) > 1 else 5.0),
                 theta=float(wl.theta), m0=wl.m0, kmeans_max_iter=wl.max_iter)
for _ in range(2):
    r = fast_filter(f, f, p)
torch.cuda.synchronize()
print("ok", r.guarded_pixels, r.min_denominator)
