"""Small filter calls for compute-sanitizer (tools/sanitize.sh): the pipelined
BLF step (k_seed_prologue, k_seed_runs, k_lloyd_coop, k_exact, the in-stream
plan + k_inverse_cholesky, K2, K3, k_finish), the NLM patch-guide path (b planes,
near-guard refinement) and the synchronous plan path."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1901_06112_b200 import FilterParams, Image, PatchGuide, SpatialKernel, fast_filter, filter_with_landmarks
from paper_1901_06112_b200.synthetic import color_scene

f32 = color_scene(48, 70, 6, 0.05, seed=3)
f = Image(data=torch.from_numpy(f32).cuda(), range_max=1.0)
which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("blf", "all"):
    r = fast_filter(f, f, FilterParams(spatial=SpatialKernel.gaussian(3.0, 9), theta=0.15, m0=16, kmeans_max_iter=6))
    torch.cuda.synchronize()
    print("blf ok", r.guarded_pixels, float(r.output.data.abs().max()))
if which in ("nlm", "all"):
    p = PatchGuide(f, 1)
    r = fast_filter(f, p, FilterParams(spatial=SpatialKernel.box(4), theta=0.06, m0=12, kmeans_max_iter=5))
    torch.cuda.synchronize()
    print("nlm ok", r.guarded_pixels)
if which in ("sync", "all"):
    os.environ["NYS_PIPELINED"] = "0"
    r = fast_filter(f, f, FilterParams(spatial=SpatialKernel.gaussian(2.0, 6), theta=0.2, m0=8, kmeans_max_iter=4))
    torch.cuda.synchronize()
    print("sync ok", r.guarded_pixels)
