"""Small invocations of every kernel on the hot path, for compute-sanitizer
(tools/sanitize.sh): BLF Gaussian (k_seed_runs, k_lloyd_coop, k_exact,
k_inverse_cholesky, k_feat_hpass_tc, k_vpass, k_finish), NLM box with the
in-kernel patch guide, a 31-band cube (chunked K3), the synchronous plan, and
the SIMT K2.  usage: san_cases.py [case ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_06112_b200 import FilterParams, Image, PatchGuide, SpatialKernel, fast_filter  # noqa: E402
from paper_1901_06112_b200.synthetic import color_scene  # noqa: E402


def blf():
    f32 = color_scene(48, 72, 6, 0.04, seed=5)
    f = Image(data=torch.from_numpy(f32).cuda(), range_max=1.0)
    p = FilterParams(spatial=SpatialKernel.gaussian(3.0, 9), theta=0.15, m0=16, kmeans_max_iter=6)
    return fast_filter(f, f, p)


def nlm():
    f32 = color_scene(40, 56, 6, 0.08, seed=7)
    f = Image(data=torch.from_numpy(f32).cuda(), range_max=1.0)
    p = FilterParams(spatial=SpatialKernel.box(4), theta=0.3 * np.sqrt(27) * 0.08, m0=16, kmeans_max_iter=5)
    return fast_filter(f, PatchGuide(f, 1), p)


def cube():
    rng = np.random.default_rng(3)
    f32 = np.clip(rng.random((31, 24, 40)) * 0.5 + 0.25, 0, 1).astype(np.float32)
    f = Image(data=torch.from_numpy(f32).cuda(), range_max=1.0)
    p = FilterParams(spatial=SpatialKernel.gaussian(2.0, 6), theta=0.25, m0=12, kmeans_max_iter=4)
    return fast_filter(f, f, p)


CASES = {"blf": blf, "nlm": nlm, "cube": cube}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    torch.cuda.set_device(0)
    for nm in names:
        rep = CASES[nm]()
        torch.cuda.synchronize()
        out = rep.output.data
        print(nm, "ok", tuple(out.shape), float(out.double().mean()), "rank", rep.retained_rank, "guarded",
              rep.guarded_pixels, flush=True)
