"""Near-guard refinement sweep on a full-size config (GPU box): stage-1 parity
(filter given the oracle's landmarks) vs the FP64 oracle for several
(NYS_REFINE_TAU, NYS_REFINE_CERR) settings, the number of pixels the
refinement changed, and the filter's device time.  One JSON line per setting.

usage: python tools/refine_sweep.py CFG [H W] [tau:cerr ...]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import nys_oracle as O  # the checker
from paper_1901_06112_b200 import FilterParams, Image, PatchGuide, SpatialKernel, filter_with_landmarks
from paper_1901_06112_b200.synthetic import CONFIGS

cfg = int(sys.argv[1])
rest = sys.argv[2:]
H = W = None
if len(rest) >= 2 and ":" not in rest[0]:
    H, W = int(rest[0]), int(rest[1])
    rest = rest[2:]
settings = [tuple(float(v) for v in s.split(":")) for s in rest] or [(0.0, 0.0), (1e-3, 1e-4), (1e-2, 1e-3), (3e-2, 3e-3)]
wl = CONFIGS[cfg]
f32 = wl.image(H=H, W=W)
f64 = f32.astype(np.float64)
nlm = wl.mode == "nlm"
t0 = time.time()
p64 = O.patch_stack(f64, 1) if nlm else f64
C, _, qe, _ = O.kmeans(O.range_vectors(p64), wl.m0, 0, wl.max_iter)
t1 = time.time()
ref = O.fast_filter_with_landmarks(f64, p64, C, wl.theta, wl.spatial, wl.sigma, wl.radius, threads=16)
t2 = time.time()
R = ref["output"]
ratio = np.abs(ref["eta"]) / ref["eps_den"]
sk = SpatialKernel.box(wl.radius) if wl.spatial == "box" else SpatialKernel.gaussian(wl.sigma, wl.radius)
params = FilterParams(spatial=sk, theta=float(wl.theta), m0=wl.m0, kmeans_max_iter=wl.max_iter)
f = Image(data=torch.from_numpy(f32).cuda(), range_max=1.0)
g = PatchGuide(f, 1) if nlm else f
base = None
for tau, cerr in settings:
    os.environ["NYS_REFINE_TAU"] = repr(tau)
    os.environ["NYS_REFINE_CERR"] = repr(cerr)
    r = filter_with_landmarks(f, g, C, params)
    out = r.output.data.double().cpu().numpy()
    times = []
    for _ in range(3):
        torch.cuda.synchronize()
        a = time.perf_counter()
        filter_with_landmarks(f, g, C, params)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - a)
    err = np.abs(out - R)
    errpx = err.max(axis=0)
    if base is None:
        base = out
    changed = int((np.abs(out - base) > 0).any(axis=0).sum())
    worst = int(np.argmax(errpx))
    print(json.dumps(dict(cfg=cfg, shape=list(f32.shape), tau=tau, cerr=cerr, oracle_s=round(t2 - t0, 1),
                          maxabs=float(err.max()), n_over_1e4=int((errpx > 1e-4).sum()),
                          n_over_1e5=int((errpx > 1e-5).sum()),
                          guarded_gpu=r.guarded_pixels, guarded_ref=ref["guarded_pixels"],
                          min_den_gpu=r.min_denominator, min_den_ref=ref["min_denominator"],
                          px_changed_vs_first=changed, worst_eta_over_eps=float(ratio.flat[worst]),
                          worst_ref=float(np.abs(R).max(axis=0).flat[worst]),
                          filter_ms=round(1e3 * min(times), 3))), flush=True)
