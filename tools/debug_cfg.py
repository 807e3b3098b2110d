"""Stage-by-stage timing of one config on the GPU (debug aid)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1901_06112_b200 import FilterParams, SpatialKernel, Image
from paper_1901_06112_b200.filters import _prepare_inputs, run_filter
from paper_1901_06112_b200.landmarks import kmeans_device
from paper_1901_06112_b200.synthetic import CONFIGS

cfg = int(sys.argv[1]); what = sys.argv[2]
wl = CONFIGS[cfg]
H = int(sys.argv[3]) if len(sys.argv) > 3 else wl.H
f = torch.from_numpy(wl.image(H=H)).cuda()
n, H, W = f.shape
pts = f.reshape(n, -1)
if what in ("seed", "km"):
    it = 1 if what == "seed" else wl.max_iter
    for rep in range(2):
        torch.cuda.synchronize(); t = time.time()
        r = kmeans_device(pts, wl.m0, 0, it)
        torch.cuda.synchronize(); print(what, rep, f"{(time.time()-t)*1e3:.2f} ms iters={r.iterations} qe={r.quant_error:.6g}", flush=True)
else:
    C = kmeans_device(pts, wl.m0, 0, 3).centroids
    sk = SpatialKernel.box(wl.radius) if wl.spatial == "box" else SpatialKernel.gaussian(wl.sigma, wl.radius)
    p = FilterParams(spatial=sk, theta=float(wl.theta), m0=wl.m0)
    img = Image(data=f, range_max=1.0)
    inp = _prepare_inputs(img, img)
    for rep in range(2):
        ev = []
        torch.cuda.synchronize(); t = time.time()
        out, plan, st = run_filter(inp, C, p, kernel_events=ev)
        torch.cuda.synchronize()
        print("filter", rep, f"{(time.time()-t)*1e3:.2f} ms", [(n_, round(a.elapsed_time(b), 3)) for n_, a, b, _ in ev], flush=True)
