"""Time fast_filter end to end on one BASELINE config at full size (or a row crop)."""
import sys, time, json
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1901_06112_b200 import FilterParams, SpatialKernel, Image, PatchGuide, fast_filter
from paper_1901_06112_b200.synthetic import CONFIGS

cfg = int(sys.argv[1])
H = int(sys.argv[2]) if len(sys.argv) > 2 else None
wl = CONFIGS[cfg]
t = time.time()
f = torch.from_numpy(wl.image(H=H)).cuda()
print(f"cfg{cfg} gen {time.time()-t:.1f}s shape {tuple(f.shape)}", flush=True)
img = Image(data=f, range_max=1.0)
g = PatchGuide(img, 1) if wl.mode == "nlm" else img
sk = SpatialKernel.box(wl.radius) if wl.spatial == "box" else SpatialKernel.gaussian(wl.sigma, wl.radius)
p = FilterParams(spatial=sk, theta=float(wl.theta), m0=wl.m0, kmeans_max_iter=wl.max_iter)
for rep in range(3):
    ev = []
    torch.cuda.synchronize(); t = time.time()
    r = fast_filter(img, g, p, kernel_events=ev)
    torch.cuda.synchronize(); dt = time.time() - t
    px = f.shape[1] * f.shape[2]
    kk = {}
    for n_, a, b, _ in ev:
        kk[n_] = kk.get(n_, 0) + a.elapsed_time(b)
    print(f"rep {rep}: {dt*1e3:.1f} ms  {px/dt/1e6:.1f} Mpix/s  k={ {k: round(v,2) for k,v in kk.items()} } "
          f"stages={ {k: round(v*1e3,2) for k,v in r.timings.items()} } qe={r.quant_error:.6g} guarded={r.guarded_pixels} "
          f"min|eta|={r.min_denominator:.3g} bands={len(ev)//2}", flush=True)
