"""Break the end-to-end (pinned host in / pinned host out) step into stages."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1901_06112_b200 import FilterParams, Image, SpatialKernel, fast_filter
from paper_1901_06112_b200.synthetic import CONFIGS
wl = CONFIGS[2]
f_np = wl.image()
f_host = torch.from_numpy(f_np).pin_memory()
params = FilterParams(spatial=SpatialKernel.gaussian(wl.sigma, wl.radius), theta=float(wl.theta), m0=wl.m0,
                      kmeans_max_iter=wl.max_iter)
img = Image(data=f_host, range_max=1.0)
dimg = Image(data=f_host.cuda(), range_max=1.0)
for name, im in (("host", img), ("device", dimg)):
    for r in range(4):
        torch.cuda.synchronize(); t = time.perf_counter()
        rep = fast_filter(im, im, params)
        torch.cuda.synchronize(); dt = (time.perf_counter() - t) * 1e3
    print(name, f"{dt:.2f} ms", {k: round(v * 1e3, 3) for k, v in rep.timings.items()})
x = torch.empty_like(f_host).cuda()
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(10): x.copy_(f_host, non_blocking=True)
torch.cuda.synchronize(); print("H2D 25MB ms", (time.perf_counter() - t) * 100)
h = torch.empty(f_host.shape, dtype=torch.float32, pin_memory=True)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(10): h.copy_(x)
torch.cuda.synchronize(); print("D2H 25MB ms", (time.perf_counter() - t) * 100)
t = time.perf_counter()
for _ in range(10): h2 = torch.empty(f_host.shape, dtype=torch.float32, pin_memory=True)
print("pinned alloc ms", (time.perf_counter() - t) * 100)
