"""CUDA-event time of the k-means stage on a config's guide (GPU box): the whole
nys_kmeans_run (seeding + Lloyd + exact pass) and seeding alone (max_iter 1), for A/B
switches given as environment variables.  usage: python tools/km_timing.py CFG"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1901_06112_b200.landmarks import kmeans_device  # noqa: E402
from paper_1901_06112_b200.synthetic import CONFIGS  # noqa: E402

wl = CONFIGS[int(sys.argv[1])]
f = torch.from_numpy(wl.image(seed=0)).cuda()
pts = f.reshape(f.shape[0], -1)


def run(it, reps=5):
    for _ in range(2):
        kmeans_device(pts, wl.m0, 0, it)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = kmeans_device(pts, wl.m0, 0, it)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts), r


full, r = run(wl.max_iter)
seed, _ = run(1)
print(f"cfg{sys.argv[1]}: kmeans {full:.3f} ms (iterations {r.iterations}), seeding+1 iter {seed:.3f} ms, "
      f"quant_error {r.quant_error:.9g}")
