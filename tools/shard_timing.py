"""CUDA-event breakdown of the one-rank sharded step (GPU box): seeding, Lloyd, exact pass,
filter.  usage: python tools/shard_timing.py"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, ".")
from bench import _params  # noqa: E402
from paper_1901_06112_b200 import parallel as P  # noqa: E402
from paper_1901_06112_b200.synthetic import CONFIGS  # noqa: E402

for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29533"), ("RANK", "0"), ("WORLD_SIZE", "1")):
    os.environ.setdefault(k, v)
torch.cuda.set_device(0)
dist.init_process_group("nccl")
wl = CONFIGS[2]
params = _params(wl)
f32 = torch.from_numpy(wl.image(seed=0)).cuda()
comm = P.Comm()
pts = f32.reshape(3, -1)
ev = []
orig_update = P._native.lib().nys_kmeanspp_update


def mark(name):
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    ev.append((name, e))


for rep in range(3):
    ev.clear()
    mark("start")
    km = P.device_distributed_kmeans(pts, comm, params.m0, 0, params.kmeans_max_iter)
    mark("kmeans")
    out, r = P.sharded_fast_filter(f32, wl.H, params, comm)
    mark("sharded_fast_filter(all)")
    torch.cuda.synchronize()
    print(rep, [(n, round(a.elapsed_time(b), 3)) for (_, a), (n, b) in zip(ev, ev[1:])])
import time
t0 = time.perf_counter()
km = P.device_distributed_kmeans(pts, comm, params.m0, 0, params.kmeans_max_iter)
torch.cuda.synchronize()
print("kmeans wall ms", (time.perf_counter() - t0) * 1e3)
