"""Host-side profile (cProfile, after warm-up) of one public-API call on the GPU box:
`numpy` -- fast_filter(Image(np.float64)) (the reference's types); `sharded` -- the
row-band path at one rank (NCCL).  usage: python tools/host_profile.py numpy|sharded"""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from bench import _params  # noqa: E402
from paper_1901_06112_b200 import Image, fast_filter  # noqa: E402
from paper_1901_06112_b200.synthetic import CONFIGS  # noqa: E402

mode = sys.argv[1]
wl = CONFIGS[2]
params = _params(wl)
f32 = wl.image(seed=0)
if mode == "numpy":
    img = Image(data=f32.astype(np.float64), range_max=1.0)
    call = lambda: fast_filter(img, img, params)  # noqa: E731
else:
    import torch.distributed as dist

    from paper_1901_06112_b200.parallel import Comm, extended_band, sharded_fast_filter

    for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29531"), ("RANK", "0"), ("WORLD_SIZE", "1")):
        os.environ.setdefault(k, v)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl")
    comm = Comm()
    H = wl.H
    ext, top = extended_band(3, 0, H, H, params.spatial.effective_radius(), wl.W, torch.float32, "cuda")
    ext[:, top:top + H].copy_(torch.from_numpy(f32))
    call = lambda: sharded_fast_filter(None, H, params, comm, False, f_ext=ext)  # noqa: E731
for _ in range(3):
    call()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    call()
torch.cuda.synchronize()
print(f"{mode}: {(time.perf_counter() - t0) / 5 * 1e3:.2f} ms per call")
pr = cProfile.Profile()
pr.enable()
call()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
