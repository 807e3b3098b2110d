"""Step-time outliers vs Python garbage collections during repeated fast_filter calls
(gc.callbacks time every collection): python tools/gc_probe.py CFG STEPS [freeze]"""
import gc
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import _guide, _params  # noqa: E402
from paper_1901_06112_b200 import Image, fast_filter  # noqa: E402
from paper_1901_06112_b200.synthetic import CONFIGS  # noqa: E402

wl = CONFIGS[int(sys.argv[1])]
steps = int(sys.argv[2])
f = Image(data=torch.from_numpy(wl.image(seed=0)).cuda(), range_max=1.0)
g = _guide(f, wl)
params = _params(wl)
for _ in range(3):
    fast_filter(f, g, params)
torch.cuda.synchronize()
if len(sys.argv) > 3:
    gc.collect()
    gc.freeze()
colls = []
t_start = {}


def cb(phase, info):
    if phase == "start":
        t_start["t"] = time.perf_counter()
    else:
        colls.append((info["generation"], (time.perf_counter() - t_start["t"]) * 1e3, len(ms)))


gc.callbacks.append(cb)
ms = []
for _ in range(steps):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    fast_filter(f, g, params)
    b.record()
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
med = sorted(ms)[len(ms) // 2]
print(f"cfg{sys.argv[1]} freeze={len(sys.argv) > 3} median {med:.3f} ms, max {max(ms):.3f}, "
      f"outliers(>1.1x) {[round(v, 2) for v in ms if v > 1.1 * med]}")
print("collections (gen, ms, step):", [(g_, round(d, 2), s) for g_, d, s in colls if d > 0.05][:20], "total", len(colls))
