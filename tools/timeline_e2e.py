"""CUPTI timeline of one cfg-2 fast_filter call from pinned host memory into a pinned output (the e2e path)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import _params  # noqa: E402
from paper_1901_06112_b200 import Image, fast_filter  # noqa: E402
from paper_1901_06112_b200.synthetic import CONFIGS  # noqa: E402

wl = CONFIGS[2]
h = torch.from_numpy(wl.image(seed=0)).pin_memory()
out = torch.empty_like(h).pin_memory()
f = Image(data=h, range_max=1.0)
params = _params(wl)
for _ in range(3):
    fast_filter(f, f, params, out=out)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        fast_filter(f, f, params, out=out)
    torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/timeline_e2e.json")
ev = json.load(open("gpurun_out/timeline_e2e.json"))["traceEvents"]
gpu = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
prev = None
for e in gpu[len(gpu) // 2:]:
    gap = (e["ts"] - prev) if prev is not None else 0.0
    print(f"gap {gap:8.1f} us  dur {e.get('dur', 0):8.1f} us  {e['name'][:70]}")
    prev = e["ts"] + e.get("dur", 0)
