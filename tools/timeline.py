"""CPU/GPU timeline of one cfg-2 fast_filter step (torch.profiler / CUPTI):
host call durations and GPU idle gaps between kernels."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import _guide, _params  # noqa: E402
from paper_1901_06112_b200 import Image, fast_filter  # noqa: E402
from paper_1901_06112_b200.synthetic import CONFIGS  # noqa: E402

wl = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
f = Image(data=torch.from_numpy(wl.image(seed=0)).cuda(), range_max=1.0)
g = _guide(f, wl)
params = _params(wl)
for _ in range(3):
    fast_filter(f, g, params)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        fast_filter(f, g, params)
    torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/timeline.json")
ev = json.load(open("gpurun_out/timeline.json"))["traceEvents"]
gpu = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
t0 = gpu[len(gpu) // 2]["ts"] if False else None
# second step only: kernels after the midpoint marker (two identical steps)
half = len(gpu) // 2
prev = None
for e in gpu[half:]:
    gap = (e["ts"] - prev) if prev is not None else 0.0
    print(f"{e['ts']:14.1f} gap {gap:8.1f} us  dur {e.get('dur', 0):8.1f} us  {e['name'][:60]}")
    prev = e["ts"] + e.get("dur", 0)

# the in-stream plan's own duration inside its host function (pipelined fast_filter)
import ctypes as C  # noqa: E402

from paper_1901_06112_b200 import _native  # noqa: E402
from paper_1901_06112_b200.filters import plan_staging_buffers  # noqa: E402

for buf in plan_staging_buffers():
    r = _native.PlanResult()
    _native.lib().nys_filter_plan_result(buf.data_ptr(), C.byref(r))
    print(f"in-stream plan: status {r.status} rank {r.rank} host function {r.host_us:.1f} us")
