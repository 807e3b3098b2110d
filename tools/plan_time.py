"""Distribution of the in-stream plan's host time over repeated cfg-2 calls."""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import _params  # noqa: E402
from paper_1901_06112_b200 import Image, _native, fast_filter  # noqa: E402
from paper_1901_06112_b200.filters import plan_staging_buffers  # noqa: E402
from paper_1901_06112_b200.synthetic import CONFIGS  # noqa: E402

wl = CONFIGS[2]
f = Image(data=torch.from_numpy(wl.image(seed=0)).cuda(), range_max=1.0)
params = _params(wl)
us = []
for k in range(35):
    fast_filter(f, f, params)
    r = _native.PlanResult()
    _native.lib().nys_filter_plan_result(plan_staging_buffers()[0].data_ptr(), C.byref(r))
    if k >= 5:
        us.append(r.host_us)
us.sort()
print(f"plan host us: min {us[0]:.1f} median {us[len(us) // 2]:.1f} p90 {us[int(len(us) * 0.9)]:.1f} max {us[-1]:.1f}")
