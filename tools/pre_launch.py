"""Cost of each host piece before a cfg-2 step's first launch (median of 200)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import _params  # noqa: E402
from paper_1901_06112_b200 import Image, _native, fast_filter  # noqa: E402
from paper_1901_06112_b200 import filters as F  # noqa: E402
from paper_1901_06112_b200 import landmarks as LM  # noqa: E402
from paper_1901_06112_b200._device import StageTimer, require_cuda, stream_ptr, workspace  # noqa: E402
from paper_1901_06112_b200.synthetic import CONFIGS  # noqa: E402

wl = CONFIGS[2]
f = Image(data=torch.from_numpy(wl.image(seed=0)).cuda(), range_max=1.0)
params = _params(wl)
fast_filter(f, f, params)
torch.cuda.synchronize()


def med(fn, n=200):
    ts = []
    for _ in range(n):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return sorted(ts)[n // 2] * 1e6


inp = F._prepare_inputs(f, f)
lib = _native.lib()
print(f"require_cuda           {med(require_cuda):6.1f} us")
print(f"stream_ptr             {med(stream_ptr):6.1f} us")
print(f"StageTimer()+mark      {med(lambda: StageTimer().mark('x')):6.1f} us")
print(f"torch.cuda.Event+rec   {med(lambda: torch.cuda.Event(enable_timing=True).record()):6.1f} us")
print(f"_check_sizes           {med(lambda: F._check_sizes(f, f)):6.1f} us")
print(f"f.width/height/chan    {med(lambda: (f.width, f.height, f.channels)):6.1f} us")
print(f"_prepare_inputs        {med(lambda: F._prepare_inputs(f, f)):6.1f} us")
print(f"_pipelined_ok          {med(lambda: F._pipelined_ok(inp, params)):6.1f} us")
print(f"workspace(1MB)         {med(lambda: workspace(1 << 20)):6.1f} us")
print(f"torch.empty f64 (200)  {med(lambda: torch.empty(200, dtype=torch.float64, device='cuda')):6.1f} us")
print(f"_seed_stream           {med(lambda: LM._seed_stream(inp.points.shape[1], 64, 0)):6.1f} us")
print(f"kmeans ws bytes        {med(lambda: lib.nys_kmeans_workspace_bytes(inp.points.shape[1], 3, 64)):6.1f} us")
print(f"nys_abi_version        {med(lambda: lib.nys_abi_version()):6.1f} us")
evs = [torch.cuda.Event(enable_timing=True) for _ in range(400)]
it = iter(evs)
print(f"Event.record (reused)  {med(lambda: next(it).record()):6.1f} us")
print(f"Event() create only    {med(lambda: torch.cuda.Event(enable_timing=True)):6.1f} us")
