"""Host-side time of the pieces between the k-means centroids' arrival and the
K2 launch in one cfg-2 fast_filter step (perf_counter around each call; the
GPU is kept busy by the previous step's queue, so these are pure host costs)."""
import sys
import time
from collections import defaultdict
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import _params  # noqa: E402
from paper_1901_06112_b200 import Image, _native, fast_filter  # noqa: E402
from paper_1901_06112_b200 import filters as F  # noqa: E402
from paper_1901_06112_b200.synthetic import CONFIGS  # noqa: E402

acc = defaultdict(float)


def wrap(obj, name, label):
    fn = getattr(obj, name)

    def w(*a, **k):
        t = time.perf_counter()
        r = fn(*a, **k)
        acc[label] += time.perf_counter() - t
        return r

    setattr(obj, name, w)


lib = _native.lib()
wrap(F, "kmeans_device", "kmeans_device (incl. waiting for the GPU)")
wrap(F, "mixing_plan", "mixing_plan")
wrap(F, "_desc", "_desc")
wrap(F, "workspace", "workspace")
for nm in ("nys_filter_prepare", "nys_filter_hpass", "nys_filter_vpass", "nys_filter_workspace_bytes",
           "nys_filter_plane_row_stride", "nys_filter_stats"):
    wrap(lib, nm, nm)
wrap(F, "run_filter", "run_filter (total)")
wrap(F, "_prepare_inputs", "_prepare_inputs")

wl = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
f = Image(data=torch.from_numpy(wl.image(seed=0)).cuda(), range_max=1.0)
params = _params(wl)
for _ in range(5):
    fast_filter(f, f, params)
torch.cuda.synchronize()
acc.clear()
N = 20
t0 = time.perf_counter()
for _ in range(N):
    fast_filter(f, f, params)
torch.cuda.synchronize()
tot = time.perf_counter() - t0
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"{v / N * 1e6:9.1f} us  {k}")
print(f"{tot / N * 1e6:9.1f} us  whole step (wall)")
