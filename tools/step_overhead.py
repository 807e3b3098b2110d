"""Host time inside one timed cfg-2 step outside the GPU's work: from the step
start to the first native launch (nys_kmeans_run), and from the step's only
host wait returning to fast_filter returning (perf_counter stamps)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import _params  # noqa: E402
from paper_1901_06112_b200 import Image, _native, fast_filter  # noqa: E402
from paper_1901_06112_b200 import filters as F  # noqa: E402
from paper_1901_06112_b200.synthetic import CONFIGS  # noqa: E402

stamps = {}
lib = _native.lib()
_run = lib.nys_kmeans_run


def run(*a):
    stamps.setdefault("launch", time.perf_counter())
    r = _run(*a)
    stamps.setdefault("launched", time.perf_counter())
    return r


lib.nys_kmeans_run = run
_res = F._Inflight.result


def result(self):
    stamps["synced"] = time.perf_counter()
    return _res(self)


F._Inflight.result = result
acc = {}


def timed(obj, name, label):
    fn = getattr(obj, name)

    def w(*a, **k):
        t = time.perf_counter()
        r = fn(*a, **k)
        acc[label] = acc.get(label, 0.0) + time.perf_counter() - t
        return r

    setattr(obj, name, w)


from paper_1901_06112_b200 import _device, landmarks  # noqa: E402

timed(_device.StageTimer, "elapsed", "StageTimer.elapsed")
timed(landmarks.PendingKMeans, "finish", "PendingKMeans.finish")
timed(F, "_output_image", "_output_image")
timed(F, "_prepare_inputs", "_prepare_inputs")
timed(F, "_check_sizes", "_check_sizes")
timed(F, "kmeans_device", "kmeans_device (python side)")
wl = CONFIGS[2]
f = Image(data=torch.from_numpy(wl.image(seed=0)).cuda(), range_max=1.0)
params = _params(wl)
for _ in range(5):
    fast_filter(f, f, params)
from paper_1901_06112_b200 import _device  # noqa: E402

pre, post, tot = [], [], []
seg = {}
for _ in range(30):
    torch.cuda.synchronize()
    stamps.clear()
    _device.STAMPS = []
    t0 = time.perf_counter()
    fast_filter(f, f, params)
    t1 = time.perf_counter()
    prev = t0
    for lab, t in _device.STAMPS + [("native call", stamps["launch"]), ("nys_kmeans_run", stamps["launched"])]:
        seg.setdefault(lab, []).append(t - prev)
        prev = t
    _device.STAMPS = None
    pre.append(stamps["launch"] - t0)
    post.append(t1 - stamps["synced"])
    tot.append(t1 - t0)
for k, v in seg.items():
    print(f"  {k:22s} {sorted(v)[len(v) // 2] * 1e6:7.1f} us")
for k, v in acc.items():
    print(f"{k}: {v / 35 * 1e6:.1f} us/step")
med = lambda v: sorted(v)[len(v) // 2] * 1e6  # noqa: E731
print(f"step start -> first launch {med(pre):.1f} us; host wait returned -> fast_filter returned {med(post):.1f} us; "
      f"step wall {med(tot):.1f} us")
