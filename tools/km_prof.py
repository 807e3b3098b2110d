"""k-means on a BASELINE config's guide (for ncu): python tools/km_prof.py CFG [reps]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1901_06112_b200 import Image, PatchGuide  # noqa: E402
from paper_1901_06112_b200.landmarks import kmeans_device  # noqa: E402
from paper_1901_06112_b200.synthetic import CONFIGS  # noqa: E402

wl = CONFIGS[int(sys.argv[1])]
f = torch.from_numpy(wl.image(seed=0)).cuda()
g = PatchGuide(Image(data=f, range_max=1.0), 1).device_planes(f) if wl.mode == "nlm" else f
pts = g.reshape(g.shape[0], -1)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    r = kmeans_device(pts, wl.m0, seed=0, max_iter=wl.max_iter)
torch.cuda.synchronize()
print("ok", r.quant_error, r.iterations)
