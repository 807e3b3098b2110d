"""k-means++ seeding micro-run for ncu: cfg-2-sized RGB points, m0 = 64."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1901_06112_b200.landmarks import kmeans_device  # noqa: E402
from paper_1901_06112_b200.synthetic import CONFIGS  # noqa: E402

f = torch.from_numpy(CONFIGS[2].image(seed=0)).cuda()
pts = f.reshape(3, -1)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    r = kmeans_device(pts, 64, seed=0, max_iter=15)
torch.cuda.synchronize()
print("ok", r.quant_error, r.iterations)
