"""One fast_filter call on a BASELINE config's synthetic image (for ncu captures)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import _guide, _params  # noqa: E402
from paper_1901_06112_b200 import Image, fast_filter  # noqa: E402
from paper_1901_06112_b200.synthetic import CONFIGS  # noqa: E402

wl = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
f = Image(data=torch.from_numpy(wl.image(seed=0)).cuda(), range_max=1.0)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    fast_filter(f, _guide(f, wl), _params(wl))
torch.cuda.synchronize()
