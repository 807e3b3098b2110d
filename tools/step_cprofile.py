"""cProfile of 30 cfg-2 fast_filter steps (host-side Python cost per call)."""
import cProfile
import pstats
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import _params  # noqa: E402
from paper_1901_06112_b200 import Image, fast_filter  # noqa: E402
from paper_1901_06112_b200.synthetic import CONFIGS  # noqa: E402

wl = CONFIGS[2]
f = Image(data=torch.from_numpy(wl.image(seed=0)).cuda(), range_max=1.0)
params = _params(wl)
for _ in range(5):
    fast_filter(f, f, params)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(30):
    fast_filter(f, f, params)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(28)
