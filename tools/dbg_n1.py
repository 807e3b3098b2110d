import sys, os
import numpy as np, torch
sys.path.insert(0, ".")
from oracle import nys_oracle as O
from paper_1901_06112_b200 import FilterParams, Image, SpatialKernel, filter_with_landmarks
from paper_1901_06112_b200.synthetic import color_scene
for n, theta in ((1, 0.3), (1, 0.1), (2, 0.3), (3, 0.3)):
    f32 = np.ascontiguousarray(color_scene(40, 72, 5, 0.03, seed=40 + n)[:n])
    f = Image(data=torch.from_numpy(f32).cuda(), range_max=1.0)
    C, _, _, _ = O.kmeans(O.range_vectors(f32.astype(np.float64)), 6, 0, 6)
    params = FilterParams(spatial=SpatialKernel.gaussian(2.0, 6), theta=theta, m0=6)
    rep = filter_with_landmarks(f, f, C, params)
    ref = O.fast_filter_with_landmarks(f32.astype(np.float64), f32.astype(np.float64), C, theta, "gaussian_fir", 2.0, 6)
    out = rep.output.data.double().cpu().numpy()
    print(n, theta, os.environ.get("NYS_K2_SIMT"), "err", np.abs(out - ref["output"]).max(), "rank", ref["retained_rank"],
          "alphas", np.array2string(ref["alphas"], precision=3), "C", np.round(C.ravel(), 3))
