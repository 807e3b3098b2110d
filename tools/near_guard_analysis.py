"""Host-side analysis of the near-guard flag rule: given a GPU
output dumped by tools/dump_out.py (refinement off), compute the FP64 oracle,
the per-pixel error and candidate FP32-error scales of eta, and report how
well each scale separates the pixels whose error exceeds a threshold.

  S0 = sum_i b_i(x) |G_i(x)|                       (contraction scale)
  S1 = sum_i b_i(x) |G_i(x)| (1 + |log2 b_i(x)|)    (+ exp-argument error of b)
  SA = sum_i b_i(x) conv(|y_i|)(x)                  (+ cancellation inside y = M b)
with G_i = conv(y_i), y = M b (FP64 y-form).

usage: python tools/near_guard_analysis.py CFG gpurun_out/out_cfgN_norefine.npy [H W]"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import nys_oracle as O
from paper_1901_06112_b200.synthetic import CONFIGS

cfg = int(sys.argv[1])
gpu = np.load(sys.argv[2]).astype(np.float64)
H = int(sys.argv[3]) if len(sys.argv) > 3 else None
W = int(sys.argv[4]) if len(sys.argv) > 4 else None
wl = CONFIGS[cfg]
f32 = wl.image(H=H, W=W)
f64 = f32.astype(np.float64)
p64 = O.patch_stack(f64, 1) if wl.mode == "nlm" else f64
C, _, _, _ = O.kmeans(O.range_vectors(p64), wl.m0, 0, wl.max_iter)
ref = O.fast_filter_with_landmarks(f64, p64, C, wl.theta, wl.spatial, wl.sigma, wl.radius, threads=8)
n, Hh, Ww = f64.shape
err = np.abs(gpu - ref["output"]).max(axis=0)
A = O.gram(C, C, wl.theta)
M = np.linalg.inv(A)
B = O.gram(C, O.range_vectors(p64), wl.theta)  # (m0, m)
Y = M @ B
G = O.spatial_conv(Y.reshape(-1, Hh, Ww), wl.spatial, wl.sigma, wl.radius).reshape(wl.m0, -1)
GA = O.spatial_conv(np.abs(Y).reshape(-1, Hh, Ww), wl.spatial, wl.sigma, wl.radius).reshape(wl.m0, -1)
lb = np.abs(np.log2(np.maximum(B, 1e-300)))
S0 = (B * np.abs(G)).sum(0)
S1 = (B * np.abs(G) * (1 + lb)).sum(0)
SA = (B * GA).sum(0)
S2 = (B * GA * (1 + lb)).sum(0)
eta = np.abs(ref["eta"]).ravel()
eps = ref["eps_den"]
res = {"cfg": cfg, "eps_den": eps, "n_px": int(err.size)}
for thr in (1e-4, 1e-5, 2e-6):
    bad = err.ravel() > thr
    res[f"n_err_gt_{thr:g}"] = int(bad.sum())
    for nm, S in (("S0", S0), ("S1", S1), ("SA", SA), ("S2", S2)):
        r = eta / np.maximum(S, 1e-300)
        if bad.any():
            worst = float(r[bad].max())  # every bad pixel is caught by tau > worst
            res[f"{nm}_maxratio_bad_{thr:g}"] = worst
            for mult in (1.0, 3.0, 10.0):
                res[f"{nm}_flagged_at_{mult:g}x_{thr:g}"] = int((r < worst * mult).sum())
print(json.dumps(res))
