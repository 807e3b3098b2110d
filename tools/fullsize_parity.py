"""Full-size (or large-crop) parity of the GPU path against the FP64 oracle on
the GPU box's host: stage 1 (filter given the oracle's landmarks) and stage 2
(GPU k-means objective).  Writes one JSON line per config."""
import json, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import nys_oracle as O
from paper_1901_06112_b200 import FilterParams, Image, PatchGuide, SpatialKernel, fast_filter, filter_with_landmarks
from paper_1901_06112_b200.synthetic import CONFIGS

cfg = int(sys.argv[1])
H = int(sys.argv[2]) if len(sys.argv) > 2 else None
W = int(sys.argv[3]) if len(sys.argv) > 3 else None
wl = CONFIGS[cfg]
f32 = wl.image(H=H, W=W)
f64 = f32.astype(np.float64)
nlm = wl.mode == "nlm"
t0 = time.time()
p64 = O.patch_stack(f64, 1) if nlm else f64
C, _, qe, _ = O.kmeans(O.range_vectors(p64), wl.m0, 0, wl.max_iter)
t1 = time.time()
ref = O.fast_filter_with_landmarks(f64, p64, C, wl.theta, wl.spatial, wl.sigma, wl.radius, threads=16)
t2 = time.time()
sk = SpatialKernel.box(wl.radius) if wl.spatial == "box" else SpatialKernel.gaussian(wl.sigma, wl.radius)
params = FilterParams(spatial=sk, theta=float(wl.theta), m0=wl.m0, kmeans_max_iter=wl.max_iter)
f = Image(data=torch.from_numpy(f32).cuda(), range_max=1.0)
g = PatchGuide(f, 1) if nlm else f
r1 = filter_with_landmarks(f, g, C, params)
out1 = r1.output.data.double().cpu().numpy()
r2 = fast_filter(f, g, params)
out2 = r2.output.data.double().cpu().numpy()
R = ref["output"]
scale = np.maximum(1.0, np.abs(R))
res = dict(cfg=cfg, shape=list(f32.shape), oracle_kmeans_s=round(t1 - t0, 1), oracle_filter_s=round(t2 - t1, 1),
           stage1_maxabs=float(np.abs(out1 - R).max()), stage1_max_scaled=float((np.abs(out1 - R) / scale).max()),
           stage1_n_over_1e4=int((np.abs(out1 - R) > 1e-4).sum()),
           guarded_gpu=r1.guarded_pixels, guarded_ref=ref["guarded_pixels"],
           rank_gpu=r1.retained_rank, rank_ref=ref["retained_rank"],
           kmeans_qe_gpu=r2.quant_error, kmeans_qe_ref=qe, kmeans_rel=abs(r2.quant_error - qe) / qe,
           stage2_maxabs=float(np.abs(out2 - R).max()), stage2_max_scaled=float((np.abs(out2 - R) / scale).max()),
           out_of_unit_range_px=int((np.abs(R) > 1.0 + 1e-9).any(axis=0).sum() if R.ndim == 3 else 0))
# conditioning: pixels whose denominator sits within 2 decades of the guard
ratio = np.abs(ref["eta"]) / ref["eps_den"]
err1 = np.abs(out1 - R).max(axis=0) if R.ndim == 3 else np.abs(out1 - R)
well = ratio >= 100.0
res.update(near_guard_px=int(((ratio >= 1) & ~well).sum()),
           stage1_maxabs_well=float(err1[well].max()) if well.any() else 0.0,
           worst_px_eta_over_eps=float(ratio.flat[int(np.argmax(err1))]),
           worst_px_ref=float(np.abs(R).max(axis=0).flat[int(np.argmax(err1))] if R.ndim == 3 else 0.0))
print(json.dumps(res), flush=True)
