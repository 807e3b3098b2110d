import sys, numpy as np, torch, ctypes as C
sys.path.insert(0, '/root/repo')
from paper_1901_06112_b200 import _native
from paper_1901_06112_b200.landmarks import kmeans_device
from paper_1901_06112_b200.nystrom import mixing_plan, PHI_FORM_COND
from paper_1901_06112_b200.synthetic import CONFIGS
wl = CONFIGS[2]
f = torch.from_numpy(wl.image(seed=0)).cuda()
km = kmeans_device(f.reshape(3, -1), 64, 0, 15)
Cc = np.ascontiguousarray(km.centroids)
lib = _native.lib()
al = np.empty(64); M = np.empty((64, 64)); u0 = np.empty(64); r = C.c_int()
rc = lib.nys_mixing_plan_lite(Cc.ctypes.data, 64, 3, float(wl.theta), 1e-8, PHI_FORM_COND, 1, al.ctypes.data, C.byref(r), M.ctypes.data, u0.ctypes.data)
full = mixing_plan(Cc, float(wl.theta), 1e-8, 15)
print("rc", rc, "rank", r.value, "full rank", full.rank, "phi", full.phi_form, "cond", full.alphas[0] / full.alphas[-1])
p = mixing_plan(Cc, float(wl.theta), 1e-8, 15, lite=True, device_inverse=True)
print("lite plan chol", p.M_is_cholesky, "rank", p.rank)
np.save("gpurun_out/cfg2_centroids.npy", Cc)
