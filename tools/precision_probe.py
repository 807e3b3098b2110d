"""FP32 emulation of candidate GPU formulations vs the FP64 oracle.

y-form: convolve y_i*f_c, y_i with y = M b at the SOURCE pixel; contract with
b_i(x) at the centre.  b-form: convolve b_i*f_c, b_i; contract with y(x)=M b(x).
"""
import sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
from oracle import nys_oracle as O
from paper_1901_06112_b200.synthetic import CONFIGS

def conv32(planes, kind, sigma, R):
    planes = planes.astype(np.float32)
    if kind == "box":
        w = np.ones(2 * R + 1, np.float32)
    else:
        w = O.gaussian_taps(sigma, R).astype(np.float32)
    def fir(a):
        n = a.shape[-1]
        pad = np.concatenate([np.repeat(a[..., :1], R, -1), a, np.repeat(a[..., -1:], R, -1)], -1)
        out = np.zeros_like(a)
        for t in range(2 * R + 1):
            out += w[t] * pad[..., t:t + n]
        return out
    r = fir(planes)
    return np.ascontiguousarray(fir(r.transpose(0, 2, 1)).transpose(0, 2, 1))

def emulate(f, p, C, theta, kind, sigma, R, form):
    n, H, W = f.shape
    vals, vecs = O.jacobi_eig(O.gram(C, C, theta))
    al, Wk = O.retain(vals, vecs, 1e-8)
    M = (Wk / al[None, :]) @ Wk.T
    u0 = Wk[:, 0]; a0 = al[0]
    f32 = f.astype(np.float32); p32 = p.astype(np.float32); C32 = C.astype(np.float32)
    inv = np.float32(1.0 / (2 * theta * theta))
    b = np.empty((C.shape[0], H, W), np.float32)
    for i in range(C.shape[0]):
        d = p32 - C32[i][:, None, None]
        b[i] = np.exp(-(d * d).sum(0) * inv)
    M32 = M.astype(np.float32); u032 = u0.astype(np.float32)
    bf = b.reshape(C.shape[0], -1)
    y = (M32 @ bf).reshape(b.shape)
    s0 = (u032 @ bf).reshape(H, W)
    if form == "y":
        planes = np.concatenate([(y[:, None] * f32[None]), y[:, None]], 1).reshape(-1, H, W)
        G = conv32(planes, kind, sigma, R).reshape(C.shape[0], n + 1, H, W)
        num = (b[:, None] * G).sum(0)
        lp = np.concatenate([s0[None] * f32, s0[None]], 0)
        LG = conv32(lp, kind, sigma, R)
        lead = s0[None] * LG / np.float32(a0)
    else:
        planes = np.concatenate([(b[:, None] * f32[None]), b[:, None]], 1).reshape(-1, H, W)
        G = conv32(planes, kind, sigma, R).reshape(C.shape[0], n + 1, H, W)
        num = (y[:, None] * G).sum(0)
        lead = s0[None] * np.tensordot(u032, G, axes=(0, 0)) / np.float32(a0)
    eta = num[n]; zeta = num[:n]
    eps = 1e-12 * (2 * R + 1) ** 2 * np.abs(al).max()
    mask = np.abs(eta) < eps
    out = zeta / np.where(mask, 1, eta)
    ok = np.abs(lead[n]) >= eps
    fb = np.where(ok, lead[:n] / np.where(ok, lead[n], 1), f32)
    out = np.where(mask, fb, out)
    return out, int(mask.sum())

def run(cfg, H, W):
    wl = CONFIGS[cfg]
    f = wl.image(H=H, W=W).astype(np.float64)
    p = O.patch_stack(f, wl.patch_radius) if wl.mode == "nlm" else f
    t = time.time()
    C, _, qe, _ = O.kmeans(O.range_vectors(p), wl.m0, 0, wl.max_iter)
    ref = O.fast_filter_with_landmarks(f, p, C, wl.theta, wl.spatial, wl.sigma, wl.radius)
    print(f"cfg{cfg} {H}x{W}: ref guarded {ref['guarded_pixels']} min|eta| {ref['min_denominator']:.3g} ({time.time()-t:.1f}s)")
    for form in ("b", "y"):
        out, g = emulate(f, p, C, wl.theta, wl.spatial, wl.sigma, wl.radius, form)
        print(f"   {form}-form maxabs {np.abs(out - ref['output']).max():.3g} guarded {g}")

if __name__ == "__main__":
    run(1, 256, 256)
    run(2, 270, 480)
    run(3, 256, 256)
    run(4, 128, 128)
    run(5, 256, 256)
