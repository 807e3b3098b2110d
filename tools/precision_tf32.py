"""Emulate y = M b with TF32 operands (tcgen05 kind::tf32) inside the y-form
filter and compare with the FP64 oracle (which variant keeps max-abs << 1e-4)."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tools")
from oracle import nys_oracle as O
from paper_1901_06112_b200.synthetic import CONFIGS
from precision_probe import conv32


def tf32(x):
    x = np.asarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = ((u + 0x1000) & 0xFFFFE000).astype(np.uint32)  # round-to-nearest to 10 mantissa bits
    return u.view(np.float32)


def run(cfg, H, W, mode):
    wl = CONFIGS[cfg]
    f = wl.image(H=H, W=W).astype(np.float64)
    p = O.patch_stack(f, 1) if wl.mode == "nlm" else f
    C, _, _, _ = O.kmeans(O.range_vectors(p), wl.m0, 0, wl.max_iter)
    ref = O.fast_filter_with_landmarks(f, p, C, wl.theta, wl.spatial, wl.sigma, wl.radius)
    vals, vecs = O.jacobi_eig(O.gram(C, C, wl.theta))
    al, Wk = O.retain(vals, vecs, 1e-8)
    M = ((Wk / al) @ Wk.T).astype(np.float32)
    u0 = Wk[:, 0].astype(np.float32)
    f32, p32, C32 = f.astype(np.float32), p.astype(np.float32), C.astype(np.float32)
    inv = np.float32(1.0 / (2 * wl.theta ** 2))
    m0 = C.shape[0]
    b = np.empty((m0,) + f.shape[1:], np.float32)
    for i in range(m0):
        d = p32 - C32[i][:, None, None]
        b[i] = np.exp(-(d * d).sum(0) * inv)
    bf = b.reshape(m0, -1)
    Mx = np.concatenate([M, u0[None]], 0)  # (m0+1, m0): the lead row rides along
    if mode == "fp32":
        Y = Mx @ bf
    elif mode == "1xtf32":
        Y = tf32(Mx) @ tf32(bf)
    elif mode == "3xtf32":
        bh, Mh = tf32(bf), tf32(Mx)
        bl, Ml = tf32(bf - bh), tf32(Mx - Mh)
        Y = Mh @ bh + Mh @ bl + Ml @ bh
    Y = Y.astype(np.float32).reshape((m0 + 1,) + f.shape[1:])
    y, s0 = Y[:m0], Y[m0]
    planes = np.concatenate([(y[:, None] * f32[None]), y[:, None]], 1).reshape(-1, *f.shape[1:])
    G = conv32(planes, wl.spatial, wl.sigma, wl.radius).reshape(m0, f.shape[0] + 1, *f.shape[1:])
    num = (b[:, None] * G).sum(0)
    LG = conv32(np.concatenate([s0[None] * f32, s0[None]], 0), wl.spatial, wl.sigma, wl.radius)
    lead = s0[None] * LG / np.float32(al[0])
    n = f.shape[0]
    eta, zeta = num[n], num[:n]
    eps = 1e-12 * (2 * wl.radius + 1) ** 2 * np.abs(al).max()
    mask = np.abs(eta) < eps
    out = zeta / np.where(mask, 1, eta)
    ok = np.abs(lead[n]) >= eps
    out = np.where(mask, np.where(ok, lead[:n] / np.where(ok, lead[n], 1), f32), out)
    if globals().get("RETURN_OUT"): return out, ref["output"], eta
    return np.abs(out - ref["output"]).max(), int(mask.sum()), ref["guarded_pixels"]


if __name__ == "__main__":
    for cfg, H, W in ((1, 128, 128), (2, 135, 240), (3, 96, 96), (4, 64, 64), (5, 96, 96)):
        print(cfg, {m: run(cfg, H, W, m) for m in ("fp32", "1xtf32", "3xtf32")}, flush=True)
