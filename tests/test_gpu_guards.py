"""Out-of-bounds write checks for the hot-path kernels (compute-sanitizer is not
available on this pool): every buffer the C ABI writes -- the plane buffer, the
output planes, the filter workspace, the k-means workspace and outputs -- is
placed between guard regions filled with a sentinel, the kernels run on odd
shapes (W not a multiple of 32, two row bands, a partial plane chunk, the NLM
patch guide, queued near-guard pixels), and the guards must come back
untouched.  The outputs are also checked against the oracle."""

import ctypes as C

import numpy as np
import pytest
import torch

from oracle import nys_oracle as O
from paper_1901_06112_b200 import SpatialKernel, _native
from paper_1901_06112_b200._device import ptr, stream_ptr
from paper_1901_06112_b200.filters import _desc
from paper_1901_06112_b200.nystrom import mixing_plan
from paper_1901_06112_b200.synthetic import color_scene

pytestmark = pytest.mark.gpu

GUARD = 4096  # floats on each side
SENT = -12345.678


class Guarded:
    """A float32 device buffer of `n` floats between two sentinel guards."""

    def __init__(self, n, fill=None):
        self.n = int(n)
        self.buf = torch.full((self.n + 2 * GUARD,), SENT, dtype=torch.float32, device="cuda")
        self.t = self.buf[GUARD:GUARD + self.n]
        if fill is not None:
            self.t.copy_(torch.as_tensor(np.ascontiguousarray(fill, np.float32).ravel()))

    @property
    def p(self):
        return ptr(self.t)

    def intact(self):
        torch.cuda.synchronize()
        return bool((self.buf[:GUARD] == SENT).all() and (self.buf[GUARD + self.n:] == SENT).all())


@pytest.mark.parametrize("case", ["blf_fir", "nlm_box", "two_channel"])
def test_filter_kernels_write_inside_their_buffers(case):
    lib = _native.lib()
    H, W = 37, 70
    if case == "blf_fir":
        f32 = color_scene(H, W, 6, 0.05, seed=5)
        sk, theta, m0, gkind = SpatialKernel.gaussian(2.0, 6), 0.15, 12, 0
    elif case == "nlm_box":
        f32 = color_scene(H, W, 5, 0.08, seed=6, lo=0.1, hi=0.9, shading=0.1)
        sk, theta, m0, gkind = SpatialKernel.box(4), 0.06, 10, 1
    else:
        f32 = np.ascontiguousarray(color_scene(H, W, 5, 0.05, seed=7)[:2])
        sk, theta, m0, gkind = SpatialKernel.gaussian(1.5, 5), 0.2, 9, 0
    n = f32.shape[0]
    f64 = f32.astype(np.float64)
    p64 = O.patch_stack(f64, 1) if gkind == 1 else f64
    rho = p64.shape[0]
    Cn, _, _, _ = O.kmeans(O.range_vectors(p64), m0, 0, 6)
    S = sk.effective_radius()
    plan = mixing_plan(Cn, theta, 1e-8, S, lite=True, device_inverse=True)
    keep = []
    d = _desc(n, rho, H, W, gkind, sk, theta, Cn, plan, keep)
    f = Guarded(n * H * W, f32)
    g = f if gkind == 1 else Guarded(rho * H * W, p64.astype(np.float32))
    wsb = int(lib.nys_filter_workspace_bytes(C.byref(d)))
    ws = Guarded((wsb + 3) // 4)
    ws.t.zero_()
    rs = int(lib.nys_filter_plane_row_stride(C.byref(d)))
    out = Guarded(n * H * W)
    stats = torch.zeros(2, dtype=torch.float64, device="cuda")
    s = stream_ptr()
    _native.check(lib.nys_filter_prepare(C.byref(d), ws.p, wsb, s), "prepare")
    R = d.radius
    for out0, rows in ((0, 20), (20, H - 20)):  # two bands
        planes = Guarded((rows + 2 * R) * rs)
        _native.check(lib.nys_filter_hpass(C.byref(d), f.p, H * W, g.p, H * W, out0, rows, planes.p, rs, ws.p, s),
                      "hpass")
        _native.check(lib.nys_filter_vpass(C.byref(d), f.p, H * W, g.p, H * W, planes.p, rs, out0, rows, out.p, H * W,
                                           ws.p, s), "vpass")
        assert planes.intact(), "plane buffer guard overwritten"
    _native.check(lib.nys_filter_finish(C.byref(d), f.p, H * W, g.p, H * W, out.p, H * W, ws.p, ptr(stats), s), "finish")
    for b, nm in ((f, "input"), (out, "output"), (ws, "workspace")):
        assert b.intact(), f"{nm} guard overwritten"
    if gkind == 0:
        assert g.intact()
    kind = "box" if sk.kind == "box" else "gaussian_fir"
    ref = O.fast_filter_with_landmarks(f64, p64, Cn, theta, kind, sk.sigma, sk.radius)
    got = out.t.reshape(n, H, W).double().cpu().numpy()
    assert np.abs(got - ref["output"]).max() <= 1e-4
    assert int(stats[1:].view(torch.int64)[0]) == ref["guarded_pixels"]


def test_kmeans_writes_inside_its_buffers():
    lib = _native.lib()
    rng = np.random.default_rng(3)
    m, rho, m0, it = 3001, 5, 13, 8
    pts = Guarded(rho * m, rng.random((rho, m)))
    wsb = int(lib.nys_kmeans_workspace_bytes(m, rho, m0))
    ws = Guarded((wsb + 3) // 4)
    Cd = Guarded(2 * m0 * rho)
    errs = Guarded(2 * it)
    stats = Guarded(2 * 4)
    qe = Guarded(2)
    asg = Guarded(2 * m)
    seeds = Guarded(2 * m0)
    g = np.random.default_rng(0)
    first = int(g.integers(m))
    unif = np.array([g.random() for _ in range(m0 - 1)], np.float64)
    _native.check(lib.nys_kmeans_run(pts.p, m, m, rho, m0, it, first, unif.ctypes.data, Cd.p, errs.p, stats.p, qe.p,
                                     asg.p, seeds.p, ws.p, wsb, stream_ptr()), "nys_kmeans_run")
    for b, nm in ((pts, "points"), (ws, "workspace"), (Cd, "centroids"), (errs, "errors"), (stats, "stats"),
                  (qe, "quant_error"), (asg, "assignment"), (seeds, "seeds")):
        assert b.intact(), f"{nm} guard overwritten"
    Cref, lab, qref, _ = O.kmeans(pts.t.reshape(rho, m).double().cpu().numpy().T, m0, 0, it)
    np.testing.assert_allclose(Cd.t.view(torch.float64).reshape(m0, rho).cpu().numpy(), Cref, rtol=0, atol=1e-9)
    assert float(qe.t.view(torch.float64)[0]) == pytest.approx(qref, rel=1e-9)
