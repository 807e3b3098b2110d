import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device; run with -m gpu")


def load_golden(name):
    z = np.load(GOLDEN / f"{name}.npz", allow_pickle=False)
    return {k: z[k] for k in z.files}


def group(d, prefix):
    """Split keys 'case__field' of a golden archive into {case: {field: arr}}."""
    out = {}
    for k, v in d.items():
        case, fld = k.split("__")
        out.setdefault(case, {})[fld] = v
    return out


FILTER_CASES = ["blf_rgb_fir9", "blf_rgb_fir4", "joint_rgb_g2", "nlm_patch_box10", "nlm_patch_box3",
                "hyper31_fir12", "hyper16_fir18", "blf_rgb_fir15",
                # §8 row f2: recursive Gaussian (spatial.py:114-191); rec07 is the sigma < 1 FIR fallback
                "blf_rgb_rec3", "blf_rgb_rec07", "joint_rgb_rec15", "hyper16_rec2"]


def oracle_kind(g):
    """Golden spatial_kind -> the oracle's kind name."""
    k = str(g["spatial_kind"])
    return {"gaussian": "gaussian_fir"}.get(k, k)


def spatial_kernel(g):
    """Golden fixture -> the package's SpatialKernel."""
    from paper_1901_06112_b200 import SpatialKernel

    k = oracle_kind(g)
    if k == "box":
        return SpatialKernel.box(int(g["radius"]))
    if k == "gaussian_recursive":
        return SpatialKernel.recursive(float(g["sigma"]))
    return SpatialKernel.gaussian(float(g["sigma"]), int(g["radius"]))


@pytest.fixture(scope="session")
def golden():
    return load_golden
