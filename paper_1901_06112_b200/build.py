"""Build the sm_100a native library in-tree: ``_lib/libnysfilter_b200.so``.

Plain ``nvcc`` (no torch extension machinery): the library is a C ABI
(``include/nysfilter_b200.h``) loaded with ctypes, statically linked against
the CUDA runtime so it travels to the GPU box as one file.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "libnysfilter_b200.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["nys_filter.cu", "nys_hpass.cu", "nys_hpass_tc.cu", "nys_vpass.cu", "nys_refine.cu", "nys_kmeans.cu", "nys_kmeans_coop.cu", "nys_recursive.cu", "nys_brute.cu", "nys_metrics.cu", "nys_pca.cu", "nys_spatial.cu",
           "nys_host.cpp"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*")) + [ROOT / "include" / "nysfilter_b200.h"]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    nvcc = _nvcc()
    OUT_DIR.mkdir(exist_ok=True)
    objs = []
    cmds = []
    # incremental: a source recompiles when it, or any shared header, is newer than its object
    hdr_t = max(p.stat().st_mtime for p in [*CSRC.glob("*.cuh"), *CSRC.glob("*.h"), ROOT / "include" / "nysfilter_b200.h"])
    for src in SOURCES:
        obj = OUT_DIR / (Path(src).stem + ".o")
        objs.append(obj)
        if not force and obj.exists() and obj.stat().st_mtime > max(hdr_t, (CSRC / src).stat().st_mtime):
            continue
        if src.endswith(".cu"):
            cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                   "-Xptxas", "-v" if verbose else "-O3", "-c", str(CSRC / src), "-o", str(obj)]
        else:
            cmd = ["g++", "-O3", "-std=c++17", "-ffp-contract=off", "-fPIC", "-c", str(CSRC / src), "-o", str(obj)]
        cmds.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r.stdout + r.stderr

    with cf.ThreadPoolExecutor(max_workers=max(1, len(cmds))) as ex:
        logs = list(ex.map(run, cmds))
    if verbose:
        for log in logs:
            sys.stderr.write(log)
    tmp = LIB.with_suffix(".so.tmp")
    run([nvcc, *ARCH, "-shared", "-cudart", "static", *map(str, objs), "-o", str(tmp)])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
