"""Benchmark: filtered megapixels/sec of the Nystrom kernel filter on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

One step = the whole hot path (BASELINE.json north_star) over one synthetic
image: k-means++ seeding + Lloyd (K0/K1), host FP64 eig of the m0 x m0
landmark kernel, features + horizontal pass (K2), vertical pass +
reconstruction + guard + division (K3).  Default workload: BASELINE.json
configs[1] (cfg 2, 1920x1080x3, m0=64, sigma_s=5/R=15, sigma_r=0.1, 15 it).

Prints ONE JSON line (rank 0).  ``value`` = Mpix/s with the input resident in
HBM (output stays in HBM); ``e2e`` = the same through the public API from
pinned host buffers with H2D/D2H inside the timed region.  L2 (126 MB) is
flushed with a 512 MB write before every timed step.  ``--impl reference``
times the CPU oracle port (oracle/nys_oracle.py; the reference is pure
Python and cannot travel to the GPU box) on a bounded row crop of the same
workload, its convolution stage on one thread like the reference's
(BLAS matmuls on the BLAS threads).
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_1901_06112_b200.synthetic import CONFIGS  # noqa: E402

METRIC = "filtered megapixels/sec (d-channel, m landmarks)"
UNIT = "Mpix/s"


def _cfg_dict(wl, extra=None):
    d = {"workload": wl.name, "H": wl.H, "W": wl.W, "channels": wl.channels, "guide": wl.mode,
         "m0": wl.m0, "spatial": wl.spatial, "sigma_s": wl.sigma, "radius": wl.radius,
         "sigma_r": round(float(wl.theta), 6), "kmeans_iters": wl.max_iter, "seed": 0}
    if extra:
        d.update(extra)
    return d


def _params(wl):
    from paper_1901_06112_b200 import FilterParams, SpatialKernel

    sk = SpatialKernel.box(wl.radius) if wl.spatial == "box" else SpatialKernel.gaussian(wl.sigma, wl.radius)
    return FilterParams(spatial=sk, theta=float(wl.theta), m0=wl.m0, seed=0, kmeans_max_iter=wl.max_iter,
                        mode=wl.mode if wl.mode != "nlm" else "nlm", patch_radius=max(wl.patch_radius, 1),
                        pca_dim=27 if wl.mode == "nlm" else 25)


def _guide(f_img, wl):
    from paper_1901_06112_b200 import PatchGuide

    return PatchGuide(f_img, wl.patch_radius) if wl.mode == "nlm" else f_img


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region.

    NVML (nvidia_ml_py) polled from a thread every ``period`` s: the timed
    region is tens of ms, too short for ``nvidia-smi -lms`` to start up."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int, period: float = 0.002):
        self.index = index
        self.period = period
        self.samples: list[tuple[float, int]] = []
        self.window = False  # set around the timed steps (the thread starts before the warm-up)
        self.max_mhz = None
        self._stop = threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            # the first call of each query initialises NVML state lazily: do it here, before the
            # timed steps, so the sampler thread only issues warm queries during them
            pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:  # pragma: no cover - no NVML
            self.t = None
        return self

    def _run(self):
        nv, h = self.nv, self.h
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                if self.window:  # only samples taken during the timed steps count
                    self.samples.append((float(sm), int(rs)))
            except Exception:  # pragma: no cover
                pass
            self._stop.wait(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        sm = [s for s, _ in self.samples]
        reasons = sorted({nm for _, r in self.samples for nm, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(sm), "source": "NVML, 2 ms polling during the timed steps"}


def _ffma_peak():
    p = ROOT / "profiles" / "ffma_peak.json"
    if p.exists():
        return json.loads(p.read_text())
    return None


def run_ours(args, rank: int, world: int):
    import torch

    from paper_1901_06112_b200 import Image, _native, fast_filter

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    dev = torch.device("cuda", torch.cuda.current_device())
    wl = CONFIGS[args.config]
    # N > 1: the frame is the data-parallel unit -- every rank filters its own image of the
    # workload (weak scaling, no collective on the data path; the max over ranks of each step's
    # device time is the step time).  An image too large for one GPU (cfg 5), or --sharded, runs
    # the row-band-sharded path instead (halo exchange + NCCL k-means, parallel.py).
    if args.sharded or (world > 1 and wl.pixels > 16 * 1024 * 1024):
        from paper_1901_06112_b200 import parallel

        return parallel.bench_sharded(args, wl, rank, world)
    import torch.distributed as dist

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        if world > 1:
            dist.barrier()

    f_np = wl.image(seed=0)
    n, H, W = f_np.shape
    px = H * W
    f_dev = torch.from_numpy(f_np).to(dev)
    f_img = Image(data=f_dev, range_max=1.0)
    g_img = _guide(f_img, wl)
    params = _params(wl)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def l2_flush():
        flush.random_(0, 255)  # 512 MB write > 126 MB L2

    # the clock sampler's thread starts before the warm-up (its first NVML queries stalled the
    # step they landed in); only its samples inside the timed window are kept
    clk = ClockSampler(torch.cuda.current_device()).__enter__()
    # warm-up (also JIT-free: the library is prebuilt)
    for _ in range(args.warmup):
        fast_filter(f_img, g_img, params)
    torch.cuda.synchronize()
    # move the startup heap (torch, numpy, the library) out of the collector's reach, as a
    # long-running server process would
    gc.collect()
    gc.freeze()

    lib = _native.lib()
    step_ms, k_ms = [], {"k_feat_hpass": 0.0, "k_vpass": 0.0}
    k_n = {"k_feat_hpass": 0, "k_vpass": 0}
    k_px = {"k_feat_hpass": 0, "k_vpass": 0}  # output pixels the timed launches produced (per band)
    launches0 = int(lib.nys_kernel_launches())
    try:
        torch.cuda.synchronize()
        clk.window = True
        for _ in range(args.steps):
            l2_flush()
            barrier()
            torch.cuda.synchronize()
            evs = []
            rep = None  # the previous step's report is released here, outside the timed window
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            rep = fast_filter(f_img, g_img, params, kernel_events=evs)
            e1.record()
            torch.cuda.synchronize()
            step_ms.append(max_over_ranks(e0.elapsed_time(e1)))
            for name, a, b, band in evs:
                k_ms[name] += a.elapsed_time(b)
                k_n[name] += 1
                k_px[name] += (band.out_rows if band is not None else H) * W
        torch.cuda.synchronize()
        clk.window = False
    finally:
        clk.__exit__(None, None, None)
    launches = int(lib.nys_kernel_launches()) - launches0
    ms = sum(step_ms) / len(step_ms)
    value = world * px / (ms * 1e-3) / 1e6  # every rank filtered one image per step

    # end to end through the public API from pinned host buffers
    f_host = torch.from_numpy(f_np).pin_memory()
    h_img = Image(data=f_host, range_max=1.0)
    hg = _guide(h_img, wl)
    h_out = torch.empty(f_host.shape, dtype=torch.float32, pin_memory=True)  # reused pinned output
    fast_filter(h_img, hg, params, out=h_out)
    e2e_ms = []
    torch.cuda.synchronize()
    rep_h = None
    for _ in range(max(1, args.steps)):
        l2_flush()
        barrier()
        torch.cuda.synchronize()
        rep_h = None  # previous report released outside the timed window
        t0 = time.perf_counter()
        rep_h = fast_filter(h_img, hg, params, out=h_out)
        torch.cuda.synchronize()
        e2e_ms.append(max_over_ranks((time.perf_counter() - t0) * 1e3))
    e2e = sum(e2e_ms) / len(e2e_ms)
    out_bytes = int(rep_h.output.data.numel() * 4)

    # end to end through the reference's own data type (image.py:33-52): a NumPy float64 Image in,
    # a NumPy float64 Image out (uploaded through a reused page-locked staging buffer and cast on
    # the device; K3 writes the float64 planes straight into page-locked host memory)
    f64 = f_np.astype(np.float64)
    n_img = Image(data=f64, range_max=1.0)
    ng = _guide(n_img, wl)
    fast_filter(n_img, ng, params)
    e2e_np_ms = []
    rep_n = None
    for _ in range(max(1, args.steps)):
        l2_flush()
        barrier()
        torch.cuda.synchronize()
        rep_n = None
        t0 = time.perf_counter()
        rep_n = fast_filter(n_img, ng, params)
        e2e_np_ms.append(max_over_ranks((time.perf_counter() - t0) * 1e3))
    assert isinstance(rep_n.output.data, np.ndarray) and rep_n.output.data.dtype == np.float64
    e2e_np = sum(e2e_np_ms) / len(e2e_np_ms)

    # roofline of the dominant kernel: algorithmic bytes of the pixels each launch produced (its
    # band's out_rows x W) / that launch's time, averaged over launches
    u = n if wl.mode != "nlm" else n  # stored input channels read (patches gathered from f)
    P = (wl.m0 + 1) * (n + 1)         # planes incl. the rank-1 lead group
    T = 2 * wl.radius + 1
    rho = n * 9 if wl.mode == "nlm" else n
    bytes_px = {"k_feat_hpass": 4 * (u + P), "k_vpass": 4 * (P + u + n)}
    # algorithmic CUDA-core FP32 ops per pixel (FIR taps, features, contraction); y = M b runs on
    # the tensor cores (3xTF32 tcgen05) and is reported apart
    fir = P * (2 if wl.spatial == "box" else T)
    flops_px = {"k_feat_hpass": fir + wl.m0 * (2 * rho + 1) + wl.m0 * n,
                "k_vpass": fir + wl.m0 * (2 * rho + 1) + 2 * P}
    tensor_mac_px = {"k_feat_hpass": 3 * wl.m0 * (wl.m0 + 1), "k_vpass": 0}
    avg = {k: k_ms[k] / max(1, k_n[k]) for k in k_ms}
    px_launch = {k: k_px[k] / max(1, k_n[k]) for k in k_px}
    dom = max(avg, key=avg.get)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = bytes_px[dom] * px_launch[dom] / (avg[dom] * 1e-3) / 1e9
    ffma = _ffma_peak()
    roof = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
            "frac": round(achieved / hbm_peak, 4), "traffic": None,
            "peak_source": "MEASURED_PEAKS.json" if peaks else "fallback",
            "bytes_per_px": bytes_px[dom], "px_per_launch": int(px_launch[dom]), "launch_ms": round(avg[dom], 4),
            "launches_per_step": k_n[dom] // max(1, args.steps),
            "kernel_ms": {k: round(v, 4) for k, v in avg.items()},
            "kernel_frac_hbm": {k: round(bytes_px[k] * px_launch[k] / (avg[k] * 1e-3) / 1e9 / hbm_peak, 4)
                                for k in avg if avg[k] > 0}}
    fma_t = flops_px[dom] * px_launch[dom] / (avg[dom] * 1e-3) / 1e12
    roof["fma"] = {"achieved_tfma": round(fma_t, 2), "ops_per_px": flops_px[dom],
                   "peak_tfma": ffma.get("tfma_per_s") if ffma else None,
                   "frac": round(fma_t / ffma["tfma_per_s"], 4) if ffma else None,
                   "counts": "CUDA-core FP32 FMA/ADD of the FIR taps, features and contraction"}
    if tensor_mac_px[dom]:
        tm = tensor_mac_px[dom] * px_launch[dom] / (avg[dom] * 1e-3) / 1e12
        roof["tensor"] = {"achieved_tmac": round(tm, 3), "macs_per_px": tensor_mac_px[dom],
                          "what": "y = M b as 3xTF32 tcgen05.mma (3 passes of m0 x (m0+1) MACs)"}
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists():
        tr = json.loads(prof.read_text()).get(wl.name, {}).get(dom)
        if tr:  # DRAM bytes per launch from one ncu --set full capture (vs bytes_per_px * px algorithmic)
            roof["traffic"] = tr["dram_bytes_per_launch"]
            roof["traffic_algorithmic_bytes"] = bytes_px[dom] * px
            roof["traffic_source"] = tr["source"]
    result = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded random-polygon scene, SURVEY §8d)",
        "config": _cfg_dict(wl, {"l2": "flushed: 512 MB write before every timed step",
                                 "parallelism": "single" if world == 1 else f"dp{world}: one image per rank, no collective"}),
        "e2e": {"value": round(world * px / (e2e * 1e-3) / 1e6, 2), "unit": UNIT, "ms_per_step": round(e2e, 3),
                "h2d_bytes_per_step": int(f_np.nbytes), "d2h_bytes_per_step": out_bytes,
                "path": "fast_filter(Image(pinned host float32), out=pinned host buffer): H2D copy in, K3 writes the output over PCIe"},
        "e2e_reference_types": {"value": round(world * px / (e2e_np * 1e-3) / 1e6, 2), "unit": UNIT,
                                "ms_per_step": round(e2e_np, 3), "h2d_bytes_per_step": int(f64.nbytes) // 2,
                                "d2h_bytes_per_step": int(f64.nbytes),
                                "path": "fast_filter(Image(numpy float64)) -> Image(numpy float64), the reference's "
                                        "call and types (image.py:33-52, filters.py:199); the float64 input is "
                                        "rounded to float32 into the page-locked staging buffer (half the bytes "
                                        "cross PCIe), the float64 output comes back in one DMA"},
        "step_ms": [round(x, 3) for x in step_ms],
        "gpu_launches": launches // max(1, args.steps),
        "gpu_launches_total": launches,
        "roofline": roof,
        "stage_ms": {k: round(v * 1e3, 3) for k, v in rep.timings.items()},
        "clocks": clk.summary(),
        "report": {"retained_rank": rep.retained_rank, "quant_error": rep.quant_error,
                   "guarded_pixels": rep.guarded_pixels, "min_denominator": rep.min_denominator},
    }
    if not args.no_cpu_baseline and world == 1:  # the CPU baseline is timed at N = 1 only
        result["cpu_baseline"] = cpu_baseline(wl, args.cpu_rows)
    return result


def _blas_threads():
    try:
        from threadpoolctl import threadpool_info

        info = threadpool_info()
        return max([i.get("num_threads", 1) for i in info] or [1])
    except Exception:  # pragma: no cover
        return os.cpu_count() or 1


def cpu_baseline(wl, rows: int, threads: int = 1):
    """CPU oracle port on a bounded row crop of the same workload.  threads = 1 runs the rank
    loop (filters.py:227-238) on one thread, as the reference's NumPy convolution stage does;
    the k-means / extrapolation matmuls use the BLAS threads, as in the reference."""
    from oracle import nys_oracle as O

    f = wl.image(seed=0, H=rows).astype(np.float64)
    p = O.patch_stack(f, wl.patch_radius) if wl.mode == "nlm" else f
    t0 = time.perf_counter()
    O.fast_filter(f, p, float(wl.theta), wl.spatial, wl.sigma, wl.radius, wl.m0, 0, wl.max_iter, threads=threads)
    dt = time.perf_counter() - t0
    px = f.shape[1] * f.shape[2]
    return {"value": round(px / dt / 1e6, 5), "unit": UNIT, "cores": max(threads, _blas_threads()),
            "kind": "port", "seconds": round(dt, 2), "host_cpus": os.cpu_count(),
            "sample": f"oracle/nys_oracle.fast_filter (FP64 NumPy restatement of the reference) on the first "
                      f"{rows} rows x {wl.W} cols of {wl.name}, k-means on that crop; rank loop (the "
                      f"convolutions) on {threads} thread{'s' if threads > 1 else ''} as in the reference, "
                      f"BLAS matmuls on {_blas_threads()}"}


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return None
    wl = CONFIGS[args.config]
    threads = 1  # the reference's convolution stage is single-threaded NumPy (spatial.py:102-109)
    rows = args.ref_rows
    for _ in range(args.warmup):
        cpu_baseline(wl, max(8, rows // 4), threads)
    vals, secs = [], []
    for _ in range(args.steps):
        r = cpu_baseline(wl, rows, threads)
        vals.append(r["value"])
        secs.append(r["seconds"])
    value = sum(vals) / len(vals)
    r["value"] = round(value, 5)
    return {"impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * sum(secs) / len(secs), 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded random-polygon scene, SURVEY §8d)",
            "config": _cfg_dict(wl, {"sample_rows": rows}),
            "cpu_baseline": r,
            "e2e": {"value": round(value, 5), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-rows", type=int, default=128, help="rows of the CPU-baseline crop")
    ap.add_argument("--ref-rows", type=int, default=64, help="rows of the reference-arm crop per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="run the row-sharded NCCL path even at one rank (exercises parallel.py on one GPU)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.sharded and world == 1:  # a one-rank NCCL group without torchrun
        for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29517"), ("RANK", "0"), ("WORLD_SIZE", "1")):
            os.environ.setdefault(k, v)
    if (world > 1 or args.sharded) and args.impl == "ours":
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    if args.impl == "reference":
        res = run_reference(args, rank, world)
    else:
        res = run_ours(args, rank, world)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
