"""Device plumbing: torch owns HBM allocations and streams, the C ABI gets raw
pointers.  No compute happens here."""

from __future__ import annotations

import threading
import warnings

import numpy as np
import torch


_CUDA_OK = False
STAMPS: list | None = None  # tools/step_overhead.py: (label, perf_counter) pairs on the host path


def stamp(label: str) -> None:
    if STAMPS is not None:
        import time

        STAMPS.append((label, time.perf_counter()))


def require_cuda() -> torch.device:
    global _CUDA_OK
    if not _CUDA_OK:
        if not torch.cuda.is_available():
            raise RuntimeError("the Nystrom B200 path needs a CUDA device (there is no CPU fallback)")
        _CUDA_OK = True
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    """cudaStream_t of the current stream (the raw query skips building a Stream object:
    this sits on the per-call critical path before the first launch)."""
    return int(torch._C._cuda_getCurrentRawStream(torch.cuda.current_device()))


_STREAMS: dict = {}


def current_stream_cached() -> torch.cuda.Stream:
    """torch's current Stream object, cached by its raw cudaStream_t (building one costs ~4 us)."""
    raw = stream_ptr()
    st = _STREAMS.get(raw)
    if st is None:
        st = torch.cuda.current_stream()
        if len(_STREAMS) > 64:
            _STREAMS.clear()
        _STREAMS[raw] = st
    return st


_TLS = threading.local()


_POOL = None


def _parallel_copy(dst: np.ndarray, src: np.ndarray, chunk: int = 4 << 20) -> None:
    """dst[:] = src for large host arrays, in ~4 MB slices on a thread pool (NumPy releases the
    GIL for the copies): one thread's memcpy bandwidth would dominate a 1080p float64 upload."""
    global _POOL
    n = src.size
    nb = n * src.itemsize
    if nb <= 2 * chunk:
        np.copyto(dst, src, casting="same_kind")
        return
    if _POOL is None:
        import concurrent.futures as cf
        import os

        _POOL = cf.ThreadPoolExecutor(max_workers=max(2, min(16, (os.cpu_count() or 2))))
    step = max(1, chunk // src.itemsize)
    futs = [_POOL.submit(np.copyto, dst[i:i + step], src[i:i + step], "same_kind") for i in range(0, n, step)]
    for fu in futs:
        fu.result()


def _staged_upload(arr: np.ndarray, dev) -> torch.Tensor:
    """H2D of a host ndarray through a page-locked float32 staging buffer reused per host thread:
    a multi-threaded host copy into it -- which also rounds a float64 array (the reference's
    Image dtype) to the float32 the kernels compute in, so half the bytes cross PCIe and no cast
    runs on the device -- then one DMA at full PCIe speed (a pageable copy runs at a fraction of
    it).  The buffer is reused once its previous DMA is done."""
    cache = getattr(_TLS, "staging", None)
    if cache is None:
        cache = _TLS.staging = {}
    key = ("f4", arr.size)
    ent = cache.get(key)
    if ent is None:
        buf = torch.empty(arr.shape, dtype=torch.float32, pin_memory=True)
        ent = cache[key] = [buf, None]
    buf, done = ent
    if done is not None:
        done.synchronize()  # the previous upload from this buffer has left it
    buf = buf.view(arr.shape)
    _parallel_copy(buf.numpy().reshape(-1), arr.reshape(-1))
    t = buf.to(dev, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record()
    ent[1] = ev
    return t


def to_device_f32(x) -> torch.Tensor:
    """Planar float32 contiguous CUDA tensor from numpy or torch input.  A float64 ndarray
    (the reference's Image dtype) is rounded to float32 on its way into the staging buffer."""
    dev = require_cuda()
    if isinstance(x, torch.Tensor):
        if x.is_cuda and x.dtype == torch.float32 and x.device == dev and x.is_contiguous():
            return x
        if not x.is_cuda and x.dtype == torch.float32 and x.is_pinned():
            return x.to(device=dev, non_blocking=True).contiguous()
        return x.to(device=dev, dtype=torch.float32).contiguous()
    arr = np.ascontiguousarray(x)
    if arr.dtype not in (np.float32, np.float64):
        arr = arr.astype(np.float64)
    return _staged_upload(arr, dev)


def workspace(nbytes: int) -> torch.Tensor:
    dev = require_cuda()
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=dev)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else int(t.data_ptr())


class StageTimer:
    """CUDA-event stamps on the current stream (FilterReport.timings)."""

    def __init__(self):
        self.events: list[tuple[str, torch.cuda.Event]] = []
        self.stream = current_stream_cached()  # Event.record() would build a Stream object per stamp

    def mark(self, name: str) -> None:
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(self.stream)
        self.events.append((name, ev))

    def lazy(self, fill) -> "LazyTimings":
        """FilterReport.timings resolved on first read (the event queries cost ~50 us,
        which would otherwise sit inside every call after its last kernel)."""
        return LazyTimings(self, fill)

    def elapsed(self) -> dict[str, float]:
        if not self.events:
            return {}
        self.events[-1][1].synchronize()
        out = {}
        for (_, a), (name, b) in zip(self.events, self.events[1:]):
            out[name] = a.elapsed_time(b) / 1e3
        return out


class LazyTimings(dict):
    """A dict of stage seconds computed from a StageTimer on first access."""

    def __init__(self, timer: StageTimer, fill):
        super().__init__()
        self._timer, self._fill = timer, fill

    def _resolve(self):
        if self._timer is not None:
            t, self._timer = self._timer, None
            dict.update(self, self._fill(t.elapsed()))

    def __getitem__(self, k):
        self._resolve()
        return dict.__getitem__(self, k)

    def __iter__(self):
        self._resolve()
        return dict.__iter__(self)

    def __len__(self):
        self._resolve()
        return dict.__len__(self)

    def __contains__(self, k):
        self._resolve()
        return dict.__contains__(self, k)

    def __repr__(self):
        self._resolve()
        return dict.__repr__(self)

    def __eq__(self, other):
        self._resolve()
        return dict.__eq__(self, other)

    def get(self, k, default=None):
        self._resolve()
        return dict.get(self, k, default)

    def keys(self):
        self._resolve()
        return dict.keys(self)

    def values(self):
        self._resolve()
        return dict.values(self)

    def items(self):
        self._resolve()
        return dict.items(self)

    def copy(self):
        self._resolve()
        return dict(self)
