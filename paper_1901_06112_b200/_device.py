"""Device plumbing: torch owns HBM allocations and streams, the C ABI gets raw
pointers.  No compute happens here."""

from __future__ import annotations

import numpy as np
import torch


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the Nystrom B200 path needs a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return int(torch.cuda.current_stream().cuda_stream)


def to_device_f32(x) -> torch.Tensor:
    """Planar float32 contiguous CUDA tensor from numpy or torch input."""
    dev = require_cuda()
    if isinstance(x, torch.Tensor):
        if not x.is_cuda and x.dtype == torch.float32 and x.is_pinned():
            return x.to(device=dev, non_blocking=True).contiguous()
        return x.to(device=dev, dtype=torch.float32).contiguous()
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    return torch.from_numpy(arr).to(dev, non_blocking=False)


def workspace(nbytes: int) -> torch.Tensor:
    dev = require_cuda()
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=dev)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else int(t.data_ptr())


class StageTimer:
    """CUDA-event stamps on the current stream (FilterReport.timings)."""

    def __init__(self):
        self.events: list[tuple[str, torch.cuda.Event]] = []

    def mark(self, name: str) -> None:
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.events.append((name, ev))

    def elapsed(self) -> dict[str, float]:
        if not self.events:
            return {}
        self.events[-1][1].synchronize()
        out = {}
        for (_, a), (name, b) in zip(self.events, self.events[1:]):
            out[name] = a.elapsed_time(b) / 1e3
        return out
