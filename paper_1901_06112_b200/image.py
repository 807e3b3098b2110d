"""Planar image containers (mirror of reference ``image.py:33-112``).

``Image.data`` is channel-planar ``(channels, height, width)``: sample
(c, x, y) is ``data[c, y, x]`` and the flat sample index is
``c*w*h + y*w + x`` (image.py:66-69).  The reference stores float64 NumPy;
this drop-in additionally accepts a CUDA ``torch.Tensor`` so a caller can
keep images resident in HBM end to end.  NumPy inputs keep the reference's
float64 read-only semantics; device tensors are used as float32.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

try:  # torch is plumbing for device memory / streams only
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None


def _is_tensor(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor)


@dataclass(frozen=True)
class Image:
    """Immutable planar raster; ``data[c, y, x]`` (image.py:33-72)."""

    data: object
    range_max: float = 255.0

    def __post_init__(self) -> None:
        if _is_tensor(self.data):
            t = self.data
            if t.dim() == 2:
                t = t.unsqueeze(0)
            if t.dim() != 3 or t.numel() == 0:
                raise ValueError("image data must be a non-empty (channels, height, width) array")
            t = t.contiguous()
            object.__setattr__(self, "data", t)
        else:
            arr = np.asarray(self.data, dtype=np.float64)
            if arr.ndim == 2:
                arr = arr[np.newaxis, :, :]
            if arr.ndim != 3 or arr.size == 0:
                raise ValueError("image data must be a non-empty (channels, height, width) array")
            if not np.all(np.isfinite(arr)):
                raise ValueError("image samples must be finite")
            arr = np.ascontiguousarray(arr)
            arr.flags.writeable = False
            object.__setattr__(self, "data", arr)
        if not self.range_max > 0:
            raise ValueError("range_max must be positive")

    @property
    def on_device(self) -> bool:
        return _is_tensor(self.data) and self.data.is_cuda

    @property
    def is_tensor(self) -> bool:
        return _is_tensor(self.data)

    @property
    def channels(self) -> int:
        return int(self.data.shape[0])

    @property
    def height(self) -> int:
        return int(self.data.shape[1])

    @property
    def width(self) -> int:
        return int(self.data.shape[2])

    @property
    def samples(self):
        """Flat planar sample vector: samples[c*w*h + y*w + x] = data[c, y, x]."""
        return self.data.reshape(-1)

    def plane(self, c: int):
        return self.data[c]

    def numpy(self) -> np.ndarray:
        if self.is_tensor:
            return self.data.detach().to("cpu", torch.float64).numpy()
        return self.data


@dataclass(frozen=True)
class RangeList:
    """All guide vectors in pixel order plus the identity index map
    (image.py:75-105)."""

    vectors: np.ndarray
    index_map: np.ndarray

    def __post_init__(self) -> None:
        vec = np.ascontiguousarray(np.asarray(self.vectors, dtype=np.float64))
        idx = np.ascontiguousarray(np.asarray(self.index_map, dtype=np.int64))
        if vec.ndim != 2 or vec.shape[0] == 0:
            raise ValueError("range list must be a non-empty (m, dim) matrix")
        if idx.shape != (vec.shape[0],):
            raise ValueError("index map length must equal the number of vectors")
        vec.flags.writeable = False
        idx.flags.writeable = False
        object.__setattr__(self, "vectors", vec)
        object.__setattr__(self, "index_map", idx)

    @property
    def m(self) -> int:
        return self.vectors.shape[0]

    @property
    def dim(self) -> int:
        return self.vectors.shape[1]


def extract_range_list(guide: Image) -> RangeList:
    """Every guide vector, duplicates kept, linear pixel order (image.py:108-112).

    The B200 path never builds this (its kernels read the planar guide in
    place); it is kept for API parity.
    """
    data = guide.numpy()
    m = guide.width * guide.height
    return RangeList(vectors=data.reshape(guide.channels, m).T.copy(),
                     index_map=np.arange(m, dtype=np.int64))
