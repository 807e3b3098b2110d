"""Planar image containers (mirror of reference ``image.py:33-112``).

``Image.data`` is channel-planar ``(channels, height, width)``: sample
(c, x, y) is ``data[c, y, x]`` and the flat sample index is
``c*w*h + y*w + x`` (image.py:66-69).  The reference stores float64 NumPy;
this drop-in additionally accepts a CUDA ``torch.Tensor`` so a caller can
keep images resident in HBM end to end.  NumPy inputs keep the reference's
float64 read-only semantics; device tensors are used as float32.
"""

from __future__ import annotations

import struct
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

    @classmethod
    def trusted(cls, data: np.ndarray, range_max: float) -> "Image":
        """Wrap a float64 (channels, height, width) array this package produced
        (e.g. the filter output K3 wrote into page-locked memory) without the
        constructor's copy and finiteness scan; read-only like every Image."""
        data.flags.writeable = False
        img = object.__new__(cls)
        object.__setattr__(img, "data", data)
        object.__setattr__(img, "range_max", float(range_max))
        return img

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


# --------------------------------------------------------------------------
# file I/O, §8 row f4: the KFC1 float cube only.  The reference also reads and
# writes PNG / PGM / PPM (image.py:115-241); 8-bit raster codecs are outside
# this build's scope (configs are synthetic in-memory arrays), so
# those suffixes raise ImageFormatError here.
#
# KFC1 layout (image.py:243-270): 20-byte little-endian header
#   bytes 0-3   b"KFC1"
#   bytes 4-19  uint32 width, height, bands, sample kind (0 = float32, 1 = float64)
# followed by bands*height*width samples, band-major then row-major (the
# planar data[c, y, x] order of Image).  Loaded cubes carry range_max 255.
# --------------------------------------------------------------------------
CUBE_MAGIC = b"KFC1"
_KFC1 = struct.Struct("<4sIIII")
_KFC1_SAMPLES = {0: np.dtype("<f4"), 1: np.dtype("<f8")}
_KFC1_KIND = {"float32": 0, "float64": 1}


class ImageFormatError(ValueError):
    """Unreadable, unsupported or inconsistent image file (image.py:29)."""


def quantize_u8(samples) -> np.ndarray:
    """8-bit quantisation of the reference's writers (image.py:115-117):
    clamp to [0, 255], then round half up."""
    q = np.clip(np.asarray(samples, dtype=np.float64), 0.0, 255.0)
    return np.floor(q + 0.5).astype(np.uint8)


def load_image(path) -> Image:
    """Read a KFC1 cube (image.py:120-133 restricted to the cube format)."""
    from pathlib import Path

    path = Path(path)
    blob = path.read_bytes()
    if blob[:4] != CUBE_MAGIC:
        raise ImageFormatError(f"{path.name}: not a KFC1 cube (PNG/PNM input is outside this build's scope)")
    return _decode_cube(memoryview(blob), path.name)


def save_image(img: Image, path, cube_dtype: str = "float64") -> None:
    """Write a ``.kfc`` cube with float32 or float64 samples, unrounded
    (image.py:136-152 restricted to the cube format)."""
    from pathlib import Path

    path = Path(path)
    if path.suffix.lower() != ".kfc":
        raise ImageFormatError(f"unsupported output format: {path.name!r} (only .kfc cubes are written)")
    if cube_dtype not in _KFC1_KIND:
        raise ValueError(f"cube_dtype must be 'float32' or 'float64', got {cube_dtype!r}")
    path.write_bytes(_encode_cube(img, _KFC1_KIND[cube_dtype]))


def _decode_cube(blob: memoryview, name: str) -> Image:
    if len(blob) < _KFC1.size:
        raise ImageFormatError(f"truncated cube header in {name}")
    _magic, width, height, bands, kind = _KFC1.unpack_from(blob, 0)
    sample = _KFC1_SAMPLES.get(kind)
    if sample is None:
        raise ImageFormatError(f"unknown cube sample-type flag {kind} in {name}")
    count = width * height * bands
    payload = blob[_KFC1.size:]
    if len(payload) != count * sample.itemsize:
        raise ImageFormatError(f"size mismatch in {name}: header implies {count} samples, "
                               f"found {len(payload) / sample.itemsize:g}")
    planes = np.frombuffer(payload, dtype=sample, count=count).reshape(bands, height, width)
    return Image(data=planes.astype(np.float64), range_max=255.0)


def _encode_cube(img: Image, kind: int) -> bytes:
    header = _KFC1.pack(CUBE_MAGIC, img.width, img.height, img.channels, kind)
    return header + img.numpy().astype(_KFC1_SAMPLES[kind], copy=False).tobytes(order="C")
