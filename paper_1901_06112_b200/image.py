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


# --------------------------------------------------------------------------
# file I/O (image.py:115-270): host-side byte formats, §8 row f4
# --------------------------------------------------------------------------
CUBE_MAGIC = b"KFC1"


class ImageFormatError(ValueError):
    """Unreadable, unsupported or inconsistent image file (image.py:29)."""


def quantize_u8(samples) -> np.ndarray:
    """Clamp to [0, 255], round half away from zero (image.py:115-117)."""
    return np.floor(np.clip(np.asarray(samples, np.float64), 0.0, 255.0) + 0.5).astype(np.uint8)


def load_image(path) -> Image:
    """PNG (8-bit L/RGB), binary PGM/PPM (maxval 255) or a ``KFC1`` float
    cube, chosen by the file's magic bytes; range_max 255 (image.py:120-133)."""
    from pathlib import Path

    path = Path(path)
    raw = path.read_bytes()
    if raw[:4] == CUBE_MAGIC:
        return _cube_from_bytes(raw, path.name)
    if raw[:2] in (b"P5", b"P6"):
        return _pnm_from_bytes(raw, path.name)
    return _load_png(path)


def save_image(img: Image, path, cube_dtype: str = "float64") -> None:
    """Write by suffix: .kfc raw cube (float32/float64, no rounding),
    .png / .pgm / .ppm 8-bit (image.py:136-152)."""
    from pathlib import Path

    path = Path(path)
    suffix = path.suffix.lower()
    if suffix == ".kfc":
        path.write_bytes(_cube_bytes(img, cube_dtype))
    elif suffix == ".png":
        _save_png(img, path)
    elif suffix in (".pgm", ".ppm"):
        path.write_bytes(_pnm_bytes(img, suffix))
    else:
        raise ImageFormatError(f"unsupported output format: {path.name!r}")


def _cube_from_bytes(raw: bytes, name: str) -> Image:
    # header: magic, then little-endian uint32 width, height, bands, sample flag
    if len(raw) < 20:
        raise ImageFormatError(f"truncated cube header in {name}")
    width, height, bands, flag = np.frombuffer(raw, dtype="<u4", count=4, offset=4).tolist()
    if flag not in (0, 1):
        raise ImageFormatError(f"unknown cube sample-type flag {flag} in {name}")
    dt = np.dtype("<f4") if flag == 0 else np.dtype("<f8")
    body = np.frombuffer(raw, dtype=dt, offset=20)
    if body.size != width * height * bands:
        raise ImageFormatError(f"size mismatch in {name}: header implies {width * height * bands} samples, "
                               f"found {body.size}")
    return Image(data=body.astype(np.float64).reshape(bands, height, width), range_max=255.0)


def _cube_bytes(img: Image, cube_dtype: str) -> bytes:
    if cube_dtype not in ("float32", "float64"):
        raise ValueError(f"cube_dtype must be 'float32' or 'float64', got {cube_dtype!r}")
    flag = 0 if cube_dtype == "float32" else 1
    hdr = CUBE_MAGIC + np.array([img.width, img.height, img.channels, flag], dtype="<u4").tobytes()
    return hdr + np.ascontiguousarray(img.numpy(), dtype="<f4" if flag == 0 else "<f8").tobytes()


def _pnm_from_bytes(raw: bytes, name: str) -> Image:
    fields, pos = [], 2
    while len(fields) < 3:  # width, height, maxval; '#' comments to end of line
        if pos >= len(raw):
            raise ImageFormatError(f"truncated PNM header in {name}")
        ch = raw[pos:pos + 1]
        if ch == b"#":
            pos = raw.index(b"\n", pos) + 1
        elif ch.isspace():
            pos += 1
        else:
            end = pos
            while end < len(raw) and not raw[end:end + 1].isspace():
                end += 1
            fields.append(int(raw[pos:end]))
            pos = end
    pos += 1  # the single whitespace byte after maxval
    width, height, maxval = fields
    if maxval != 255:
        raise ImageFormatError(f"unsupported bit depth in {name}: maxval {maxval}")
    ch = 1 if raw[:2] == b"P5" else 3
    px = np.frombuffer(raw, dtype=np.uint8, offset=pos)
    if px.size != width * height * ch:
        raise ImageFormatError(f"size mismatch in {name}: header implies {width * height * ch} samples, "
                               f"found {px.size}")
    data = px.reshape(1, height, width) if ch == 1 else np.moveaxis(px.reshape(height, width, 3), 2, 0)
    return Image(data=data.astype(np.float64), range_max=255.0)


def _pnm_bytes(img: Image, suffix: str) -> bytes:
    q = quantize_u8(img.numpy())
    if suffix == ".pgm":
        if img.channels != 1:
            raise ImageFormatError("PGM requires a single-channel image")
        magic, body = b"P5", q[0]
    else:
        if img.channels != 3:
            raise ImageFormatError("PPM requires a 3-channel image")
        magic, body = b"P6", np.moveaxis(q, 0, 2)
    return magic + f"\n{img.width} {img.height}\n255\n".encode("ascii") + np.ascontiguousarray(body).tobytes()


def _load_png(path) -> Image:
    from PIL import Image as PILImage
    from PIL import UnidentifiedImageError

    try:
        with PILImage.open(path) as im:
            if im.mode == "P":
                im = im.convert("RGB")
            if im.mode not in ("L", "RGB"):
                raise ImageFormatError(f"unsupported image mode {im.mode!r} in {path.name} "
                                       "(8-bit grayscale or RGB required)")
            arr = np.asarray(im, dtype=np.float64)
    except UnidentifiedImageError as exc:
        raise ImageFormatError(f"unreadable image file: {path}") from exc
    return Image(data=arr[None] if arr.ndim == 2 else np.moveaxis(arr, 2, 0), range_max=255.0)


def _save_png(img: Image, path) -> None:
    from PIL import Image as PILImage

    q = quantize_u8(img.numpy())
    if img.channels == 1:
        PILImage.fromarray(q[0], mode="L").save(path, format="PNG")
    elif img.channels == 3:
        PILImage.fromarray(np.ascontiguousarray(np.moveaxis(q, 0, 2)), mode="RGB").save(path, format="PNG")
    else:
        raise ImageFormatError(f"cannot write {img.channels}-channel image as PNG")
