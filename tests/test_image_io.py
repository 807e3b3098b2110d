"""§8 row f4: the KFC1 float cube (image.py:243-270), host-side.

The golden bytes were written by the reference's own save_image
(tools/make_golden.py); no GPU is needed.  PNG / PGM / PPM are outside this
build's scope and raise ImageFormatError."""

import numpy as np
import pytest

from conftest import load_golden
from paper_1901_06112_b200 import CUBE_MAGIC, Image, ImageFormatError, load_image, quantize_u8, save_image


def test_cube_bytes_match_reference(tmp_path):
    g = load_golden("image_io")
    img = Image(data=g["cube"], range_max=1.0)
    for dt in ("float32", "float64"):
        p = tmp_path / f"c_{dt}.kfc"
        save_image(img, p, cube_dtype=dt)
        assert p.read_bytes() == g[f"cube_{dt}"].tobytes()
        back = load_image(p)
        assert back.range_max == 255.0 and back.data.shape == (5, 6, 7)
        want = g["cube"].astype(np.float32).astype(np.float64) if dt == "float32" else g["cube"]
        assert np.array_equal(back.data, want)
    with pytest.raises(ValueError):
        save_image(img, tmp_path / "x.kfc", cube_dtype="float16")


def test_cube_errors(tmp_path):
    bad = tmp_path / "bad.kfc"
    bad.write_bytes(CUBE_MAGIC + np.array([2, 2, 1, 0], "<u4").tobytes() + b"\0" * 12)
    with pytest.raises(ImageFormatError, match="size mismatch"):
        load_image(bad)
    bad.write_bytes(CUBE_MAGIC + np.array([1, 1, 1, 7], "<u4").tobytes() + b"\0" * 8)
    with pytest.raises(ImageFormatError, match="flag"):
        load_image(bad)
    bad.write_bytes(CUBE_MAGIC + b"\0" * 6)
    with pytest.raises(ImageFormatError, match="truncated"):
        load_image(bad)


def test_raster_formats_are_out_of_scope(tmp_path):
    rgb = np.round(np.random.default_rng(1).uniform(0, 255, (3, 9, 11)))
    for name in ("a.png", "a.ppm", "a.pgm", "a.bmp"):
        with pytest.raises(ImageFormatError):
            save_image(Image(data=rgb, range_max=255.0), tmp_path / name)
    (tmp_path / "c.pgm").write_bytes(b"P5\n3 1\n255\n\x01\x02\x03")
    with pytest.raises(ImageFormatError, match="KFC1"):
        load_image(tmp_path / "c.pgm")


def test_quantize_u8_matches_reference_writer():
    g = load_golden("image_io")
    # the reference's PPM writer stored quantize_u8(rgb) channel-interleaved after its header
    body = np.frombuffer(g["pnm_ppm"].tobytes()[-g["rgb"].size:], np.uint8)
    q = quantize_u8(g["rgb"])
    assert np.array_equal(body, np.moveaxis(q, 0, 2).ravel())
