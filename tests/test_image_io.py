"""§8 row f4: KFC1 cube and PNM/PNG I/O (image.py:115-270), host-side.

The golden bytes were written by the reference's own save_image
(tools/make_golden.py); no GPU is needed."""

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


def test_pnm_bytes_match_reference(tmp_path):
    g = load_golden("image_io")
    for nm, key in (("ppm", "rgb"), ("pgm", "gray")):
        p = tmp_path / f"x.{nm}"
        save_image(Image(data=g[key], range_max=255.0), p)
        assert p.read_bytes() == g[f"pnm_{nm}"].tobytes()
        back = load_image(p)
        assert np.array_equal(back.data, quantize_u8(g[key]).astype(np.float64))


def test_png_roundtrip_and_errors(tmp_path):
    rgb = np.round(np.random.default_rng(1).uniform(0, 255, (3, 9, 11)))
    p = tmp_path / "a.png"
    save_image(Image(data=rgb, range_max=255.0), p)
    assert np.array_equal(load_image(p).data, rgb)
    with pytest.raises(ImageFormatError):
        save_image(Image(data=rgb[:2], range_max=255.0), tmp_path / "b.png")
    with pytest.raises(ImageFormatError):
        save_image(Image(data=rgb, range_max=255.0), tmp_path / "b.bmp")
    with pytest.raises(ImageFormatError):
        save_image(Image(data=rgb, range_max=255.0), tmp_path / "b.pgm")
    bad = tmp_path / "bad.kfc"
    bad.write_bytes(CUBE_MAGIC + np.array([2, 2, 1, 0], "<u4").tobytes() + b"\0" * 12)
    with pytest.raises(ImageFormatError, match="size mismatch"):
        load_image(bad)
    bad.write_bytes(CUBE_MAGIC + np.array([1, 1, 1, 7], "<u4").tobytes() + b"\0" * 8)
    with pytest.raises(ImageFormatError, match="flag"):
        load_image(bad)
    (tmp_path / "t.ppm").write_bytes(b"P6\n2 2\n65535\n" + b"\0" * 24)
    with pytest.raises(ImageFormatError, match="bit depth"):
        load_image(tmp_path / "t.ppm")
    (tmp_path / "c.pgm").write_bytes(b"P5\n# comment\n3 1\n255\n\x01\x02\x03")
    assert load_image(tmp_path / "c.pgm").data.ravel().tolist() == [1.0, 2.0, 3.0]
