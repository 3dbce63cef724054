"""Pins of the RGB-D unpacking oracle (R42)."""
import numpy as np

from oracle import rgbd
from paper_2312_10070_b200 import inputs


def test_unpack_values_and_layout():
    H, W = 3, 5
    rgb = np.zeros((H, W, 3), np.uint8)
    rgb[1, 2] = (0, 128, 255)
    rgb[2, 4] = (1, 2, 3)
    d = np.zeros((H, W), np.uint16)
    d[0, 1] = 5000
    d[2, 3] = 65535
    c, z = rgbd.unpack(rgb, d, 1.0 / 5000)
    assert c.shape == (3, H, W) and z.shape == (H, W) and c.dtype == np.float32
    assert c[0, 1, 2] == 0.0 and c[2, 1, 2] == 1.0  # 255 / 255 is exactly 1
    assert c[1, 1, 2] == np.float32(128) / np.float32(255)
    assert abs(float(c[1, 1, 2]) - 128 / 255) <= 2 ** -24  # correctly rounded
    assert tuple(c[:, 2, 4] * 255) == (1.0, 2.0, 3.0)
    assert abs(float(z[0, 1]) - 1.0) < 1e-7  # 5000 units of 0.2 mm
    assert abs(float(z[2, 3]) - 13.107) < 1e-5
    assert (z[d == 0] == 0).all()  # invalid depth stays invalid


def test_brute_force_loops():
    rng = np.random.default_rng(0)
    H, W = 7, 9
    rgb = rng.integers(0, 256, (H, W, 3), dtype=np.uint8)
    d = rng.integers(0, 65536, (H, W), dtype=np.uint16)
    c, z = rgbd.unpack(rgb, d, 1 / 6553.5)
    for j in range(H):
        for i in range(W):
            for ch in range(3):
                assert c[ch, j, i] == np.float32(float(rgb[j, i, ch]) / 255.0)
            assert z[j, i] == np.float32(np.float32(d[j, i]) * np.float32(1 / 6553.5))


def test_quantize_round_trip():
    rng = np.random.default_rng(1)
    rgb = rng.integers(0, 256, (4, 6, 3), dtype=np.uint8)
    d = rng.integers(0, 65536, (4, 6), dtype=np.uint16)
    c, z = rgbd.unpack(rgb, d, inputs.DEPTH_SCALE)
    r2, d2 = inputs.quantize_rgbd(c, z)  # the synthetic sensor frames of the e2e leg
    assert np.array_equal(r2, rgb) and np.array_equal(d2, d)
