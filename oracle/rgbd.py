"""Oracle of the RGB-D input unpacking (gs_unpack_rgbd) — TEST INFRASTRUCTURE ONLY.

Plain numpy; shares nothing with the CUDA path.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / ``--impl
reference`` leg may import it.

P:113 ("the RGBD frame"), P:216 ("C_i and D_i are the input color and depth
map at frame i"), P:234 ("trajectories from an RGBD sensor"): the sensors'
frames are 8-bit RGB and 16-bit depth in units of a dataset scale (DESIGN.md
R42).  The targets are  C[c][j][i] = rgb[j][i][c] / 255  and
D[j][i] = depth16[j][i] * scale, both rounded once to fp32 (the division and
the product of two fp32 numbers, correctly rounded).
"""
from __future__ import annotations

import numpy as np


def unpack(rgb8, depth16, scale):
    """(color [3, H, W] fp32, depth [H, W] fp32) from rgb8 [H, W, 3] uint8 and
    depth16 [H, W] uint16."""
    rgb = np.asarray(rgb8, np.uint8)
    d = np.asarray(depth16, np.uint16)
    color = (rgb.astype(np.float32) / np.float32(255.0)).transpose(2, 0, 1).copy()
    depth = d.astype(np.float32) * np.float32(scale)
    return color, depth

