"""Experiment: per-warp-block hit tests of the compositing kernels on one
BJ.configs[3] view: entries whose conservative box (entry_box) meets an 8x8
(forward) or 16x8 (backward) block vs entries with a pixel of the block at
e >= kExpMin (the exact geometric test), ignoring termination."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import math  # noqa: E402

import torch  # noqa: E402

from paper_2312_10070_b200 import Params, Rasterizer, inputs  # noqa: E402

s = inputs.config3()
d = torch.device("cuda")
P = Params.from_numpy(*s.params(), device=d)
v = torch.as_tensor(s.views[0], device=d)
r = Rasterizer(s.n, s.cam, device=d)
r.size_for(P, v)
r.forward(P, v)
torch.cuda.synchronize()
H, W = s.cam.height, s.cam.width
TX = (W + 15) // 16
tr = r.tile_range.cpu()
idx = r.sorted_idx
uv, coef = r.proj.uv, r.proj.coef
kExpMin, kExpSkip = -7.994353294373, -7.995
ys, xs = torch.meshgrid(torch.arange(16, device=d), torch.arange(16, device=d), indexing="ij")
tot = {}
for (bw, bh) in ((8, 8), (16, 8)):
    tot[(bw, bh)] = [0, 0]
for t in range(tr.shape[0]):
    b, e_ = int(tr[t, 0]), int(tr[t, 1])
    if e_ <= b:
        continue
    tx, ty = t % TX, t // TX
    g = idx[b:e_].long()
    u = (uv[g, 0] - tx * 16).double()
    vv = (uv[g, 1] - ty * 16).double()
    c = coef[g].double()
    R2 = c[:, 3] - kExpSkip
    ok = R2 > 0
    R = torch.sqrt(torch.clamp(R2, min=0))
    hy = R / c[:, 2] + 0.05
    hx = R * torch.sqrt(c[:, 2] ** 2 + c[:, 1] ** 2) / (c[:, 0] * c[:, 2]) + 0.05
    X = xs.double().reshape(1, -1)
    Y = ys.double().reshape(1, -1)
    y1 = c[:, 0:1] * (u[:, None] - X) + c[:, 1:2] * (vv[:, None] - Y)
    y2 = c[:, 2:3] * (vv[:, None] - Y)
    e = (c[:, 3:4] - y1 * y1 - y2 * y2).reshape(-1, 16, 16)
    for (bw, bh) in ((8, 8), (16, 8)):
        for by in range(0, 16, bh):
            for bx in range(0, 16, bw):
                box = ok & (u + hx >= bx) & (u - hx <= bx + bw - 1) & (vv + hy >= by) & (vv - hy <= by + bh - 1)
                exact = (e[:, by:by + bh, bx:bx + bw] >= kExpMin).flatten(1).any(1)
                tot[(bw, bh)][0] += int(box.sum())
                tot[(bw, bh)][1] += int((box & exact).sum())
for k, (nb, ne) in tot.items():
    print("block %dx%d: box hits %d, with a pixel at alpha >= 1/255 %d (%.1f%%)" % (k[0], k[1], nb, ne, 100 * ne / nb))
