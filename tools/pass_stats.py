"""Per-(warp footprint, entry) pass statistics of the backward on one
BJ.configs[3] view: for candidate warp footprints, how many (footprint,
entry) pairs have a passing pixel (the backward processes those) and how many
pixels pass in them.  Runs on the GPU box (torch on cuda)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_10070_b200 import Params, Rasterizer, inputs  # noqa: E402

s = inputs.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]()
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
nc = r.frame.n_contrib
kExpMin = -7.994353294373
fps = [(8, 4), (16, 2), (8, 8), (16, 4), (16, 8), (16, 16)]
acc = {f: [0, 0, 0] for f in fps}  # processed pairs, passing pixels, hit pairs (any pixel of fp in list)
ys, xs = torch.meshgrid(torch.arange(16, device=d), torch.arange(16, device=d), indexing="ij")
for t in range(tr.shape[0]):
    b, e_ = int(tr[t, 0]), int(tr[t, 1])
    if e_ <= b:
        continue
    tx, ty = t % TX, t // TX
    g = idx[b:e_].long()
    u = uv[g, 0] - tx * 16
    vv = uv[g, 1] - ty * 16
    c = coef[g].double()
    X = xs.double().reshape(1, -1)
    Y = ys.double().reshape(1, -1)
    y1 = c[:, 0:1] * (u[:, None] - X) + c[:, 1:2] * (vv[:, None] - Y)
    y2 = c[:, 2:3] * (vv[:, None] - Y)
    e = c[:, 3:4] - y1 * y1 - y2 * y2
    py, px = ty * 16 + ys.reshape(-1), tx * 16 + xs.reshape(-1)
    inside = (py < H) & (px < W)
    last = torch.zeros(256, dtype=torch.long, device=d)
    last[inside] = nc[py[inside], px[inside]].long()
    pos = torch.arange(e_ - b, device=d)[:, None]
    ps = (e >= kExpMin) & (pos < last[None, :])  # [L, 256]
    ps = ps.reshape(-1, 16, 16)
    for (fw, fh) in fps:
        blk = ps.reshape(-1, 16 // fh, fh, 16 // fw, fw).sum(dim=(2, 4))  # [L, nby, nbx]
        acc[(fw, fh)][0] += int((blk > 0).sum())
        acc[(fw, fh)][1] += int(blk.sum())
for f in fps:
    n, p, _ = acc[f]
    print("footprint %2dx%-2d  processed (warp, entry) %8d  passing px %9d  px/entry %.1f of %d" % (
        f[0], f[1], n, p, p / max(n, 1), f[0] * f[1]))
