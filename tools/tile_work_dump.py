"""Experiment: per-tile work of one BJ.configs[3] view for schedule studies
(the compositing launches' heavy-tile tails).  Saves, per tile: the list
length, the largest n_contrib of each 8x8 block (the forward's warps) and of
each 16x8 strip (the backward's warps), and the forward's entries scanned
(stats) summed per 8x8 block, to gpurun_out/tile_work.npz."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2312_10070_b200 import Params, Rasterizer, inputs  # noqa: E402

d = torch.device("cuda")
s = inputs.config3()
P = Params.from_numpy(*s.params(), device=d)
out = {}
for vi in range(2):
    v = torch.as_tensor(s.views[vi], device=d)
    r = Rasterizer(s.n, s.cam, device=d)
    r.size_for(P, v)
    r.forward(P, v, stats=True)
    torch.cuda.synchronize()
    H, W = s.cam.height, s.cam.width
    TX, TY = (W + 15) // 16, (H + 15) // 16
    nc = torch.zeros(TY * 16, TX * 16, dtype=torch.int32, device=d)
    nc[:H, :W] = r.frame.n_contrib.view(H, W)
    sc = torch.zeros(TY * 16, TX * 16, dtype=torch.int32, device=d)
    sc[:H, :W] = r.frame.stats[0].view(H, W)
    blk = nc.view(TY, 2, 8, TX, 2, 8).amax(dim=(2, 5))           # [TY, 2, TX, 2] 8x8 blocks
    strip = nc.view(TY, 2, 8, TX, 16).amax(dim=(2, 4))            # [TY, 2, TX] 16x8 strips
    scan = sc.view(TY, 2, 8, TX, 2, 8).amax(dim=(2, 5))
    rng = r.tile_range.cpu().numpy() if hasattr(r, "tile_range") else None
    out[f"v{vi}_blk"] = blk.cpu().numpy()
    out[f"v{vi}_strip"] = strip.cpu().numpy()
    out[f"v{vi}_scan"] = scan.cpu().numpy()
    if rng is not None:
        out[f"v{vi}_len"] = (rng[:, 1] - rng[:, 0]).reshape(TY, TX)
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/tile_work.npz", **out)
print("saved", {k: v.shape for k, v in out.items()})
