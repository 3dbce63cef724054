"""Debug: one view of a config through project -> bin_sort -> render -> backward
with host checks of the binning invariants between the stages."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2312_10070_b200 import GS_GRAD_PARAMS, Grads, Params, Rasterizer, inputs  # noqa: E402
from paper_2312_10070_b200.raster import GS_BWD_PIXELS_ONLY  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
s = {1: inputs.config1, 3: inputs.config3, 4: inputs.config4}[cfg]()
d = torch.device("cuda")
P = Params.from_numpy(*s.params(), device=d)
v = torch.as_tensor(s.views[0], device=d)
r = Rasterizer(s.n, s.cam, device=d)
r.size_for(P, v)
torch.cuda.synchronize()
Pn = int(r.n_pairs.item())
rng = r.tile_range.cpu().numpy()
order = r.tile_order.cpu().numpy()
idx = r.sorted_idx[:Pn].cpu().numpy()
print("pairs", Pn, "capacity", r.capacity, "T", r.T)
print("order perm:", np.array_equal(np.sort(order), np.arange(r.T)))
print("ranges contiguous:", rng[0, 0] == 0 and (rng[1:, 0] == rng[:-1, 1]).all() and rng[-1, 1] == Pn)
print("idx in range:", idx.min() >= 0, idx.max() < s.n)
r.render()
torch.cuda.synchronize()
nc = r.frame.n_contrib.cpu().numpy()
print("n_contrib max", nc.max(), "max list", (rng[:, 1] - rng[:, 0]).max())
bo = r.bwd_order.cpu().numpy()
print("bwd order perm:", np.array_equal(np.sort(bo), np.arange(r.T)))
gc, gd, ga = inputs.upstream_maps(11, s.cam)
t = lambda a: torch.as_tensor(np.ascontiguousarray(a, np.float32), device=d)
g = Grads.zeros(s.n, d)
r.backward(P, v, GS_GRAD_PARAMS | GS_BWD_PIXELS_ONLY, g, dL_dcolor=t(gc), dL_ddepth=t(gd), dL_dalpha=t(ga))
torch.cuda.synchronize()
print("bwd pixels ok")
