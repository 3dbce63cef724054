"""Per-tile work distribution of one BJ.configs[3] view (list length, sum of
n_contrib, scanned entries) -- explains the compositing kernels' tail."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2312_10070_b200 import Params, Rasterizer, inputs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
s = {1: inputs.config1, 2: inputs.config2, 3: inputs.config3, 4: inputs.config4}[cfg]()
d = torch.device("cuda")
P = Params.from_numpy(*s.params(), device=d)
v = torch.as_tensor(s.views[0], device=d)
r = Rasterizer(s.n, s.cam, device=d)
r.size_for(P, v)
r.forward(P, v, stats=True)
torch.cuda.synchronize()
tr = r.tile_range.cpu().numpy()
L = tr[:, 1] - tr[:, 0]
work = r.tile_work.cpu().numpy().astype(np.float64)
TX = (s.cam.width + 15) // 16
H, W = s.cam.height, s.cam.width
sc = r.frame.stats[0].cpu().numpy().astype(np.float64)
TY = (H + 15) // 16
pad = np.zeros((TY * 16, TX * 16))
pad[:H, :W] = sc
scan = pad.reshape(TY, 16, TX, 16).sum(axis=(1, 3)).ravel()
for name, x in (("list length", L), ("sum n_contrib (bwd work)", work), ("sum scanned (fwd work)", scan)):
    q = np.percentile(x, [50, 90, 99, 100])
    print(f"{name:26s} mean {x.mean():10.1f}  p50 {q[0]:10.1f}  p90 {q[1]:10.1f}  p99 {q[2]:10.1f}  max {q[3]:10.1f}  "
          f"max/mean {q[3] / x.mean():.2f}  top-148 share {np.sort(x)[-148:].sum() / x.sum():.3f}")
