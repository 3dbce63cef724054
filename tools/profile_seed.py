"""gs_seed at BJ.configs[3] size (500k existing Gaussians, 1200x680, M_k = 50000), for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_10070_b200 import Params, Rasterizer, inputs  # noqa: E402
from paper_2312_10070_b200.raster import gs_seed, lib  # noqa: E402

s = inputs.config3()
dev = torch.device("cuda:0")
P = Params.from_numpy(*s.params(), device=dev)
v = torch.as_tensor(s.views[0], device=dev)
r = Rasterizer(s.n, s.cam, device=dev)
r.size_for(P, v)
r.forward(P, v)
alpha = r.frame.alpha.clone()
depth = (r.frame.depth / alpha.clamp_min(1e-6)).contiguous()
H, W = alpha.shape
alpha[H // 4:3 * H // 4, W // 4:3 * W // 4] = 0.0
K = 50000
Ps = Params(*[torch.cat([getattr(P, k), torch.zeros(K, 4, device=dev)]).contiguous()
              for k in ("mean_opa", "quat", "logscale", "rgb")])
ws = torch.empty((lib().gs_seed_workspace_bytes(r.cam, s.n, K) + 15) // 16 * 4, dtype=torch.float32, device=dev)
n_new = torch.zeros(1, dtype=torch.int32, device=dev)
for _ in range(2):
    gs_seed(r.cam, s.views[0], r.frame.color, depth, alpha, 0.6, 0.01, K, 1, Ps, s.n, ws, n_new)
torch.cuda.synchronize()
print("accepted", int(n_new.item()))
if len(sys.argv) > 1:
    import numpy as np
    E = P.mean_opa.cpu().numpy()[:, :3].astype(np.float64)
    c = np.floor(E / 0.1).astype(np.int64)
    _, cnt = np.unique(c, axis=0, return_counts=True)
    print("existing: cells", len(cnt), "max per cell", cnt.max(), "mean", cnt.mean())
    print("means range", E.min(0), E.max(0))
