"""Experiment: scanned / contributed / replayed entries of the tracking view
(BJ.configs[2], the start pose) -> algorithmic flops of one forward and one
backward launch (bench.py's SURVEY §8(d) counts) for the tracking kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_10070_b200 import Params, Rasterizer, inputs  # noqa: E402

d = torch.device("cuda")
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
s = {2: inputs.config2, 3: inputs.config3}[cfg]()
P = Params.from_numpy(*s.params(), device=d)
v = torch.as_tensor(s.extra["start_view"] if cfg == 2 else s.views[0], device=d)
r = Rasterizer(s.n, s.cam, device=d)
r.size_for(P, v)
r.forward(P, v, stats=True)
st = r.frame.stats
sc, c = int(st[0].sum().item()), int(st[1].sum().item())
rp = int(r.frame.n_contrib.sum().item())
print(f"config {cfg}: pairs {int(r.n_pairs.item())} scanned {sc} contrib {c} replayed {rp}")
print(f"fwd GFLOP {(10 * sc + 11 * c) / 1e9:.3f}  bwd GFLOP {(10 * rp + 64 * c) / 1e9:.3f} "
      f"(pose-only bwd without the colour terms: {(10 * rp + 52 * c) / 1e9:.3f})")
