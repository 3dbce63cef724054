"""A few eager tracking iterations of BJ.configs[2] for ncu launch lists
(python tools/ncu_times.py "." python tools/profile_track.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_10070_b200 import Params, Rasterizer, inputs  # noqa: E402
from paper_2312_10070_b200.pipeline import TrackingLoop  # noqa: E402

d = torch.device("cuda")
s = inputs.config2()
P = Params.from_numpy(*s.params(), device=d)
gt = torch.as_tensor(s.extra["gt_view"], device=d)
r = Rasterizer(s.n, s.cam, device=d)
r.size_for(P, gt)
r.forward(P, gt)
tc, td = r.frame.color.clone(), r.frame.depth.clone()
loop = TrackingLoop(P, s.cam, tc, td, torch.as_tensor(s.extra["start_view"], device=d), iters=3)
loop.size()
loop.prepare()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    loop.iteration()
torch.cuda.synchronize()
