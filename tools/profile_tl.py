"""gs_tracking_loss on BJ.configs[2]-sized rendered maps, for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_10070_b200 import Params, Rasterizer, inputs  # noqa: E402

s = inputs.config2()
dev = torch.device("cuda:0")
P = Params.from_numpy(*s.params(), device=dev)
r = Rasterizer(s.n, s.cam, device=dev)
gt = torch.as_tensor(s.extra["gt_view"], device=dev)
r.size_for(P, gt)
r.forward(P, gt)
tc, td = r.frame.color.clone(), r.frame.depth.clone()
r.forward(P, torch.as_tensor(s.extra["start_view"], device=dev))
for _ in range(3):
    r.compute_tracking_loss(tc, td)
    r.compute_loss(tc, td)
torch.cuda.synchronize()
if len(sys.argv) > 1:
    import numpy as np
    f = r.frame
    ec = ((f.color - tc).abs().sum(0) / 3).cpu().numpy().astype(np.float32)
    ed = (f.depth - td).abs().cpu().numpy().astype(np.float32)
    for name, e in (("color", ec), ("depth", ed)):
        k = e.view(np.uint32).ravel()
        for sh in (24, 16, 8):
            b = np.bincount((k >> sh) & 255, minlength=256)
            print(name, sh, "max bin share %.3f" % (b.max() / k.size), "zeros %.3f" % (k == 0).mean())
