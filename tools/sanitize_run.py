"""Driver for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
one small pass over every kernel of the S1-S7 path on BJ.configs[0] and [1]
(or a given config list), including the flag-ordered paths (the tracking
forward -> backward overlap with tile_done) and a 2-view MapStep with the fused L1 loss.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [0 1]

Prints "sanitize_run ok" at the end; the sanitizer's own summary line
("ERROR SUMMARY: 0 errors") is the evidence.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2312_10070_b200 import GS_GRAD_PARAMS, GS_GRAD_POSE, Grads, Params, Rasterizer, inputs  # noqa: E402
from paper_2312_10070_b200.pipeline import MapStep, TrackingLoop  # noqa: E402


def run(cfg):
    d = torch.device("cuda:0")
    s = {0: inputs.config0, 1: inputs.config1}[cfg]()
    P = Params.from_numpy(*s.params(), device=d)
    v = torch.as_tensor(s.views[0], device=d)
    r = Rasterizer(s.n, s.cam, device=d)
    r.size_for(P, v)
    r.forward(P, v, stats=True)
    tc, td = r.frame.color.clone(), r.frame.depth.clone()
    tc.add_(0.05)
    r.compute_loss(tc, td)
    g = Grads.zeros(s.n, d)
    r.backward(P, v, GS_GRAD_PARAMS | GS_GRAD_POSE, g)
    r.pose_grad(v, dL_dview=torch.zeros(12, device=d), dL_dtwist=torch.zeros(6, device=d),
                dL_dqt=torch.zeros(7, device=d))
    # tracking: fused L1 forward -> overlapped pose backward (tile_done flags) -> Adam step
    loop = TrackingLoop(P, s.cam, tc, td, v.clone(), iters=3)
    loop.size()
    loop.run()
    assert loop.r.flag_timeouts() == 0
    loop_m = TrackingLoop(P, s.cam, tc, td, v.clone(), iters=2, masked=(0.5, 50.0))
    loop_m.size()
    loop_m.run()
    # mapping: two views, fused L1 loss, atomic S6, plus the SSIM colour term
    views = torch.stack([v, v]).contiguous()
    ms = MapStep(P, views, s.cam, {0: tc, 1: tc}, {0: td, 1: td}, device=d, lanes=2)
    ms.size()
    ms.step()
    ms.ssim = 0.2
    ms.step()
    counters = torch.cat([r.counters, loop.r.counters] + [x.counters for x in ms.lanes]).cpu()
    torch.cuda.synchronize()
    print(f"config {cfg}: counters {counters.tolist()}")


if __name__ == "__main__":
    cfgs = [int(x) for x in sys.argv[1:]] or [0, 1]
    for c in cfgs:
        run(c)
    print("sanitize_run ok")
