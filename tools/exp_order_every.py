"""Experiment: tracking iterations/s vs how often the launch order is refreshed (TrackingLoop.order_every)."""
import os, sys, statistics
sys.path.insert(0, os.getcwd())
import torch
from paper_2312_10070_b200 import Params, Rasterizer, inputs
from paper_2312_10070_b200.pipeline import TrackingLoop
d = torch.device("cuda")
s = inputs.config2()
P = Params.from_numpy(*s.params(), device=d)
gt = torch.as_tensor(s.extra["gt_view"], device=d)
r = Rasterizer(s.n, s.cam, device=d); r.size_for(P, gt); r.forward(P, gt)
tc, td = r.frame.color.clone(), r.frame.depth.clone(); del r
for oe in ([int(x) for x in sys.argv[1:]] or (1, 4, 8, 16, 32)):
    loop = TrackingLoop(P, s.cam, tc, td, torch.as_tensor(s.extra["start_view"], device=d), iters=100)
    loop.order_every = oe
    loop.size(); loop.capture()
    ts = []
    for _ in range(5):
        loop.reset(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); loop.graph.replay(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(oe, 100 / (statistics.median(ts) * 1e-3))
    del loop; torch.cuda.empty_cache()
