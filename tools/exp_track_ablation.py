"""Experiment (timing only: skipped stages leave stale buffers, results are
wrong): the marginal in-graph cost of each stage of a tracking iteration
(BJ.configs[2], 100 iterations captured in one CUDA graph), by dropping it."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_10070_b200 import Params, Rasterizer, inputs  # noqa: E402
from paper_2312_10070_b200.raster import GS_BWD_PIXELS_ONLY, GS_GRAD_POSE  # noqa: E402
from paper_2312_10070_b200.pipeline import TrackingLoop  # noqa: E402
from paper_2312_10070_b200.raster import gs_bin_sort, gs_render_fwd_l1, gs_tile_order  # noqa: E402

d = torch.device("cuda")
s = inputs.config2()
P = Params.from_numpy(*s.params(), device=d)
gt = torch.as_tensor(s.extra["gt_view"], device=d)
r0 = Rasterizer(s.n, s.cam, device=d)
r0.size_for(P, gt)
r0.forward(P, gt)
tc, td = r0.frame.color.clone(), r0.frame.depth.clone()
del r0


def run(skip):
    loop = TrackingLoop(P, s.cam, tc, td, torch.as_tensor(s.extra["start_view"], device=d), iters=100)
    loop.size()
    loop.prepare()
    loop.iteration()  # fills every buffer once (a dropped stage then reads stale, valid data)
    torch.cuda.synchronize()

    def it(i=0):
        r = loop.r
        if "project" not in skip:
            r.project(loop.params, loop.view)
        if "sort" not in skip:
            gs_bin_sort(r.proj, r.n, r.cam, r.sort_ws, r.capacity, r.sorted_idx, r.tile_range, r.n_pairs,
                        r.counters, tile_order=None)
        ov = "bwd" not in skip
        if "fwd" not in skip:
            gs_render_fwd_l1(r.proj, r.sorted_idx, r.tile_range, r.cam, r.frame, loop.tc, loop.td, r.scales,
                             r.dL_dcolor, r.dL_ddepth, tile_order=r.bwd_order, tile_work=r.tile_work,
                             tile_done=r._tile_done() if ov else None)
            if i % 8 == 0 and "order" not in skip:
                gs_tile_order(r.tile_work, r.T, r.bwd_order)
        if "bwd" not in skip:
            flags = GS_GRAD_POSE | (GS_BWD_PIXELS_ONLY if "gauss" in skip else 0)
            r.backward(loop.params, loop.view, flags, overlap="fwd" not in skip)
        if "pose" not in skip and "gauss" not in skip and "bwd" not in skip:
            r.pose_grad(loop.view, loop.stepcfg, loop.adam, dL_dtwist=loop.dtwist)
    loop.iteration = it
    loop.capture()
    for _ in range(2):
        loop.run()
    torch.cuda.synchronize()
    t = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        loop.reset()
        e0.record()
        loop.graph.replay()
        e1.record()
        torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1) * 10)  # us per iteration
    return statistics.median(t)


sets = [s.split("+") for s in sys.argv[1:]] or [["pose"], ["gauss"], ["bwd"], ["order"], ["sort"], ["project"],
                                               ["fwd"], ["project", "sort"]]
base = run(set())
print(f"full iteration {base:.1f} us")
for sk in sets:
    v = run(set(sk))
    print(f"without {'+'.join(sk):16s} {v:7.1f} us  (stage cost {base - v:6.1f} us)")
