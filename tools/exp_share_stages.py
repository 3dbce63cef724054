"""Experiment (not a bench number): marginal cost of each stage of rank 0's
share at k = 8 ranks (one BJ.configs[3] view, MapStep(world=8) with the
all-reduce left out), measured by dropping the stage from the captured step
(stale buffers stand in for its outputs); graph replay, L2 flushed between
timed replays, median of 40."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_10070_b200.pipeline import MapStep
import bench
dev = torch.device("cuda")
s, P, views, tc, td = bench.make_workload(3, dev, 0, 1)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
ms = MapStep(P, views, s.cam, tc, td, rank=0, world=8, allreduce=lambda b: None, device=dev)
ms.overlap = True
ms.allreduce = None
ms.size()
for _ in range(3): ms.step()
def make(skip):
    noop = lambda *args: None
    hooks = {}
    if "project" in skip and "sort" in skip: hooks["front"] = noop
    elif "sort" in skip: hooks["front"] = lambda r, k, v: r.project(ms.params, ms.views[v])
    elif "project" in skip: hooks["front"] = lambda r, k, v: r.bin_sort(order=ms.fwd_order(r, v) is None)
    for st in ("fwd", "bwd", "gauss"):
        if st in skip: hooks[st] = noop
    return hooks
def timeit(hooks, n=40):
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        ms.step(hooks); ms.step(hooks)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        ms.step(hooks)
    t = []
    for _ in range(n):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); t.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(x.elapsed_time(y) for x, y in t) * 1e3
base = timeit(make(set()))
print(f"k8 share (graph, flushed) {base:.1f} us")
for sk in (["sort"], ["project"], ["project", "sort"], ["gauss"], ["fwd"], ["bwd"], ["fwd", "bwd"], ["bwd", "gauss"]):
    t = timeit(make(set(sk)))
    print(f"  without {'+'.join(sk):20s} {t:7.1f} us  (stage cost {base - t:6.1f} us)")
