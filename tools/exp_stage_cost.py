"""Experiment (not a bench number): effective cost of each stage inside the
pipelined mapping step, measured by dropping it from the step (stale buffers
stand in for its outputs).  BJ.configs[3], 8 views, 4 lanes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_10070_b200 import raster  # noqa: E402
from paper_2312_10070_b200.pipeline import MapStep  # noqa: E402
import bench  # noqa: E402

dev = torch.device("cuda")
s, P, views, tc, td = bench.make_workload(3, dev, 0, 1)
lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 8
sched = sys.argv[2] if len(sys.argv) > 2 else "lanes"
ms = MapStep(P, views, s.cam, tc, td, device=dev, lanes=lanes, schedule=sched)
ms.size()


def make(skip):
    noop = lambda *args: None
    hooks = {}
    if "project" in skip and "sort" in skip:
        hooks["front"] = noop
    elif "sort" in skip:
        hooks["front"] = lambda r, k, v: r.project(ms.params, ms.views[v])
    elif "project" in skip:
        hooks["front"] = lambda r, k, v: r.bin_sort()

    def fwd(r, k, v, tgt=None):
        if "fwd" not in skip:
            r.render()
        if "loss" not in skip:
            r.compute_loss(ms.tgt_color[v], ms.tgt_depth[v], None, ms.lc, ms.ld)
    hooks["fwd"] = fwd
    if "bwd" in skip:
        hooks["bwd"] = noop
    if "gauss" in skip:
        hooks["gauss"] = noop
    return hooks


def timeit(hooks, n=20):
    for _ in range(5):
        ms.step(hooks)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        ms.step(hooks)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


base = timeit(make(set()))
print(f"{sched} lanes {lanes}: full step {base:.3f} ms ({base / 8 * 1e3:.0f} us/view)")
for sk in (["sort"], ["project", "sort"], ["loss"], ["gauss"], ["fwd"], ["bwd"], ["fwd", "bwd"],
           ["project", "sort", "loss", "gauss"]):
    t = timeit(make(set(sk)))
    print(f"  without {'+'.join(sk):28s} {t:.3f} ms  (stage costs {(base - t) / 8 * 1e3:6.1f} us/view)")
