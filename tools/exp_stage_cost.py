"""Experiment (not a bench number): effective cost of each stage inside the
pipelined mapping step, measured by dropping it from the step (stale buffers
stand in for its outputs; the parameters do not change between steps, so
those are the same values).  BJ.configs[3], 8 views, 8 lanes, the bench's
configuration (fused L1 loss, forward -> backward tile overlap)."""
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
ms = MapStep(P, views, s.cam, tc, td, device=dev, lanes=lanes)
ms.overlap = True
ms.size()


def make(skip):
    noop = lambda *args: None
    hooks = {}
    if "project" in skip and "sort" in skip:
        hooks["front"] = noop
    elif "sort" in skip:
        hooks["front"] = lambda r, k, v: r.project(ms.params, ms.views[v])
    elif "project" in skip:
        hooks["front"] = lambda r, k, v: r.bin_sort(order=ms.fwd_order(r, v) is None)
    if "fwd" in skip:
        hooks["fwd"] = noop
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
print(f"lanes {lanes}: full step {base:.3f} ms ({base / 8 * 1e3:.0f} us/view)")
for sk in (["sort"], ["project"], ["project", "sort"], ["gauss"], ["fwd"], ["bwd"], ["fwd", "bwd"],
           ["project", "sort", "gauss"]):
    t = timeit(make(set(sk)))
    print(f"  without {'+'.join(sk):28s} {t:.3f} ms  (stage costs {(base - t) / 8 * 1e3:6.1f} us/view)")
