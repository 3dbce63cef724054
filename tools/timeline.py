"""Experiment: per-lane stage timeline of one pipelined mapping step
(BJ.configs[3], 8 views): CUDA events around every stage of every view,
printed as start/end (us) relative to the step start.  Events add a little
overhead; for the shape of the schedule only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_10070_b200.pipeline import MapStep  # noqa: E402
import bench  # noqa: E402

dev = torch.device("cuda")
s, P, views, tc, td = bench.make_workload(3, dev, 0, 1)
lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ms = MapStep(P, views, s.cam, tc, td, device=dev, lanes=lanes)
ms.overlap = True
ms.size()
ev = {}


def wrap(name, fn):
    def h(r, k, v, *rest):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn(r, k, v, *rest)
        b.record()
        ev[(k, name)] = (a, b)
    return h


hooks = {n: wrap(n, getattr(ms, "stage_" + n)) for n in ("front", "fwd", "bwd", "gauss")}
for _ in range(5):
    ms.step(hooks)
torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True)
t1 = torch.cuda.Event(enable_timing=True)
# steady state: the measured step is queued behind two others (the host runs
# ahead), so its timeline shows the GPU's schedule, not the host's enqueue
ms.step(hooks)
ms.step(hooks)
t0.record()
ms.step(hooks)
t1.record()
torch.cuda.synchronize()
print("step %.1f us" % (t0.elapsed_time(t1) * 1e3))
print("view  " + "  ".join("%-15s" % n for n in ("front", "fwd+loss", "bwd", "gauss")))
for k in range(len(ms.mine)):
    row = []
    for n in ("front", "fwd", "bwd", "gauss"):
        a, b = ev[(k, n)]
        row.append("%6.0f-%-6.0f  " % (t0.elapsed_time(a) * 1e3, t0.elapsed_time(b) * 1e3))
    print("%4d  %s" % (k, "".join(row)))
