"""Experiment: the end-to-end step with parts of the upload / unpack path disabled (copies only, no gradient scales)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2312_10070_b200.pipeline import HostInputs, MapStep
from paper_2312_10070_b200 import pipeline as PL
import bench
dev = torch.device("cuda")
s, P, views, tc, td = bench.make_workload(3, dev, 0, 1)
ms = MapStep(P, views, s.cam, tc, td, device=dev)
ms.size()
def timeit(fn, n=30):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
print("device-resident  %.3f" % timeit(ms.step))
host = HostInputs(ms.params, ms.views, ms.tgt_color, ms.tgt_depth, ms.mine, ms.losses.shape[0])
print("host all         %.3f" % timeit(lambda: ms.step(host=host)))
def copies_only(v, cam, c, d, *rest):
    host.dev_rgb8[v].copy_(host.rgb8[v], non_blocking=True)
    host.dev_d16[v].copy_(host.d16[v], non_blocking=True)
orig = host.upload_targets
host.upload_targets = copies_only
print("frames copied, no unpack  %.3f" % timeit(lambda: ms.step(host=host)))
host.upload_targets = orig
orig_scales = PL.gs_loss_scales
PL.gs_loss_scales = lambda *a, **k: None
print("no scales        %.3f" % timeit(lambda: ms.step(host=host)))
PL.gs_loss_scales = orig_scales
print("host all again   %.3f" % timeit(lambda: ms.step(host=host)))
