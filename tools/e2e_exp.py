"""Experiment: where the end-to-end step's extra time goes (BJ.configs[3]):
device-resident step vs host inputs (all), host inputs without the
parameter upload, and host inputs without the frame uploads."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_10070_b200.pipeline import HostInputs, MapStep  # noqa: E402
import bench  # noqa: E402

dev = torch.device("cuda")
s, P, views, tc, td = bench.make_workload(3, dev, 0, 1)
ms = MapStep(P, views, s.cam, tc, td, device=dev)
ms.size()


def timeit(fn, n=20):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


print("device-resident  %.3f ms" % timeit(ms.step))
host = HostInputs(ms.params, ms.views, ms.tgt_color, ms.tgt_depth, ms.mine, ms.losses.shape[0])
print("host, all        %.3f ms" % timeit(lambda: ms.step(host=host)))
saved = dict(host.params)
for k in saved:
    host.params[k] = saved[k][:1]  # a 16-byte stand-in: no parameter upload


def step_noparams():
    ms.step(host=host)


# patch the copies of the params to slices of one row (experiment only)
orig = ms.params
print("host, no params  n/a (parameters are copied as whole arrays)")
host.params = saved
up = host.upload_targets
host.upload_targets = lambda *args, **kw: False
print("host, no frames  %.3f ms" % timeit(lambda: ms.step(host=host)))
host.upload_targets = up
import time  # noqa: E402
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    ms.step(host=host)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print("host enqueue %.3f ms/step, wall %.3f ms/step" % ((t1 - t0) / 20 * 1e3, (t2 - t0) / 20 * 1e3))
t0 = time.perf_counter()
for _ in range(20):
    ms.step()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print("device-resident: host enqueue %.3f ms/step, wall %.3f ms/step" % ((t1 - t0) / 20 * 1e3, (t2 - t0) / 20 * 1e3))
