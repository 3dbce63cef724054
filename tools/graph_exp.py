"""Experiment: the pipelined mapping step (BJ.configs[3], 8 views) replayed
as one CUDA graph vs launched eagerly from Python."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time  # noqa: E402

import torch  # noqa: E402

from paper_2312_10070_b200.pipeline import MapStep  # noqa: E402
import bench  # noqa: E402

dev = torch.device("cuda")
s, P, views, tc, td = bench.make_workload(3, dev, 0, 1)
lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ms = MapStep(P, views, s.cam, tc, td, device=dev, lanes=lanes)
ms.overlap = True  # as the bench
ms.size()
for _ in range(5):
    ms.step()
torch.cuda.synchronize()
ref = ms.grads.buf.clone()


def timeit(fn, n=30):
    fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    a.record()
    for _ in range(n):
        fn()
    h1 = time.perf_counter()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3, (h1 - h0) / n * 1e6


print("eager: %.1f us/step device, %.1f us/step host enqueue" % timeit(ms.step))
g = torch.cuda.CUDAGraph()
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    ms.step()
torch.cuda.current_stream().wait_stream(side)
torch.cuda.synchronize()
with torch.cuda.graph(g):
    ms.step()
torch.cuda.synchronize()
g.replay()
torch.cuda.synchronize()
got = ms.grads.buf
print("graph grads max rel diff vs eager: %.2e" % ((got - ref).abs().max() / ref.abs().max()).item())
print("graph: %.1f us/step device, %.1f us/step host enqueue" % timeit(g.replay))
