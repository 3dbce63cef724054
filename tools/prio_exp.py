"""Experiment: stream priorities in the pipelined mapping step (BJ.configs[3],
8 views), each variant captured in a CUDA graph and replayed:
  base      8 lanes, default priority
  halves    lanes 0-3 high priority, 4-7 low
  front_hi  every view's front stage (project + bin_sort) on a high-priority
            stream, the rest of its chain on its low-priority lane
  back_hi   the front on the lane, the rest on a high-priority stream per lane
  two       two independent steps in one graph (fill / drain bound)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_10070_b200.pipeline import MapStep  # noqa: E402
import bench  # noqa: E402

dev = torch.device("cuda")
s, P, views, tc, td = bench.make_workload(3, dev, 0, 1)
lo, hi = torch.cuda.Stream.priority_range()  # (low, high) numerically: high is more negative


def make(variant):
    ms = MapStep(P, views, s.cam, tc, td, device=dev, lanes=8)
    ms.size()
    if variant == "halves":
        ms.streams = [torch.cuda.Stream(priority=hi if k < 4 else lo) for k in range(8)]
    if variant in ("front_hi", "back_hi"):
        ms.streams = [torch.cuda.Stream(priority=lo) for _ in range(8)]
        extra = [torch.cuda.Stream(priority=hi) for _ in range(8)]
        ms.all_streams = ms.streams + extra
        front_on_extra = variant == "front_hi"
        orig = {n: getattr(ms, "stage_" + n) for n in ("front", "fwd", "bwd", "gauss")}
        ev = {}

        def front(r, k, v):
            if front_on_extra:
                cur = torch.cuda.current_stream()
                extra[k].wait_stream(cur)
                with torch.cuda.stream(extra[k]):
                    orig["front"](r, k, v)
                cur.wait_stream(extra[k])
            else:
                orig["front"](r, k, v)

        def later(name):
            def f(r, k, v, *rest):
                if front_on_extra:
                    return orig[name](r, k, v, *rest)
                cur = torch.cuda.current_stream()
                extra[k].wait_stream(cur)
                with torch.cuda.stream(extra[k]):
                    orig[name](r, k, v, *rest)
                cur.wait_stream(extra[k])
            return f
        ms.hooks = {"front": front, "fwd": later("fwd"), "bwd": later("bwd"), "gauss": later("gauss")}
    else:
        ms.hooks = None
    return ms


def graph_of(fns):
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(3):
            for f in fns:
                f()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for f in fns:
            f()
    return g


def timeit(g, n=30):
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


for variant in ("base", "halves", "front_hi", "back_hi"):
    ms = make(variant)
    g = graph_of([lambda ms=ms: ms.step(ms.hooks)])
    print("%-9s %.1f us/step" % (variant, timeit(g)))
    del g, ms
    torch.cuda.empty_cache()
m1, m2 = make("base"), make("base")
side2 = torch.cuda.Stream()


def two():
    cur = torch.cuda.current_stream()
    side2.wait_stream(cur)
    m1.step()
    with torch.cuda.stream(side2):
        m2.step()
    cur.wait_stream(side2)


g = graph_of([two])
print("two independent steps concurrently: %.1f us (per step %.1f)" % (timeit(g), timeit(g) / 2))
