#!/usr/bin/env python
"""Benchmark of the Gaussian-SLAM rasterizer hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config 3]

One *step* = one multi-view sub-map mapping iteration of BJ.configs[3]
(500k Gaussians, 1200x680, 8 keyframe views): per view gs_project ->
gs_bin_sort -> gs_render_fwd_l1 (compositing with the L1 loss gradient and
tile loss sums fused) -> gs_loss_from_tiles -> gs_render_bwd (all
parameters), the views on 8 concurrent streams, and for N > 1 one NCCL
all-reduce of the gradient buffer.  Views are sharded
round-robin across ranks (strong scaling: 8 views in total for every N).
Metric: fwd+bwd megapixels/s = (8 x 1200 x 680 / 1e6) / step time, max over
ranks.  Also reported: tracking iterations/s (BJ.configs[2], 100 iterations
in one CUDA graph, N = 1 only), the roofline of the dominant kernel, the
oracle as a CPU baseline, and the end-to-end number with host buffers.

--impl reference times the fp64 CPU oracle (the only reference this tier has)
on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fwd+bwd megapixels/s at 1200x680 (500k Gaussians)"
UNIT = "MP/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3, choices=[1, 3, 4])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tracking", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time the mapping step launched eagerly, not replayed")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no clocks/cpu/e2e/tracking)")
    ap.add_argument("--lanes", type=int, default=8, help="per-view buffer sets (and lane streams)")
    ap.add_argument("--no-overlap", action="store_true",
                    help="stream-ordered forward -> backward (no per-tile flag overlap) in the timed step")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: tests of the multi-rank branch on one GPU)")
    ap.add_argument("--small", action="store_true",
                    help="tests only: BJ.configs[3] reduced to 40k Gaussians, 4 views of 320x184")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)

class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", str(self.index)], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p is not None:
            time.sleep(0.25)
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        self.f.flush()
        rows = [l.split(",") for l in open(self.f.name).read().strip().splitlines() if l.strip()]
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for k, nm in enumerate(names):
                if len(r) > 5 + k and "Active" in r[5 + k] and "Not" not in r[5 + k]:
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


# ---------------------------------------------------------------------------
# workload

def make_workload(cfg, device, rank, world, small=False):
    import torch
    from paper_2312_10070_b200 import Params, Rasterizer, inputs
    if small:  # tests only (bench.py --small)
        s = inputs.config3(seed=5, n=40_000, n_views=4)
        s.cam = inputs.Camera(320, 184, 160.0, 160.0, 159.5, 91.5)
    else:
        s = {1: inputs.config1, 3: inputs.config3, 4: inputs.config4}[cfg]()
    P = Params.from_numpy(*s.params(), device=device)
    views = torch.as_tensor(s.views, device=device)
    V = views.shape[0]
    tc, td = {}, {}
    if "target_params" in s.extra:
        # targets = renders of the perturbed copy, rendered by this path at setup
        Pt = Params.from_numpy(*s.extra["target_params"], device=device)
        r = Rasterizer(s.n, s.cam, device=device)
        for v in range(rank, V, world):
            r.size_for(Pt, views[v])
            r.forward(Pt, views[v])
            tc[v] = r.frame.color.clone()
            td[v] = r.frame.depth.clone()
        del r
    else:
        for v in range(V):
            tc[v] = torch.as_tensor(s.extra["tgt_color"][v], device=device)
            td[v] = torch.as_tensor(s.extra["tgt_depth"][v], device=device)
    torch.cuda.synchronize()
    return s, P, views, tc, td


def union_ms(intervals):
    """Length of the union of [t0, t1] intervals (ms)."""
    tot, end = 0.0, None
    for t0, t1 in sorted(intervals):
        if end is None or t0 > end:
            tot += t1 - t0
            end = t1
        elif t1 > end:
            tot += t1 - end
            end = t1
    return tot


def active_ms(step_ms, evs, per_step):
    """Per step, the time at least one launch of a kernel is running: the
    union of its launches' CUDA-event intervals (on their lane streams),
    placed on the step's timeline by the step-start event."""
    out = []
    for i, (s0, _) in enumerate(step_ms):
        iv = [(s0.elapsed_time(e0), s0.elapsed_time(e1)) for e0, e1 in evs[i * per_step:(i + 1) * per_step]]
        out.append(union_ms(iv))
    return statistics.mean(out)


def roofline_for(step, stats_views, peaks, sm_mhz, fwd_ms, bwd_ms, fwd_active=None, bwd_active=None):
    """FP32-pipe roofline of the compositing kernels.

    Algorithmic flops: forward 10 s + 11 c per pixel, backward
    10 r + 64 c per pixel (r = entries replayed = n_contrib, c = composited).
    Peak = 148 SMs x 128 FP32 lanes x 2 flop x the SM clock measured during the
    run (no measured FP32 peak exists in MEASURED_PEAKS.json)."""
    s = sum(x["scanned"] for x in stats_views)
    c = sum(x["contrib"] for x in stats_views)
    r = sum(x["replayed"] for x in stats_views)
    nv = len(stats_views)
    fwd_flops = (10 * s + 11 * c) / nv     # per launch (one view)
    bwd_flops = (10 * r + 64 * c) / nv
    mhz = sm_mhz or peaks.get("sm_max_mhz", 1965.0)
    peak = 148 * 128 * 2 * mhz * 1e6 / 1e12
    out = {}
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):  # dram bytes of the dominant kernel from the committed ncu --set full capture
        traffic = json.load(open(tp)).get("dram_bytes_per_launch")
    for name, fl, ms, act in (("render_bwd_pixels", bwd_flops, bwd_ms, bwd_active),
                              ("render_fwd", fwd_flops, fwd_ms, fwd_active)):
        if act is not None:  # in-step: all launches of the step over the time any of them runs
            ach = fl * nv / (act * 1e-3) / 1e12 if act else None
        else:  # one launch alone
            ach = fl / (ms * 1e-3) / 1e12 if ms else None
        out[name] = {"bound": "alu", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                     "frac": ach / peak if ach else None,
                     "traffic": traffic if name == "render_bwd_pixels" else None, "flops_per_launch": fl,
                     "ms_per_launch": ms}
        if act is not None:
            out[name].update({"launches_per_step": nv, "ms_active_per_step": act,
                              "method": "algorithmic flops of the step's launches of this kernel / the time at "
                                        "least one of them runs (union of their CUDA-event intervals on the lane "
                                        "streams); launches of different views overlap in the step"})
    return out


def bench_ours(a):
    import torch
    import torch.distributed as dist
    from paper_2312_10070_b200 import raster
    from paper_2312_10070_b200.pipeline import MapStep, kernels_per_view

    world, rank, local = dist_env()
    if world != a.gpus:
        if a.gpus != 1 or world != 1:
            print(f"warning: --gpus {a.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    # one process per GPU; with --backend gloo (tests) several ranks may share one GPU
    local_dev = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local_dev)
    device = torch.device("cuda", local_dev)
    group = None
    if world > 1:
        if a.backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group("gloo")
    sm_count = raster.device_check(local_dev)
    s, P, views, tc, td = make_workload(a.config, device, rank, world, a.small)
    V = views.shape[0]
    ms = MapStep(P, views, s.cam, tc, td, rank, world, group, device=device, lanes=a.lanes)
    ms.size()
    # per-view work counts for the roofline (untimed)
    stats_views = []
    for v in ms.mine:
        ms.r.forward(P, views[v], stats=True)
        st = ms.r.frame.stats
        stats_views.append({"scanned": int(st[0].sum().item()), "contrib": int(st[1].sum().item()),
                            "replayed": int(ms.r.frame.n_contrib.sum().item()),
                            "pairs": int(ms.r.n_pairs.item())})
    torch.cuda.synchronize()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)
    stream = torch.cuda.current_stream()

    # events around the dominant kernels inside the timed steps (on their lane stream)
    ev_fwd, ev_bwd = [], []

    def timed_fwd(r, k, v, tgt_ready=None):
        # MapStep.stage_fwd with CUDA events around the compositing launch
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if ms.fused_loss and ms.ssim == 0.0:
            if tgt_ready is not None:
                st.wait_event(tgt_ready)
            if r.loss_part is None:
                r.loss_part = torch.empty(2 * r.T, dtype=torch.float64, device=r.device)
            order = ms.fwd_order(r, v)
            e0.record(st)
            raster.gs_render_fwd_l1(r.proj, r.sorted_idx, r.tile_range, r.cam, r.frame, ms.tgt_color[v],
                                    ms.tgt_depth[v], ms.tgt_scales[v], r.dL_dcolor, r.dL_ddepth,
                                    tile_order=r.tile_order if order is None else order, tile_work=r.tile_work,
                                    loss_part=r.loss_part)
            e1.record(st)
            ms._lane_view[id(r)] = v
            raster.gs_tile_order(r.tile_work, r.T, r.bwd_order)
            raster.gs_loss_from_tiles(r.cam, r.loss_part, ms.tgt_scales[v], ms.lc, ms.ld, r.loss)
        else:
            e0.record(st)
            raster.gs_render_fwd(r.proj, r.sorted_idx, r.tile_range, r.cam, r.frame, False, tile_order=r.tile_order,
                                 tile_work=r.tile_work)
            e1.record(st)
            raster.gs_tile_order(r.tile_work, r.T, r.bwd_order)
            if tgt_ready is not None:
                st.wait_event(tgt_ready)
            r.compute_loss(ms.tgt_color[v], ms.tgt_depth[v], None, ms.lc, ms.ld, ms.ssim)
        ev_fwd.append((e0, e1))
        ms.losses[k].copy_(r.loss)

    def timed_bwd(r, k, v):
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r.backward(ms.params, ms.views[v], raster.GS_GRAD_PARAMS | raster.GS_BWD_PIXELS_ONLY, ms.grads,
                   event_pair=(b0, b1))
        ev_bwd.append((b0, b1))

    hooks = {"fwd": timed_fwd, "bwd": timed_bwd}
    ms.overlap = not a.no_overlap

    # the timed steps run the product path as is: MapStep.step() captured once
    # as a CUDA graph and replayed (MapStep.capture / replay; one process),
    # or launched eagerly (--no-graph, and every multi-process run)
    for _ in range(max(a.warmup, 3)):
        ms.step()
    torch.cuda.synchronize()
    use_graph = world == 1 and not a.no_graph
    if use_graph:
        ms.capture()
        for _ in range(2):
            ms.replay()
        torch.cuda.synchronize()
    run_step = ms.replay if use_graph else ms.step
    if world > 1:
        dist.barrier()
    step_ms = []
    with Clocks(local_dev) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for _ in range(a.steps):
            flush.zero_()  # L2 flush between timed steps (outside the step events)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run_step()
            e1.record(stream)
            step_ms.append((e0, e1))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    clocks = clk.summary()
    per_step = [e0.elapsed_time(e1) for e0, e1 in step_ms]
    tot = sum(per_step)
    # secondary (in-step) roofline: a few more steps with CUDA events around the
    # compositing launches on their lane streams (stream-ordered stages: events
    # between the forward and the backward would defeat their tile overlap)
    inst_steps = []
    for i in range(2 + max(3, a.steps // 3)):
        if i == 2:
            ev_fwd.clear()
            ev_bwd.clear()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ms.step(hooks)
        e1.record(stream)
        if i >= 2:
            inst_steps.append((e0, e1))
    torch.cuda.synchronize()
    fwd_ms = statistics.mean(e0.elapsed_time(e1) for e0, e1 in ev_fwd) if ev_fwd else None
    bwd_ms = statistics.mean(e0.elapsed_time(e1) for e0, e1 in ev_bwd) if ev_bwd else None
    t = torch.tensor([tot], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / a.steps
    W, H = s.cam.width, s.cam.height
    mp = V * W * H / 1e6
    value = mp / (ms_per_step * 1e-3)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    nvw = len(ms.mine)
    roof = roofline_for(ms, stats_views, peaks, clocks.get("sm_mhz"), fwd_ms, bwd_ms,
                        active_ms(inst_steps, ev_fwd, nvw), active_ms(inst_steps, ev_bwd, nvw))
    # the same kernels timed alone (one view at a time, no other stream active;
    # skipped under --profile so that ncu's launch list ends with a step)
    iso_f, iso_b = [], []
    r0 = ms.lanes[0]
    fused = ms.fused_loss and ms.ssim == 0.0
    for v in ([] if a.profile else ms.mine):
        for rep in range(4):  # the first pass of a view sets its launch order (as a step does); 3 timed after
            e0, e1, e2, e3 = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            r0.project(P, views[v])
            r0.bin_sort()
            if fused:  # the compositing kernel the step runs (S3 + S4 fused), in the step's launch order
                if r0.loss_part is None:
                    r0.loss_part = torch.empty(2 * r0.T, dtype=torch.float64, device=r0.device)
                order = ms.fwd_order(r0, v)
                e0.record()
                raster.gs_render_fwd_l1(r0.proj, r0.sorted_idx, r0.tile_range, r0.cam, r0.frame, tc[v], td[v],
                                        ms.tgt_scales[v], r0.dL_dcolor, r0.dL_ddepth,
                                        tile_order=r0.tile_order if order is None else order,
                                        tile_work=r0.tile_work, loss_part=r0.loss_part)
                e1.record()
                ms._lane_view[id(r0)] = v
                raster.gs_tile_order(r0.tile_work, r0.T, r0.bwd_order)
            else:
                e0.record()
                raster.gs_render_fwd(r0.proj, r0.sorted_idx, r0.tile_range, r0.cam, r0.frame, False,
                                     tile_order=r0.tile_order, tile_work=r0.tile_work)
                e1.record()
                raster.gs_tile_order(r0.tile_work, r0.T, r0.bwd_order)
                r0.compute_loss(tc[v], td[v], None, ms.lc, ms.ld)
            r0.backward(P, views[v], raster.GS_GRAD_PARAMS | raster.GS_BWD_PIXELS_ONLY, ms.grads, event_pair=(e2, e3))
            r0.backward(P, views[v], raster.GS_GRAD_PARAMS | raster.GS_BWD_GAUSS_ONLY, ms.grads)
            torch.cuda.synchronize()
            if rep:
                iso_f.append(e0.elapsed_time(e1))
                iso_b.append(e2.elapsed_time(e3))
    roof_iso = roofline_for(ms, stats_views, peaks, clocks.get("sm_mhz"), statistics.median(iso_f),
                            statistics.median(iso_b)) if iso_f else {"render_fwd": None, "render_bwd_pixels": None}
    launches = (ms.launches_per_step() + 0) * a.steps
    q = np.percentile(per_step, [10, 50, 90])  # this rank's step-time spread (ms)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": max(a.warmup, 3),
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "ms_per_step_p10_p50_p90": [float(x) for x in q],
        "dtype": "f32", "data": "synthetic (seeded BJ.configs[%d] generator; targets = render of a perturbed copy)"
        % a.config,
        "config": {"workload": (f"BJ.configs[{a.config}] sub-map mapping iteration" if not a.small else
                                "BJ.configs[3] reduced (40k Gaussians, 4 views of 320x184; tests only)"),
                   "gaussians": s.n,
                   "width": W, "height": H, "views_per_step": V, "views_per_rank": len(ms.mine),
                   "parallelism": (f"view-sharded dp{world}, {a.backend.upper()} all-reduce of gradients"
                                   if world > 1 else "1 GPU"),
                   "l2": "256 MiB buffer written between timed steps (outside the step events)",
                   "launch": ("MapStep.capture(): the step as one CUDA graph, replayed" if use_graph else
                              "MapStep.step() launched eagerly"),
                   "pairs_per_view": int(np.mean([x["pairs"] for x in stats_views])),
                   "scanned_per_px": sum(x["scanned"] for x in stats_views) / (len(stats_views) * W * H),
                   "contrib_per_px": sum(x["contrib"] for x in stats_views) / (len(stats_views) * W * H)},
        # primary: the dominant kernel timed alone (CUDA events on its stream, median of 3 x views);
        # the in-step figures (launches of several views overlap on the lane streams) are secondary
        "roofline": roof_iso["render_bwd_pixels"] if roof_iso["render_bwd_pixels"] else roof["render_bwd_pixels"],
        "roofline_other": {"render_fwd_isolated": roof_iso["render_fwd"],
                           "render_bwd_pixels_in_step": roof["render_bwd_pixels"],
                           "render_fwd_in_step": roof["render_fwd"],
                           "note": "isolated = one launch timed alone (median of 3 x views); in_step = the step's "
                                   "launches of the kernel over the union of their CUDA-event intervals (the lane "
                                   "streams run several views concurrently)"},
        "clocks": clocks, "gpu_launches": launches, "sm_count": sm_count,
    }
    if not a.profile:  # the same step with Eq. 10's SSIM colour term (lambda = 0.2), every rank
        ms.ssim = 0.2
        for _ in range(3):
            ms.step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        nss = max(3, a.steps // 2)
        for _ in range(nss):
            ms.step()
        e1.record(stream)
        torch.cuda.synchronize()
        ms.ssim = 0.0
        t_ss = torch.tensor([e0.elapsed_time(e1) / nss], dtype=torch.float64, device=device)
        if world > 1:
            dist.all_reduce(t_ss, op=dist.ReduceOp.MAX)
        line["mapping_ssim"] = {"metric": METRIC + ", colour loss with Eq. 10's SSIM term (lambda = 0.2)",
                                "value": mp / (float(t_ss.item()) * 1e-3), "unit": UNIT,
                                "ms_per_step": float(t_ss.item())}
    if not a.profile:  # NEXT(3) epilogue: Eq. 11 + Adam over all Gaussians (after the all-reduce)
        from paper_2312_10070_b200.raster import Optimizer
        opt = Optimizer(s.n, device)
        Pc = type(P)(*[getattr(P, k).clone() for k in ("mean_opa", "quat", "logscale", "rgb")])
        for _ in range(3):
            opt.regularize(Pc, ms.grads, 1.0)
            opt.step(Pc, ms.grads)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(20):
            opt.regularize(Pc, ms.grads, 1.0)
            opt.step(Pc, ms.grads)
        e1.record(stream)
        torch.cuda.synchronize()
        t_opt = e0.elapsed_time(e1) / 20
        # algorithmic bytes: Eq. 11 reads log-scales and read-modify-writes their gradients (48 B);
        # Adam reads 4 gradients (64 B) and read-modify-writes 4 parameters (128 B) and 8 moments (256 B)
        nbytes = s.n * (48 + 64 + 128 + 256)
        line["optimizer"] = {"what": "Eq. 11 regulariser + one Adam step over all %d Gaussians" % s.n,
                             "ms": t_opt, "achieved_gbs": nbytes / (t_opt * 1e-3) / 1e9,
                             "hbm_peak_gbs": peaks.get("hbm_gbs"), "bytes": nbytes}
    if not a.profile:  # NEXT(4): seeding one keyframe against the 500k-Gaussian sub-map
        from paper_2312_10070_b200.raster import gs_seed, lib as _gslib
        r0 = ms.lanes[0]
        r0.forward(P, views[0])
        alpha = r0.frame.alpha.clone()
        depth = (r0.frame.depth / alpha.clamp_min(1e-6)).contiguous()
        H_, W_ = alpha.shape
        alpha[H_ // 4:3 * H_ // 4, W_ // 4:3 * W_ // 4] = 0.0  # an unmapped window: every pixel a candidate
        cap = s.n + 50000
        Ps = type(P)(*[torch.cat([getattr(P, k), torch.zeros(50000, 4, device=device)]).contiguous()
                       for k in ("mean_opa", "quat", "logscale", "rgb")])
        sws = torch.empty((_gslib().gs_seed_workspace_bytes(r0.cam, s.n, 50000) + 15) // 16 * 4,
                          dtype=torch.float32, device=device)
        n_new = torch.zeros(1, dtype=torch.int32, device=device)
        vh = views[0].cpu()
        for _ in range(2):
            gs_seed(r0.cam, vh, r0.frame.color, depth, alpha, 0.6, 0.01, 50000, 1, Ps, s.n, sws, n_new)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(10):
            gs_seed(r0.cam, vh, r0.frame.color, depth, alpha, 0.6, 0.01, 50000, 1, Ps, s.n, sws, n_new)
        e1.record(stream)
        torch.cuda.synchronize()
        line["seeding"] = {"what": "gs_seed: M_k = 50000 alpha-gated samples of a 1200x680 keyframe against "
                                   "%d existing Gaussians (rho = 1 cm)" % s.n,
                           "ms": e0.elapsed_time(e1) / 10, "accepted": int(n_new.item()), "capacity": cap}
    if not a.profile and not a.no_e2e:  # every rank: the step contains the all-reduce
        line["e2e"] = e2e_ours(a, s, ms, device, world)
    if world > 1:
        dist.barrier()
    if rank == 0 and world == 1 and not a.profile and not a.no_tracking:
        line["scaling_budget"] = scaling_budget(a, s, P, views, tc, td, device, ms_per_step)
        line["single_view"] = bench_single_view(device, a)
        line["tracking"] = bench_tracking(device)
        line["tracking_masked"] = bench_tracking(device, masked=(0.5, 50.0))
    if rank == 0 and world == 1 and not a.profile and not a.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(a, s)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def e2e_ours(a, s, ms, device, world=1):
    """Same metric through the public API with HOST buffers: every step copies
    its inputs (Gaussian parameters, view poses, this rank's RGB-D frames as
    8-bit RGB + 16-bit depth, R42) from pinned host memory and reads the
    per-view losses back (MapStep.step(host=...): the frames of later views
    upload while earlier views compute, and a step's uploads overlap the
    previous step's compute through two alternating device input sets)."""
    import torch
    from paper_2312_10070_b200.pipeline import HostInputs
    host = HostInputs(ms.params, ms.views, ms.tgt_color, ms.tgt_depth, ms.mine, ms.losses.shape[0])
    for _ in range(2):
        ms.step(host=host)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = max(3, a.steps // 2)
    for _ in range(n):
        ms.step(host=host)
    e1.record()
    torch.cuda.synchronize()
    ms_step = e0.elapsed_time(e1) / n
    if world > 1:  # max over ranks
        t = torch.tensor([ms_step], dtype=torch.float64, device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_step = float(t.item())
    mp = ms.V * s.cam.width * s.cam.height / 1e6
    return {"value": mp / (ms_step * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(host.h2d_bytes()),
            "d2h_bytes_per_step": int(host.d2h_bytes()), "ms_per_step": ms_step,
            "note": "inputs (parameters, poses, this rank's 8-bit RGB + 16-bit depth frames) uploaded every step; "
                    "the per-view losses are read back; the gradient buffer stays on the device, where the "
                    "optimiser (gs_adam_step) consumes it"}


def scaling_budget(a, s, P, views, tc, td, device, ms_1gpu):
    """Strong-scaling budget of the view-sharded step on this one GPU: the
    measured step time of rank 0's share at k = 2, 4, 8 ranks (its views only,
    no all-reduce), plus a MODELLED NCCL all-reduce of the [4][N][4] fp32
    gradient buffer at the pool's measured 8-rank bus bandwidth (725 GB/s,
    B200_PROFILING.md): t_AR = 2 (k - 1) / k x bytes / busbw.  The projection
    is T(1) / (t_share + t_AR); the driver's own multi-GPU runs supersede it."""
    import torch
    from paper_2312_10070_b200.pipeline import MapStep
    busbw = 725e9
    nbytes = 4 * s.n * 16
    out = {"model": "projected_speedup = T(1) / (measured rank-0 share + modelled all-reduce); busbw 725 GB/s "
                    "(measured 8-rank all-reduce on this pool); not a multi-GPU measurement",
           "l2": "256 MiB buffer written between timed shares (as for T(1))",
           "allreduce_bytes": nbytes}
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)
    for k in (2, 4, 8):
        ms = MapStep(P, views, s.cam, tc, td, rank=0, world=k, allreduce=lambda buf: None, device=device,
                     lanes=a.lanes)
        ms.overlap = not a.no_overlap
        ms.size()
        for _ in range(3):
            ms.step()
        torch.cuda.synchronize()
        run_step = ms.step
        if not a.no_graph:  # launched as T(1) is: captured once (the all-reduce is modelled, not run)
            ms.allreduce = None
            ms.capture()
            run_step = ms.replay
        t = []
        for _ in range(max(10, a.steps // 2)):
            flush.zero_()  # L2 flushed between timed shares, as for T(1) (outside the events)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run_step()
            e1.record()
            t.append((e0, e1))
        torch.cuda.synchronize()
        share = statistics.median(e0.elapsed_time(e1) for e0, e1 in t)
        ar = 2 * (k - 1) / k * nbytes / busbw * 1e3
        out[f"k{k}"] = {"views_per_rank": len(ms.mine), "ms_share": share, "ms_allreduce_model": ar,
                        "projected_speedup": ms_1gpu / (share + ar), "step": "MapStep"}
        del ms
    return out


def bench_single_view(device, a):
    """BJ.configs[1]: one 640x480 view of 100k Gaussians, fwd + bwd w.r.t. all
    parameters per step (project, bin_sort, render with the fused L1 loss,
    per-pixel and per-Gaussian backward; one stream), MP/s = 0.3072 / step."""
    import torch
    from paper_2312_10070_b200 import Params, inputs
    from paper_2312_10070_b200.pipeline import MapStep
    s = inputs.config1()
    P = Params.from_numpy(*s.params(), device=device)
    views = torch.as_tensor(s.views, device=device)
    tc = {0: torch.as_tensor(s.extra["tgt_color"][0], device=device)}
    td = {0: torch.as_tensor(s.extra["tgt_depth"][0], device=device)}
    ms = MapStep(P, views, s.cam, tc, td, device=device, lanes=1)
    ms.overlap = not a.no_overlap
    ms.size()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)
    for _ in range(5):
        ms.step()
    torch.cuda.synchronize()
    run_step = ms.step
    if not a.no_graph:  # as the main line: the step captured once, replayed
        ms.capture()
        run_step = ms.replay
    t = []
    for _ in range(max(a.steps, 20)):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run_step()
        e1.record()
        t.append((e0, e1))
    torch.cuda.synchronize()
    ms_step = [e0.elapsed_time(e1) for e0, e1 in t]
    med = statistics.median(ms_step)
    mp = s.cam.width * s.cam.height / 1e6
    return {"metric": "fwd+bwd megapixels/s, one 640x480 view of 100k Gaussians (BJ.configs[1])",
            "value": mp / (med * 1e-3), "unit": UNIT, "ms_per_step_median": med,
            "ms_per_step_p10_p90": [float(x) for x in np.percentile(ms_step, [10, 90])],
            "gpu_launches_per_step": ms.launches_per_step(), "l2": "256 MiB buffer written between steps",
            "launch": "CUDA graph replay" if not a.no_graph else "eager", "overlap": ms.overlap}


def bench_tracking(device, masked=None):
    """BJ.configs[2]: 200k Gaussians, 1200x680, 100 pose iterations in one CUDA graph
    (masked = (lambda_c, inlier_mult): the Eq. 15 masked loss instead of L1)."""
    import torch
    from paper_2312_10070_b200 import Params, Rasterizer, inputs
    from paper_2312_10070_b200.pipeline import TrackingLoop
    s = inputs.config2()
    P = Params.from_numpy(*s.params(), device=device)
    gt = torch.as_tensor(s.extra["gt_view"], device=device)
    r = Rasterizer(s.n, s.cam, device=device)
    r.size_for(P, gt)
    r.forward(P, gt)
    tc, td = r.frame.color.clone(), r.frame.depth.clone()
    del r
    loop = TrackingLoop(P, s.cam, tc, td, torch.as_tensor(s.extra["start_view"], device=device), iters=100,
                        masked=masked)
    loop.size()
    loop.capture()
    for _ in range(2):
        loop.run()
    torch.cuda.synchronize()
    times = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        loop.reset()
        e0.record()
        loop.graph.replay()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    med = statistics.median(times)
    v = loop.view.cpu().numpy().astype(np.float64)
    R, t = v[:9].reshape(3, 3), v[9:]
    rot_err = np.degrees(np.arccos(np.clip((np.trace(R) - 1) / 2, -1, 1)))
    sv = s.extra["start_view"].astype(np.float64)
    rot0 = np.degrees(np.arccos(np.clip((np.trace(sv[:9].reshape(3, 3)) - 1) / 2, -1, 1)))
    return {"metric": "tracking iterations/s (BJ.configs[2], 200k Gaussians, 1200x680)",
            "loss": "L1 colour + L1 depth (BJ.configs[2])" if masked is None else
                    "Eq. 15 masked: alpha^3 x inlier (50 x median), lambda_c = %g" % masked[0],
            "value": 100 / (med * 1e-3), "unit": "iter/s", "ms_per_iter": med / 100,
            "graph": ("100 iterations captured once (project, sort, render with the L1 gradient maps fused "
                      "(gs_render_fwd_l1; scales once per frame), pose bwd, pose grad + Adam)") if masked is None else
                     "100 iterations captured once (project, sort, render, loss, pose bwd, pose grad + Adam)",
            "gpu_launches_per_iter": loop.launches_per_iter(),
            "flag_timeouts": loop.flag_timeouts(),
            "start_err": {"rot_deg": float(rot0), "trans_cm": float(np.linalg.norm(sv[9:]) * 100)},
            "final_err": {"rot_deg": float(rot_err), "trans_cm": float(np.linalg.norm(t) * 100)}}


def cpu_baseline(a, s, max_views=None):
    """The fp64 oracle as it stands, on this host's cores: the full mapping step
    (projection, binning, compositing, L1 loss and backward of every pixel) of
    the first `max_views` views of the workload (all of them by default)."""
    import oracle
    t0 = time.perf_counter()
    p64 = oracle.params64(*s.params())
    cam = s.cam
    V = s.views.shape[0] if max_views is None else min(max_views, s.views.shape[0])
    tp = oracle.params64(*s.extra["target_params"]) if "target_params" in s.extra else None
    tsum = 0.0
    for v in range(V):
        view = s.views[v].astype(np.float64)
        if tp is not None:  # targets (not timed): the oracle's own render of the perturbed copy
            tgt = oracle.forward(tp, view, cam)
            tc_, td_ = tgt["color"], tgt["depth"]
        else:
            tc_, td_ = s.extra["tgt_color"][v], s.extra["tgt_depth"][v]
        ta = time.perf_counter()
        fr = oracle.forward(p64, view, cam)
        _, gc, gd = oracle.loss(cam, fr["color"], fr["depth"], tc_, td_, None, 1.0 / V, 1.0 / V)
        oracle.backward(p64, view, cam, fr["sorted_idx"], fr["tile_range"], gc, gd)
        tsum += time.perf_counter() - ta
    mp = V * cam.width * cam.height / 1e6
    return {"value": mp / tsum, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"{V} of {s.views.shape[0]} views of BJ.configs[{a.config}], every pixel (projection, binning, "
                      f"compositing, L1 loss, backward incl. gradient magnitude scales); {tsum:.1f} s timed, "
                      f"{time.perf_counter() - t0:.1f} s with target renders",
            "s_per_view": tsum / V}


def bench_reference(a):
    """--impl reference: the fp64 oracle timed on the host cores (rank 0 only)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    from paper_2312_10070_b200 import inputs
    s = {1: inputs.config1, 3: inputs.config3, 4: inputs.config4}[a.config]()
    oracle.build()
    # each "step" is a bounded sample: one view of the workload (warm-up steps are not timed)
    vals = []
    for i in range(a.warmup + a.steps):
        r = cpu_baseline(a, s, max_views=1)
        if i >= a.warmup:
            vals.append(r)
    v = statistics.median(x["value"] for x in vals)
    per_view = statistics.median(x["s_per_view"] for x in vals)
    V = s.views.shape[0]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": per_view * V * 1e3,
            "ms_per_step_note": f"extrapolated: the median timed 1-view sample x {V} views (each timed step is one "
                                f"view of the {V}-view workload)",
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator)",
            "config": {"workload": f"BJ.configs[{a.config}] sub-map mapping iteration (oracle, sampled)",
                       "gaussians": s.n, "width": s.cam.width, "height": s.cam.height, "views_per_step": V},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": vals[0]["cores"], "kind": "oracle",
                             "sample": vals[0]["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    if a.impl == "reference":
        bench_reference(a)
    else:
        bench_ours(a)


if __name__ == "__main__":
    main()
