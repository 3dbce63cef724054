"""Orchestration of the C-ABI calls for the two optimisations of Gaussian-SLAM.

* ``MapStep`` — one multi-view sub-map mapping iteration (Eq. 12
  colour L1 + depth L1 terms): for each keyframe view of this rank
  gs_project -> gs_bin_sort -> gs_render_fwd -> gs_loss -> gs_render_bwd,
  gradients accumulated (+=) into one contiguous buffer, then one NCCL
  all-reduce (SUM) across ranks when world_size > 1.  The
  1/V view mean is folded into gs_loss's lambdas, so the SUM is the mean.
* ``TrackingLoop`` — frame-to-model tracking (Eqs. 14): K
  iterations of render -> L1 loss -> pose-only backward -> gs_pose_grad with
  the device-side Adam step, captured once in a CUDA graph (no host sync).

No arithmetic of the method happens here: only buffer management and the
order of calls.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .raster import (GS_BWD_ATOMIC_ACC, GS_BWD_GAUSS_ONLY, GS_BWD_PIXELS_ONLY, GS_GRAD_PARAMS, GS_GRAD_POSE, Grads, Params, Rasterizer,
                     gs_loss_scales, gs_unpack_rgbd, lib)


class HostInputs:
    """Pinned host buffers of one mapping step's inputs (parameters, view
    poses, this rank's RGB-D targets) and its per-view loss output.

    frames="rgbd16" (default): the targets are held as the sensors' frames,
    8-bit RGB [H][W][3] + 16-bit depth [H][W] in units of depth_scale
    (R42), uploaded as such and unpacked on the
    device (gs_unpack_rgbd); frames="f32": fp32 planar targets, uploaded as is."""

    def __init__(self, params: Params, views, tgt_color, tgt_depth, mine, n_losses, frames="rgbd16",
                 depth_scale=None):
        from . import inputs
        pin = lambda t: t.detach().cpu().contiguous().pin_memory()
        self.params = {k: pin(getattr(params, k)) for k in ("mean_opa", "quat", "logscale", "rgb")}
        self.views = pin(views)
        self.frames = frames
        self.depth_scale = inputs.DEPTH_SCALE if depth_scale is None else depth_scale
        if frames == "rgbd16":
            self.rgb8, self.d16, self.dev_rgb8, self.dev_d16 = {}, {}, {}, {}
            for v in mine:
                r8, d16 = inputs.quantize_rgbd(tgt_color[v].cpu().numpy(), tgt_depth[v].cpu().numpy(),
                                               self.depth_scale)
                self.rgb8[v] = torch.from_numpy(r8).pin_memory()
                self.d16[v] = torch.from_numpy(d16.view(np.int16)).pin_memory()
                self.dev_rgb8[v] = torch.empty_like(self.rgb8[v], device=tgt_color[v].device)
                self.dev_d16[v] = torch.empty_like(self.d16[v], device=tgt_color[v].device)
        elif frames == "f32":
            self.tgt_color = {v: pin(tgt_color[v]) for v in mine}
            self.tgt_depth = {v: pin(tgt_depth[v]) for v in mine}
        else:
            raise ValueError(frames)
        self.mine = list(mine)
        self.loss = torch.empty(n_losses, 4, dtype=torch.float32).pin_memory()

    def upload_targets(self, v, cam, tgt_color, tgt_depth, scales=None, lambda_color=1.0, lambda_depth=1.0):
        """On the current (copy) stream: view v's frame into its device targets
        (and, if given, its gs_loss_scales into scales; returns whether it did)."""
        if self.frames == "rgbd16":
            self.dev_rgb8[v].copy_(self.rgb8[v], non_blocking=True)
            self.dev_d16[v].copy_(self.d16[v], non_blocking=True)
            gs_unpack_rgbd(cam, self.dev_rgb8[v], self.dev_d16[v], self.depth_scale, tgt_color, tgt_depth,
                           scales=scales, lambda_color=lambda_color, lambda_depth=lambda_depth)
            return scales is not None
        tgt_color.copy_(self.tgt_color[v], non_blocking=True)
        tgt_depth.copy_(self.tgt_depth[v], non_blocking=True)
        return False

    def h2d_bytes(self):
        b = sum(t.numel() * t.element_size() for t in self.params.values()) + self.views.numel() * 4
        if self.frames == "rgbd16":
            return b + sum(self.rgb8[v].numel() + 2 * self.d16[v].numel() for v in self.mine)
        return b + sum(t.numel() * 4 for t in self.tgt_color.values()) + sum(t.numel() * 4 for t in self.tgt_depth.values())

    def d2h_bytes(self):
        return self.loss.numel() * 4


def shard_views(n_views, rank, world):
    """Round-robin view assignment: rank r takes views r, r + world, ..."""
    return list(range(rank, n_views, world))


class MapStep:
    """One mapping iteration over this rank's views.

    Views are pipelined over `lanes` CUDA streams (default 8: every view of a BJ.configs[3] step in flight), each with its own
    Rasterizer buffers: the latency-bound sort / loss kernels of one view
    overlap the compute-bound compositing kernels of another.  The
    per-Gaussian phases of gs_render_bwd add into the shared gradient buffer
    atomically (GS_BWD_ATOMIC_ACC), so no view waits for another.
    """

    def __init__(self, params: Params, views, cam, tgt_color, tgt_depth, rank=0, world=1, group=None,
                 lambda_color=1.0, lambda_depth=1.0, device="cuda", lanes=8, allreduce=None,
                 ssim=0.0, atomic_gauss=True, fused_loss=True, ar_chunks=None):
        """ssim: the lambda of Eq. 10's colour loss (0: L1 colour only, as
        BJ.configs[3]; the paper uses 0.2).  atomic_gauss: the
        per-view S6 adds into the gradient buffer atomically
        (GS_BWD_ATOMIC_ACC), so the views' Gaussian phases need no ordering;
        else they are serialised in view order (events).  fused_loss (L1
        loss, ssim = 0): the loss is computed by the compositing kernel
        (gs_render_fwd_l1, per-view scales from prepare_targets).
        ar_chunks (world > 1): the per-Gaussian phase runs in this many
        Gaussian ranges and each range's gradients (four contiguous component
        slices) are all-reduced on a communication stream as soon as every
        view has chained it, so the reduction overlaps the rest of S6
        (default 1: one all-reduce of the whole buffer after S6; the chunked
        form is correct on 2 ranks (tests) but its speed needs > 1 GPU to
        measure)."""
        self.ssim = ssim
        self.params = params
        self.views = views                  # [V, 12] device tensor (all views)
        self.V = views.shape[0]
        self.mine = shard_views(self.V, rank, world)
        self.tgt_color = tgt_color          # dict view -> [3,H,W] (only this rank's views needed)
        self.tgt_depth = tgt_depth
        self.world = world
        self.group = group
        # SUM across ranks (S8); default: NCCL through torch.distributed when world > 1
        self.allreduce = allreduce if allreduce is not None else (
            (lambda buf: torch.distributed.all_reduce(buf, op=torch.distributed.ReduceOp.SUM, group=group))
            if world > 1 else None)
        self.lc = lambda_color / self.V     # R20: mean over the V views of an iteration
        self.ld = lambda_depth / self.V
        nl = max(1, min(lanes, len(self.mine)))
        self.lanes = [Rasterizer(params.n, cam, device=device) for _ in range(nl)]
        self.streams = [torch.cuda.Stream(device=device) for _ in range(nl)]
        self.r = self.lanes[0]
        self.grads = Grads.zeros(params.n, device)
        # per view: (total, L1 colour, L1 depth, SSIM if ssim > 0)
        self.losses = torch.zeros(max(len(self.mine), 1), 4, dtype=torch.float32, device=device)
        self.copy_stream = None  # host-input uploads (created on the first step(host=...))
        # the upload stream runs at the highest CUDA stream priority: its
        # frame-unpacking kernels are scheduled ahead of the lanes' queued
        # compute CTAs, so the next step's targets are ready when its
        # forwards start (end to end at BJ.configs[3]: 2.85 -> 2.70 ms per step
        # against 2.58 device-resident; priorities -1 and -3 measure the same)
        self.copy_priority = None  # None: the highest (torch.cuda.Stream.priority_range()[1])
        self._slots = None
        self.fused_loss = fused_loss  # used while self.ssim == 0 (the L1 loss is pixel-local)
        self.tgt_scales = {}
        self.atomic_gauss = atomic_gauss
        self.ar_chunks = 1 if ar_chunks is None else max(1, int(ar_chunks))
        self.comm_stream = torch.cuda.Stream(device=device) if world > 1 else None
        # the forward of a view is launched in its previous step's work order
        # (the backward's heaviest-first order of the same view on the same
        # lane: the parameters move little between steps); scheduling only
        self.reuse_order = True
        self._lane_view = {}
        # overlap (fused L1 loss, a view whose lane rendered it last step): its
        # per-pixel backward starts tile by tile as its forward finishes
        # (per-tile flags + programmatic dependent launch, as in tracking), both
        # in the previous step's work order; the order refresh and the loss
        # reduction follow.  On by default since the end of round 2 (graph-
        # replayed step): 2534 -> 2537 MP/s at 8 views, the one-view share
        # 0.393 -> 0.388 ms, the 2-view share 0.708 -> 0.683 ms, single view
        # 1513 -> 1519 MP/s (first measured no faster, round 2 start)
        self.overlap = True
        self._pending = {}
        self.graph = None

    def fwd_order(self, r, v):
        """Tile launch order for view v's forward on lane r (None: gs_bin_sort's)."""
        return r.bwd_order if self.reuse_order and self._lane_view.get(id(r)) == v else None

    def size(self, slack=1.25):
        """Setup only (host sync): pair capacity = slack x max pairs over my views."""
        best = 0
        r = self.lanes[0]
        for v in self.mine:
            r.project(self.params, self.views[v])
            r.set_capacity(max(r.capacity, 1))
            r.bin_sort()
            torch.cuda.synchronize()
            best = max(best, int(r.n_pairs.item()))
        for r in self.lanes:
            r.set_capacity(int(best * slack) + 1024)
            r.counters[2].zero_()  # the sizing passes' own overflows
        if self.fused_loss:
            self.prepare_targets()
        return best

    def overflowed(self, collective=True):
        """Host sync: pair-capacity overflows the lanes' gs_bin_sort calls
        recorded (gs_counters.n_overflow; an overflowing view is rendered
        empty) since the lanes' counters were last zeroed.  With world > 1
        (and a process group) the MAX over ranks — a collective every rank
        must call — so that all ranks take the same repeat decision."""
        n = torch.stack([r.counters[2] for r in self.lanes]).sum().reshape(1)
        if collective and self.world > 1 and torch.distributed.is_available() and torch.distributed.is_initialized():
            torch.distributed.all_reduce(n, op=torch.distributed.ReduceOp.MAX, group=self.group)
        return int(n.item())

    def step_checked(self, hooks=None, host=None, slack=1.25):
        """step(); then, if a view of ANY rank overflowed its pair capacity,
        every rank re-sizes its lanes and runs the step again (host sync; the
        decision is collective, so the ranks' all-reduces stay paired, and the
        repeated step starts from zeroed gradients).  For loops whose
        Gaussians change between steps (mapping with the optimiser)."""
        g = self.step(hooks, host)
        if self.overflowed():
            self.size(slack)
            g = self.step(hooks, host)
        return g

    def capture(self):
        """The device-resident step (no host inputs, no hooks) captured once as
        one CUDA graph over the lane streams; replay() then runs it with a few
        µs of host work instead of ~1.5 ms of Python launches per step
        (tools/graph_exp.py).  Single process only (the graph holds no
        collective).  The captured step uses the lanes' state at capture time
        (work orders, overlap path): capture after a few warm-up steps, and
        again after re-sizing."""
        if self.allreduce is not None:
            raise ValueError("MapStep.capture: world > 1 (the all-reduce is not captured)")
        main = torch.cuda.current_stream()
        side = torch.cuda.Stream(device=self.params.mean_opa.device)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            self.step()  # warm-up on a side stream (lazy buffers)
        main.wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.step()
        torch.cuda.synchronize()
        self.graph = g
        return g

    def replay(self):
        """One step by graph replay (capture() first); returns the gradients."""
        self.graph.replay()
        return self.grads

    # -- the four stages of one view ---------------------------------------------
    def stage_front(self, r, k, v):
        """S1 + S2: projection and binning (no launch order from the binning
        when the forward will reuse the lane's work order for this view)."""
        r.project(self.params, self.views[v])
        r.bin_sort(order=self.fwd_order(r, v) is None)

    def stage_fwd(self, r, k, v, tgt_ready=None):
        """S3 + S4 once the view's targets are on the device (tgt_ready):
        with fused_loss (L1, ssim = 0) one compositing kernel also writes the
        loss gradient maps and per-tile loss sums (gs_render_fwd_l1 +
        gs_loss_from_tiles); else compositing, then gs_loss (+ gs_ssim)."""
        if self.fused_loss and self.ssim == 0.0:
            if tgt_ready is not None:
                torch.cuda.current_stream().wait_event(tgt_ready)
            if self.overlap and self.reuse_order and self._lane_view.get(id(r)) == v:
                # the backward must be the next launch on this stream (stage_bwd)
                r.render_l1_overlapped(self.tgt_color[v], self.tgt_depth[v], self.tgt_scales[v])
                self._pending[id(r)] = (k, v)
                return
            r.render_l1(self.tgt_color[v], self.tgt_depth[v], self.lc, self.ld, self.tgt_scales[v],
                        order=self.fwd_order(r, v))
            self._lane_view[id(r)] = v
        else:
            r.render()
            if tgt_ready is not None:
                torch.cuda.current_stream().wait_event(tgt_ready)
            r.compute_loss(self.tgt_color[v], self.tgt_depth[v], None, self.lc, self.ld, self.ssim)
        self.losses[k].copy_(r.loss)

    def prepare_targets(self):
        """The per-view gradient scales of the fused L1 loss (gs_loss_scales,
        once per target frame): call again after changing the targets."""
        self.tgt_scales = {v: self.tgt_scales.get(v) if self.tgt_scales else None for v in self.mine}
        for v in self.mine:
            if self.tgt_scales[v] is None:
                self.tgt_scales[v] = torch.zeros(4, dtype=torch.float32, device=self.tgt_depth[v].device)
            self.lanes[0].loss_scales(self.tgt_depth[v], self.lc, self.ld, out=self.tgt_scales[v])

    def stage_bwd(self, r, k, v):
        """S5: the per-pixel backward phase (overlapped with its forward's
        tail when stage_fwd left it pending; then the next step's order and
        the loss value)."""
        if self._pending.pop(id(r), None) is not None:
            r.backward(self.params, self.views[v], GS_GRAD_PARAMS | GS_BWD_PIXELS_ONLY, self.grads, overlap=True)
            r.finish_l1(self.lc, self.ld, self.tgt_scales[v])
            self.losses[k].copy_(r.loss)
            return
        r.backward(self.params, self.views[v], GS_GRAD_PARAMS | GS_BWD_PIXELS_ONLY, self.grads)

    def stage_gauss(self, r, k, v):
        """S6: the per-Gaussian phase (+= into the shared gradient buffer)."""
        r.backward(self.params, self.views[v],
                   GS_GRAD_PARAMS | GS_BWD_GAUSS_ONLY | (GS_BWD_ATOMIC_ACC if self.atomic_gauss else 0), self.grads)

    def step(self, hooks=None, host=None):
        """One mapping iteration.  hooks: optional dict overriding stages
        ("front", "fwd", "bwd", "gauss") with functions of the same signature.

        View k runs all its stages on lane stream k % lanes (8 lanes: every
        view of a BJ.configs[3] step in flight), so the latency-bound binning
        of some views and the tails of the compositing launches of others
        fill each other's idle SMs; the per-Gaussian phases add atomically
        into the gradient buffer (or, with atomic_gauss=False, are serialised
        in view order by events).  (Measured and dropped in round 1: one
        stream per stage, 8% slower; one multi-view S6 after all pixel phases,
        3.61 vs 3.15 ms per step.)

        host: optional HostInputs (pinned host buffers of this step's inputs).
        A copy stream uploads the parameters and poses, then every view's
        RGB-D targets in view order; the front stage waits for the
        parameters, the loss only for its view's targets, so the uploads
        overlap compute.  The per-view losses are read back into host.loss."""
        st = {"front": self.stage_front, "fwd": self.stage_fwd, "bwd": self.stage_bwd, "gauss": self.stage_gauss}
        if hooks:
            st.update(hooks)
        main = torch.cuda.current_stream()
        tgt_ready = {v: None for v in self.mine}
        rgb_ready = None

        def fwd(r, k, v):  # the forward reads the colours: wait for their upload
            if rgb_ready is not None:
                torch.cuda.current_stream().wait_event(rgb_ready)
            st["fwd"](r, k, v, tgt_ready[v])
        slot = None
        if host is not None:
            if self.copy_stream is None:
                prio = self.copy_priority
                if prio is None:
                    prio = torch.cuda.Stream.priority_range()[1]
                self.copy_stream = torch.cuda.Stream(device=self.params.mean_opa.device, priority=prio)
                # two device input sets used alternately: the uploads of step
                # k + 1 overlap the compute of step k (they wait only for the
                # step that last read their set, k - 1)
                clone = Params(*(getattr(self.params, n).clone() for n in ("mean_opa", "quat", "logscale", "rgb")))
                if self.fused_loss and not self.tgt_scales:
                    self.prepare_targets()
                self._slots = [(self.params, self.views, self.tgt_color, self.tgt_depth, self.tgt_scales),
                               (clone, self.views.clone(), {v: t.clone() for v, t in self.tgt_color.items()},
                                {v: t.clone() for v, t in self.tgt_depth.items()},
                                {v: t.clone() for v, t in self.tgt_scales.items()})]
                self.scale_ws = torch.empty_like(self.lanes[0].loss_ws)
                self._released = [main.record_event(), main.record_event()]
                self._slot = 0
            slot = self._slot
            self._slot ^= 1
            self.params, self.views, self.tgt_color, self.tgt_depth, self.tgt_scales = self._slots[slot]
            cs = self.copy_stream
            cs.wait_event(self._released[slot])  # the step that last read this set is done
            with torch.cuda.stream(cs):
                # the projection's inputs first; the colours (read from the
                # forward on) and the frames follow while the fronts run
                for name in ("mean_opa", "quat", "logscale"):
                    getattr(self.params, name).copy_(host.params[name], non_blocking=True)
                self.views.copy_(host.views, non_blocking=True)
                params_ready = cs.record_event()
                self.params.rgb.copy_(host.params["rgb"], non_blocking=True)
                rgb_ready = cs.record_event()
                for v in self.mine:
                    # the new frame and (fused loss) its gradient scales, in the unpacking pass
                    done = host.upload_targets(v, self.r.cam, self.tgt_color[v], self.tgt_depth[v],
                                               self.tgt_scales[v] if self.fused_loss else None, self.lc, self.ld)
                    if self.fused_loss and not done:
                        gs_loss_scales(self.r.cam, self.tgt_depth[v], self.lc, self.ld, self.scale_ws,
                                       self.tgt_scales[v])
                    tgt_ready[v] = cs.record_event()  # also orders the colours before every loss
            main.wait_event(params_ready)
        self.grads.zero_()
        start = main.record_event()
        for s in self.streams:
            s.wait_event(start)
        chunked = (self.allreduce is not None and self.ar_chunks > 1 and self.atomic_gauss
                   and "gauss" not in (hooks or {}))
        bounds = self.chunk_bounds() if chunked else None
        chunk_ev = {}  # (lane, chunk) -> event after the lane's last view chained that chunk
        prev = start
        for k, v in enumerate(self.mine):
            lane = k % len(self.lanes)
            s, r = self.streams[lane], self.lanes[lane]
            with torch.cuda.stream(s):
                st["front"](r, k, v)
                fwd(r, k, v)
                st["bwd"](r, k, v)
                if not self.atomic_gauss:
                    s.wait_event(prev)
                if chunked:
                    for c, (i0, i1) in enumerate(bounds):
                        r.backward_gauss_range(self.params, self.views[v], self.grads, i0, i1,
                                               GS_GRAD_PARAMS | GS_BWD_ATOMIC_ACC)
                        chunk_ev[(lane, c)] = s.record_event()
                else:
                    st["gauss"](r, k, v)
                prev = s.record_event()
        if chunked:
            # S8 chunk by chunk on the communication stream (overlaps the rest of S6)
            cs = self.comm_stream
            cs.wait_event(start)
            with torch.cuda.stream(cs):
                for c, (i0, i1) in enumerate(bounds):
                    for lane in range(len(self.lanes)):
                        if (lane, c) in chunk_ev:
                            cs.wait_event(chunk_ev[(lane, c)])
                    for comp in range(4):  # each component slice [i0, i1) is contiguous
                        self.allreduce(self.grads.buf[comp, i0:i1])
        for s in self.streams:
            main.wait_stream(s)
        if host is not None:
            main.wait_stream(self.copy_stream)
        if chunked:
            main.wait_stream(self.comm_stream)
        elif self.allreduce is not None:
            self.allreduce(self.grads.buf)
        if host is not None:
            host.loss.copy_(self.losses, non_blocking=True)
            self._released[slot] = main.record_event()
        return self.grads

    def chunk_bounds(self):
        """Gaussian ranges of the chunked S6 / S8 (multiples of 128)."""
        n, c = self.params.n, self.ar_chunks
        step = ((n + c - 1) // c + 127) // 128 * 128
        return [(i, min(i + step, n)) for i in range(0, n, step)]

    def launches_per_step(self):
        """Kernels of ours launched per step; the fused L1
        loss takes 1 launch (gs_loss_from_tiles) instead of gs_loss's 3."""
        per_view = kernels_per_view(self.r.cam, capacity=self.r.capacity) - (
            2 if self.fused_loss and self.ssim == 0.0 else 0)
        return len(self.mine) * per_view


def kernels_per_view(cam, loss=True, bwd=True, capacity=0):
    """Kernels of ours per view (the sort's memset is a copy-engine node, not a kernel):
    project 1; bin_sort: prep, tile counts, emit, tile sort, mid-list sort,
    long-list sort = 6; render 1 + backward tile order 1; loss 3; backward 2.
    (capacity: kept for callers; the launches no longer depend on it.)"""
    n = 1 + 6 + 2
    if loss:
        n += 3
    if bwd:
        n += 2
    return n


class TrackingLoop:
    """K tracking iterations on one GPU, graph-captured."""

    def __init__(self, params: Params, cam, tgt_color, tgt_depth, start_view, iters=100, lambda_color=1.0,
                 lambda_depth=1.0, step=(2e-3, 1e-3, 0.9, 0.999, 1e-8), device="cuda", masked=None,
                 fused_loss=True):
        """masked: None for the L1 colour + depth loss of BJ.configs[2], or
        (lambda_c, inlier_mult) for the masked tracking loss of Eq. 15.
        fused_loss (L1 only): the gradient maps are written by the forward
        kernel (gs_render_fwd_l1, the same values as gs_loss) and no loss value
        is computed per iteration; else gs_loss runs after the forward."""
        self.masked = masked
        self.fused_loss = fused_loss
        self.reuse_order = True  # launch orders from the previous iteration (scheduling only)
        self.order_every = 4     # ... refreshed from the forward's work every 4 iterations (2930 -> 2941 it/s vs 8)
        self.overlap = True      # the backward starts tile by tile as the forward finishes (PDL)
        self.params = params
        self.r = Rasterizer(params.n, cam, device=device)
        self.tc, self.td = tgt_color, tgt_depth
        self.start = start_view.clone()
        self.view = start_view.clone()
        self.adam = torch.zeros(13, dtype=torch.float64, device=device)  # gs_pose_grad's fp64 Adam state
        self.dtwist = torch.zeros(6, dtype=torch.float32, device=device)
        self.iters = iters
        self.lc, self.ld = lambda_color, lambda_depth
        self.stepcfg = step
        self.graph = None

    def size(self, slack=1.5):
        P = self.r.size_for(self.params, self.view)
        self.r.set_capacity(int(P * slack) + 4096)
        return P

    def prepare(self):
        """Once per target frame: the L1 gradient scales (fused mode)."""
        if self.masked is None and self.fused_loss:
            self.r.loss_scales(self.td, self.lc, self.ld)

    def iteration(self, i=0):
        r = self.r
        if self.masked is None and self.fused_loss:
            # S1-S3 with the L1 gradient maps written by the forward (gs_render_fwd_l1)
            r.forward_l1(self.params, self.view, self.tc, self.td, reuse_order=self.reuse_order,
                         refresh_order=not self.reuse_order or i % self.order_every == 0, overlap=self.overlap)
        else:
            r.forward(self.params, self.view)
            if self.masked is None:
                r.compute_loss(self.tc, self.td, None, self.lc, self.ld)
            else:
                r.compute_tracking_loss(self.tc, self.td, *self.masked)
        r.backward(self.params, self.view, GS_GRAD_POSE, overlap=self.overlap and self.masked is None and self.fused_loss)
        r.pose_grad(self.view, self.stepcfg, self.adam, dL_dtwist=self.dtwist)

    def flag_timeouts(self):
        """Host sync: timed-out waits of the overlapped backward (must be 0;
        include/gs.h gs_render_bwd tile_done)."""
        return self.r.flag_timeouts()

    def reset(self):
        self.view.copy_(self.start)
        self.adam.zero_()

    def capture(self):
        self.reset()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.prepare()
            for _ in range(2):  # warm-up outside capture (lazy attributes, module load)
                self.iteration()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        self.reset()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.prepare()  # once per target frame, inside the timed graph
            for i in range(self.iters):
                self.iteration(i)
        self.graph = g
        return g

    def run(self):
        self.reset()
        if self.graph is None:
            self.prepare()
            for i in range(self.iters):
                self.iteration(i)
        else:
            self.graph.replay()

    def launches_per_iter(self):
        # masked loss: 6 kernels (residual + digit 0, 3 digit passes, apply, final) instead of 3;
        # fused L1: none (the forward writes the maps; + 2 per graph for the scales)
        if self.masked is None and self.fused_loss:
            return kernels_per_view(self.r.cam, capacity=self.r.capacity) + 1 - 3
        return kernels_per_view(self.r.cam, capacity=self.r.capacity) + 1 + (3 if self.masked is not None else 0)
