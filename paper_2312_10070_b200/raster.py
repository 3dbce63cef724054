"""Thin torch-facing binding of the C-ABI (include/gs.h).

Functions named like the C entry points (``gs_project`` ... ``gs_pose_grad``)
only marshal torch CUDA tensors into pointers and call the library on the
current torch stream: every step of the path runs in the CUDA kernels of
``csrc/``.  PyTorch is used for device memory, streams and process groups only.

``Rasterizer`` owns the buffers of one (N, camera) problem and strings the
calls together; ``Params`` / ``Grads`` hold the four float4 SoA arrays.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import (GS_BWD_ATOMIC_ACC, GS_BWD_GAUSS_ONLY, GS_BWD_PIXELS_ONLY, GS_GRAD_PARAMS, GS_GRAD_POSE, GsAdamCfg, GsCamera, GsError,
                   GsParams, GsPoseStep, GsProj, GsView, check, lib)

__all__ = ["Params", "Grads", "Proj", "Frame", "Rasterizer", "camera", "gs_project", "gs_bin_sort",
           "gs_render_fwd", "gs_render_fwd_l1", "gs_loss_scales", "gs_loss_from_tiles", "gs_tile_order", "gs_loss", "gs_tracking_loss", "gs_ssim", "gs_iso_reg", "gs_adam_step", "gs_prune", "gs_seed", "gs_gradient_mask", "seed_first_keyframe", "gs_unpack_rgbd", "Optimizer", "gs_render_bwd", "gs_pose_grad", "GS_GRAD_PARAMS", "GS_GRAD_POSE", "GS_BWD_PIXELS_ONLY", "GS_BWD_GAUSS_ONLY", "GS_BWD_ATOMIC_ACC",
           "GsError", "device_check"]


def _p(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise GsError("tensor is not on a CUDA device")
    if not t.is_contiguous():
        raise GsError("tensor must be contiguous")
    return C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def camera(cam) -> GsCamera:
    """gs_camera from an inputs.Camera (or any object with the same fields)."""
    return GsCamera(int(cam.width), int(cam.height), float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy),
                    float(cam.z_near), float(cam.z_far))


def device_check(device=0):
    sm = C.c_int(0)
    check(lib().gs_check_device(int(device), C.byref(sm)), "gs_check_device")
    return sm.value


@dataclass
class Params:
    mean_opa: torch.Tensor  # [N,4] (x, y, z, opacity logit)
    quat: torch.Tensor      # [N,4] (w, x, y, z)
    logscale: torch.Tensor  # [N,4]
    rgb: torch.Tensor       # [N,4]

    @property
    def n(self):
        return self.mean_opa.shape[0]

    def c(self):
        return GsParams(_p(self.mean_opa), _p(self.quat), _p(self.logscale), _p(self.rgb), self.n)

    @staticmethod
    def from_numpy(mean_opa, quat, logscale, rgb, device="cuda"):
        f = lambda a: torch.as_tensor(a, dtype=torch.float32).contiguous().to(device)
        return Params(f(mean_opa), f(quat), f(logscale), f(rgb))


@dataclass
class Grads:
    """Parameter gradients in the gs_params layout, views of ONE contiguous
    [4, N, 4] buffer so a single NCCL all-reduce covers them."""
    buf: torch.Tensor

    @staticmethod
    def zeros(n, device="cuda"):
        return Grads(torch.zeros(4, n, 4, dtype=torch.float32, device=device))

    @property
    def mean_opa(self):
        return self.buf[0]

    @property
    def quat(self):
        return self.buf[1]

    @property
    def logscale(self):
        return self.buf[2]

    @property
    def rgb(self):
        return self.buf[3]

    def zero_(self):
        self.buf.zero_()
        return self


class Proj:
    """gs_proj buffers for n Gaussians."""

    def __init__(self, n, device="cuda"):
        m = max(n, 1)
        self.n = n
        self.uv = torch.empty(m, 2, dtype=torch.float64, device=device)
        self.conic_o = torch.empty(m, 4, dtype=torch.float32, device=device)
        self.coef = torch.empty(m, 4, dtype=torch.float32, device=device)
        self.rgbz = torch.empty(m, 4, dtype=torch.float32, device=device)
        self.depth = torch.empty(m, dtype=torch.float32, device=device)
        self.rect = torch.empty(m, 4, dtype=torch.int16, device=device)
        self.tiles_touched = torch.empty(m, dtype=torch.int32, device=device)

    def c(self):
        return GsProj(_p(self.uv), _p(self.conic_o), _p(self.coef), _p(self.rgbz), _p(self.depth),
                      _p(self.rect), _p(self.tiles_touched))


class Frame:
    """Rendered frame buffers (planar)."""

    def __init__(self, H, W, device="cuda"):
        self.color = torch.empty(3, H, W, dtype=torch.float32, device=device)
        self.depth = torch.empty(H, W, dtype=torch.float32, device=device)
        self.alpha = torch.empty(H, W, dtype=torch.float32, device=device)
        self.T_final = torch.empty(H, W, dtype=torch.float32, device=device)
        self.n_contrib = torch.empty(H, W, dtype=torch.int32, device=device)
        self.stats = torch.empty(2, H, W, dtype=torch.int32, device=device)


# ---------------------------------------------------------------------------
# Entry points, same names as include/gs.h


def gs_project(params: Params, view, cam: GsCamera, proj: Proj, counters=None, stream=None):
    check(lib().gs_project(params.c(), _p(view), cam, proj.c(), _p(counters), _stream(stream)), "gs_project")


def gs_bin_sort(proj: Proj, n, cam: GsCamera, ws, capacity, sorted_idx, tile_range, n_pairs, counters=None,
                stream=None, tile_order=None):
    check(lib().gs_bin_sort(proj.c(), int(n), cam, _p(ws), ws.numel() * ws.element_size(), int(capacity),
                            _p(sorted_idx), _p(tile_range), _p(tile_order), _p(n_pairs), _p(counters),
                            _stream(stream)), "gs_bin_sort")


def gs_render_fwd(proj: Proj, sorted_idx, tile_range, cam: GsCamera, frame: Frame, stats=False, stream=None,
                  tile_order=None, tile_work=None):
    check(lib().gs_render_fwd(proj.c(), _p(sorted_idx), _p(tile_range), _p(tile_order), cam, _p(frame.color), _p(frame.depth),
                              _p(frame.alpha), _p(frame.T_final), _p(frame.n_contrib),
                              _p(frame.stats) if stats else None, _p(tile_work), _stream(stream)),
          "gs_render_fwd")


def gs_render_fwd_l1(proj: Proj, sorted_idx, tile_range, cam: GsCamera, frame: Frame, tgt_color, tgt_depth, scales,
                     dL_dcolor, dL_ddepth, stream=None, tile_order=None, tile_work=None, loss_part=None,
                     tile_done=None):
    check(lib().gs_render_fwd_l1(proj.c(), _p(sorted_idx), _p(tile_range), _p(tile_order), cam, _p(frame.color),
                                 _p(frame.depth), _p(frame.alpha), _p(frame.T_final), _p(frame.n_contrib),
                                 _p(tile_work), _p(tgt_color), _p(tgt_depth), _p(scales), _p(dL_dcolor),
                                 _p(dL_ddepth), _p(loss_part), _p(tile_done), _stream(stream)),
          "gs_render_fwd_l1")


def gs_loss_from_tiles(cam: GsCamera, loss_part, scales, lambda_color, lambda_depth, loss, stream=None):
    check(lib().gs_loss_from_tiles(cam, _p(loss_part), _p(scales), float(lambda_color), float(lambda_depth), _p(loss),
                                   _stream(stream)), "gs_loss_from_tiles")


def gs_loss_scales(cam: GsCamera, tgt_depth, lambda_color, lambda_depth, ws, scales, stream=None):
    check(lib().gs_loss_scales(cam, _p(tgt_depth), float(lambda_color), float(lambda_depth), _p(ws),
                               ws.numel() * ws.element_size(), _p(scales), _stream(stream)), "gs_loss_scales")


def gs_tile_order(work, T, order, stream=None):
    check(lib().gs_tile_order(_p(work), int(T), _p(order), _stream(stream)), "gs_tile_order")


def gs_loss(cam: GsCamera, color, depth, tgt_color, tgt_depth, weight, lambda_color, lambda_depth, ws, loss,
            dL_dcolor, dL_ddepth, stream=None):
    check(lib().gs_loss(cam, _p(color), _p(depth), _p(tgt_color), _p(tgt_depth), _p(weight), float(lambda_color),
                        float(lambda_depth), _p(ws), ws.numel() * ws.element_size(), _p(loss), _p(dL_dcolor),
                        _p(dL_ddepth), _stream(stream)), "gs_loss")


def gs_tracking_loss(cam: GsCamera, color, depth, alpha, tgt_color, tgt_depth, lambda_c, inlier_mult, ws, loss,
                     dL_dcolor, dL_ddepth, stream=None):
    check(lib().gs_tracking_loss(cam, _p(color), _p(depth), _p(alpha), _p(tgt_color), _p(tgt_depth), float(lambda_c),
                                 float(inlier_mult), _p(ws), ws.numel() * ws.element_size(), _p(loss),
                                 _p(dL_dcolor), _p(dL_ddepth), _stream(stream)), "gs_tracking_loss")


def gs_ssim(cam: GsCamera, color, tgt_color, weight, ws, loss, dL_dcolor, stream=None):
    check(lib().gs_ssim(cam, _p(color), _p(tgt_color), float(weight), _p(ws), ws.numel() * ws.element_size(),
                        _p(loss), _p(dL_dcolor), _stream(stream)), "gs_ssim")


def gs_iso_reg(params: Params, lambda_reg, g_logscale, ws, loss, stream=None):
    check(lib().gs_iso_reg(params.c(), float(lambda_reg), _p(g_logscale), _p(ws), ws.numel() * ws.element_size(),
                           _p(loss), _stream(stream)), "gs_iso_reg")


def gs_adam_step(params: Params, grads: "Grads", moments, cfg: GsAdamCfg, counters=None, stream=None):
    check(lib().gs_adam_step(params.c(), _p(grads.mean_opa), _p(grads.quat), _p(grads.logscale), _p(grads.rgb),
                             _p(moments), C.byref(cfg), _p(counters), _stream(stream)), "gs_adam_step")


def gs_prune(params: Params, moments, o_thre, out: Params, moments_out, ws, n_out, stream=None):
    check(lib().gs_prune(params.c(), _p(moments), float(o_thre), out.c(), _p(moments_out), _p(ws),
                         ws.numel() * ws.element_size(), _p(n_out), _stream(stream)), "gs_prune")


def gs_seed(cam: GsCamera, view, color, depth, alpha, alpha_n, rho, max_new, seed, params: Params, n, ws, n_new,
            stream=None):
    """NEXT(4): append the seeded Gaussians of one keyframe to params (arrays of
    capacity >= n + max_new) after the first n; n_new (device) = accepted count.
    view: the keyframe's T_wc as 12 host floats (R row-major, t)."""
    import numpy as np
    v = np.asarray(view.detach().cpu() if hasattr(view, "detach") else view, np.float32).ravel()
    gv = GsView((C.c_float * 9)(*v[:9]), (C.c_float * 3)(*v[9:12]))
    cap = params.mean_opa.shape[0]
    P = GsParams(_p(params.mean_opa), _p(params.quat), _p(params.logscale), _p(params.rgb), int(n))
    check(lib().gs_seed(cam, C.byref(gv), _p(color), _p(depth), _p(alpha), float(alpha_n), float(rho), int(max_new),
                        int(seed) & 0xFFFFFFFF, P, int(cap), _p(ws), ws.numel() * ws.element_size(), _p(n_new),
                        _stream(stream)), "gs_seed")


def gs_gradient_mask(cam: GsCamera, color, depth, q, pseudo_alpha, ws, threshold_m2=None, stream=None):
    """R43: pseudo_alpha (device [H, W]) = 0 on the high-colour-gradient
    valid-depth pixels of the keyframe, 1 elsewhere (gs_seed with alpha_n 0.5)."""
    check(lib().gs_gradient_mask(cam, _p(color), _p(depth), float(q), _p(pseudo_alpha), _p(threshold_m2), _p(ws),
                                 ws.numel() * ws.element_size(), _stream(stream)), "gs_gradient_mask")


def seed_first_keyframe(cam: GsCamera, view, color, depth, params: Params, n, M_u, M_c, seed, rho=0.01, q=0.95):
    """The first keyframe of a sub-map (R43): M_u uniform samples, then
    M_c samples of the high-colour-gradient set against the sub-map holding
    the first batch; params (capacity >= n + M_u + M_c) gets both batches
    after the first n.  Host-synchronising (the second batch starts after the
    first's count).  Returns (n_u, n_c)."""
    import numpy as np  # noqa: F401
    d = color.device
    H, W = depth.shape
    ws = torch.empty((max(lib().gs_seed_workspace_bytes(cam, n + M_u, max(M_u, M_c)),
                          lib().gs_gradient_mask_workspace_bytes(cam)) + 15) // 16 * 4, dtype=torch.float32, device=d)
    n_new = torch.zeros(1, dtype=torch.int32, device=d)
    gs_seed(cam, view, color, depth, torch.zeros(H, W, dtype=torch.float32, device=d), 0.6, rho, M_u, seed, params,
            n, ws, n_new)
    n_u = int(n_new.item())
    pseudo = torch.empty(H, W, dtype=torch.float32, device=d)
    gs_gradient_mask(cam, color, depth, q, pseudo, ws)
    gs_seed(cam, view, color, depth, pseudo, 0.5, rho, M_c, seed + 1, params, n + n_u, ws, n_new)
    return n_u, int(n_new.item())


def gs_unpack_rgbd(cam: GsCamera, rgb8, depth16, depth_scale, tgt_color, tgt_depth, stream=None, scales=None,
                   lambda_color=1.0, lambda_depth=1.0):
    """An 8-bit RGB [H][W][3] + 16-bit depth [H][W] frame (device tensors,
    uint8 / int16 or uint16 storage) into fp32 planar targets [3][H][W], [H][W];
    scales (device [4], optional): the frame's gs_loss_scales in the same pass."""
    check(lib().gs_unpack_rgbd(cam, _p(rgb8), _p(depth16), float(depth_scale), _p(tgt_color), _p(tgt_depth),
                               _p(scales), float(lambda_color), float(lambda_depth), _stream(stream)),
          "gs_unpack_rgbd")


class Optimizer:
    """Device-side mapping optimiser (NEXT(3)): Adam over the four float4
    parameter arrays with per-group learning rates (S:231 defaults), the
    Eq. 11 isotropic regulariser folded into the gradient before the step,
    and opacity pruning as a stable compaction of parameters and
    moments.  The moments are one [n][8][4] buffer."""

    DEFAULT_LR = dict(lr_mean=1e-4, lr_quat=1e-3, lr_logscale=1e-3, lr_opacity=5e-2, lr_rgb=2.5e-3)

    def __init__(self, n, device="cuda", betas=(0.9, 0.999), eps=1e-8, **lr):
        self.lr = dict(self.DEFAULT_LR, **lr)
        self.betas, self.eps = betas, eps
        self.t = 0
        self.moments = torch.zeros(max(n, 1), 8, 4, dtype=torch.float32, device=device)
        self.ws = torch.empty((lib().gs_opt_workspace_bytes(max(n, 1)) + 15) // 16 * 4, dtype=torch.float32,
                              device=device)
        self.reg_loss = torch.zeros(2, dtype=torch.float32, device=device)
        self.n_out = torch.zeros(1, dtype=torch.int32, device=device)

    def cfg(self):
        return GsAdamCfg(self.lr["lr_mean"], self.lr["lr_quat"], self.lr["lr_logscale"], self.lr["lr_opacity"],
                         self.lr["lr_rgb"], self.betas[0], self.betas[1], self.eps, self.t)

    def regularize(self, params: Params, grads: "Grads", lambda_reg=1.0):
        """Eq. 11 (x lambda_reg): self.reg_loss = (lambda_reg L_reg, L_reg) and the
        log-scale gradients += its gradient."""
        self.reg_loss.zero_()
        gs_iso_reg(params, lambda_reg, grads.logscale, self.ws, self.reg_loss)
        return self.reg_loss

    def step(self, params: Params, grads: "Grads", counters=None):
        self.t += 1
        gs_adam_step(params, grads, self.moments, self.cfg(), counters)

    def prune(self, params: Params, o_thre, out: Params, moments_out):
        """Kept Gaussians -> out (same capacity), moments -> moments_out;
        self.n_out (device) = kept count."""
        gs_prune(params, self.moments, o_thre, out, moments_out, self.ws, self.n_out)
        return self.n_out


def gs_render_bwd(params: Params, view, cam: GsCamera, proj: Proj, sorted_idx, tile_range, T_final, n_contrib,
                  dL_dcolor, dL_ddepth, dL_dalpha, flags, ws, grads: Grads = None, pose_partials=None,
                  stream=None, event_pair=None, tile_order=None, tile_done=None):
    """event_pair: optional (start, end) torch.cuda.Event recorded around the call."""
    g = grads
    if event_pair is not None:
        event_pair[0].record(torch.cuda.current_stream() if stream is None else stream)
    check(lib().gs_render_bwd(params.c(), _p(view), cam, proj.c(), _p(sorted_idx), _p(tile_range),
                              _p(tile_order), _p(T_final),
                              _p(n_contrib), _p(dL_dcolor), _p(dL_ddepth), _p(dL_dalpha), int(flags), _p(ws),
                              ws.numel() * ws.element_size(),
                              _p(g.mean_opa) if g is not None else None, _p(g.quat) if g is not None else None,
                              _p(g.logscale) if g is not None else None, _p(g.rgb) if g is not None else None,
                              _p(pose_partials), _p(tile_done), _stream(stream)), "gs_render_bwd")
    if event_pair is not None:
        event_pair[1].record(torch.cuda.current_stream() if stream is None else stream)


def gs_pose_grad(view, pose_partials, n_partials, step=None, adam_state=None, dL_dview=None, dL_dtwist=None,
                 dL_dqt=None, stream=None):
    st = None
    if step is not None:
        st = C.byref(GsPoseStep(*[float(x) for x in step]))
    check(lib().gs_pose_grad(_p(view), _p(pose_partials), int(n_partials), st, _p(adam_state), _p(dL_dview),
                             _p(dL_dtwist), _p(dL_dqt), _stream(stream)), "gs_pose_grad")


# ---------------------------------------------------------------------------


class _GradView:
    """Grads-like access to a [4, m, 4] slice of a gradient buffer (each
    component array contiguous, not the whole slice)."""

    def __init__(self, g):
        self.mean_opa, self.quat, self.logscale, self.rgb = (g.buf[k] for k in range(4))


class Rasterizer:
    """All buffers of one (N Gaussians, camera) problem; no allocation in the
    per-iteration calls, so a whole iteration can be CUDA-graph captured."""

    def __init__(self, n, cam, capacity=None, device="cuda"):
        self.n = n
        self.cam_py = cam
        self.cam = camera(cam)
        self.device = device
        L = lib()
        self.T = L.gs_num_tiles(self.cam)
        if self.T <= 0:
            raise GsError("invalid camera")
        H, W = cam.height, cam.width
        self.proj = Proj(n, device)
        self.sort_ws = torch.empty(4, dtype=torch.float32, device=device)  # sized by set_capacity
        self.tile_range = torch.empty(self.T, 2, dtype=torch.int32, device=device)
        self.tile_order = torch.empty(self.T, dtype=torch.int32, device=device)
        self.tile_work = torch.empty(self.T, dtype=torch.int32, device=device)
        # a valid launch order from the start (forward_l1(reuse_order=True) may launch with it)
        self.bwd_order = torch.arange(self.T, dtype=torch.int32, device=device)
        self.n_pairs = torch.zeros(1, dtype=torch.int64, device=device)
        self.counters = torch.zeros(4, dtype=torch.int64, device=device)
        self.frame = Frame(H, W, device)
        self.loss_ws = torch.empty((L.gs_loss_workspace_bytes(self.cam) + 15) // 16 * 4, dtype=torch.float32,
                                   device=device)
        self.loss = torch.zeros(4, dtype=torch.float32, device=device)  # total, L1 colour, depth, SSIM
        self.ssim_ws = None
        self.tl_ws = None  # gs_tracking_loss workspace, allocated on first use
        self.scales = None  # gs_loss_scales output (forward_l1)
        self.loss_part = None  # per-tile |residual| sums (render_l1)
        self.tile_done = None  # per-tile forward -> backward flags (overlap) + timeout count
        self.tl_loss = None
        self.dL_dcolor = torch.zeros(3, H, W, dtype=torch.float32, device=device)
        self.dL_ddepth = torch.zeros(H, W, dtype=torch.float32, device=device)
        # zeroed once; gs_render_bwd returns it zeroed (include/gs.h)
        self.bwd_ws = torch.zeros((L.gs_bwd_workspace_bytes(n) + 15) // 16 * 4, dtype=torch.float32, device=device)
        self.n_partials = L.gs_pose_partials_count(n)
        self.pose_partials = torch.zeros(self.n_partials, 12, dtype=torch.float32, device=device)
        self.capacity = 0
        self.sorted_idx = torch.empty(1, dtype=torch.int32, device=device)
        self.set_capacity(1 if capacity is None else capacity)

    @property
    def grad2d(self):
        """The [N, 12] 2-D gradient scratch, (u, v, A, B), (C, p_z, logit, 0),
        (r, g, b, 0): holds the 2-D gradients only between a
        GS_BWD_PIXELS_ONLY and a GS_BWD_GAUSS_ONLY call."""
        return self.bwd_ws[: self.n * 12].view(self.n, 12)

    def set_capacity(self, capacity):
        """Pair capacity of the binning (sorted_idx and the sort workspace)."""
        capacity = int(max(capacity, 1))
        if capacity > self.capacity:
            ws = lib().gs_binsort_workspace_bytes(self.n, capacity, self.cam)
            if ws == 0:
                raise GsError("gs_binsort_workspace_bytes: problem not supported")
            self.sort_ws = torch.empty((ws + 15) // 16 * 4, dtype=torch.float32, device=self.device)
            self.sorted_idx = torch.empty(capacity, dtype=torch.int32, device=self.device)
            self.capacity = capacity

    def size_for(self, params: Params, view, slack=1.25):
        """Host-synchronising helper (setup only): project + sort once and size
        the pair capacity to slack x the pair count."""
        self.project(params, view)
        self.bin_sort()
        P = int(self.n_pairs.item())
        if P > self.capacity:
            self.set_capacity(int(P * slack) + 1024)
            self.bin_sort()
        return P

    # -- stages ---------------------------------------------------------------
    def project(self, params: Params, view):
        gs_project(params, view, self.cam, self.proj, self.counters)

    def bin_sort(self, order=True):
        """S2; order=False: no heaviest-first launch order (a caller that
        launches the forward in a reused work order; the binning then takes
        its multi-CTA counts step)."""
        gs_bin_sort(self.proj, self.n, self.cam, self.sort_ws, self.capacity, self.sorted_idx, self.tile_range,
                    self.n_pairs, self.counters, tile_order=self.tile_order if order else None)

    def render(self, stats=False):
        gs_render_fwd(self.proj, self.sorted_idx, self.tile_range, self.cam, self.frame, stats,
                      tile_order=self.tile_order, tile_work=self.tile_work)
        gs_tile_order(self.tile_work, self.T, self.bwd_order)  # the backward's heaviest-first order

    def forward(self, params: Params, view, stats=False):
        self.project(params, view)
        self.bin_sort()
        self.render(stats)
        return self.frame

    def loss_scales(self, tgt_depth, lambda_color=1.0, lambda_depth=1.0, out=None):
        """gs_loss_scales of a target frame into out (default self.scales, for
        forward_l1 / render_l1)."""
        if out is None:
            if self.scales is None:
                self.scales = torch.zeros(4, dtype=torch.float32, device=self.device)
            out = self.scales
        gs_loss_scales(self.cam, tgt_depth, lambda_color, lambda_depth, self.loss_ws, out)
        return out

    def render_l1(self, tgt_color, tgt_depth, lambda_color, lambda_depth, scales, order=None):
        """S3 + S4 fused (after project + bin_sort): gs_render_fwd_l1 writes the
        frame and gs_loss's gradient maps and per-tile |residual| sums, then
        gs_loss_from_tiles -> self.loss[:3]; scales from loss_scales (same
        lambdas).  order: the forward's tile launch order (default: gs_bin_sort's
        list-length order); scheduling only."""
        if self.loss_part is None:
            self.loss_part = torch.empty(2 * self.T, dtype=torch.float64, device=self.device)
        gs_render_fwd_l1(self.proj, self.sorted_idx, self.tile_range, self.cam, self.frame, tgt_color, tgt_depth,
                         scales, self.dL_dcolor, self.dL_ddepth, tile_order=self.tile_order if order is None else order,
                         tile_work=self.tile_work, loss_part=self.loss_part)
        gs_tile_order(self.tile_work, self.T, self.bwd_order)
        gs_loss_from_tiles(self.cam, self.loss_part, scales, lambda_color, lambda_depth, self.loss)
        return self.loss

    def render_l1_overlapped(self, tgt_color, tgt_depth, scales):
        """render_l1's forward for an overlapped backward: launched in (and the
        backward reading) the previous call's work order self.bwd_order, with
        the per-tile completion flags; the NEXT launch on this stream must be
        backward(..., overlap=True), then finish_l1."""
        if self.loss_part is None:
            self.loss_part = torch.empty(2 * self.T, dtype=torch.float64, device=self.device)
        gs_render_fwd_l1(self.proj, self.sorted_idx, self.tile_range, self.cam, self.frame, tgt_color, tgt_depth,
                         scales, self.dL_dcolor, self.dL_ddepth, tile_order=self.bwd_order,
                         tile_work=self.tile_work, loss_part=self.loss_part, tile_done=self._tile_done())

    def finish_l1(self, lambda_color, lambda_depth, scales):
        """After render_l1_overlapped + backward: the next work order and the
        loss value (self.loss[:3])."""
        gs_tile_order(self.tile_work, self.T, self.bwd_order)
        gs_loss_from_tiles(self.cam, self.loss_part, scales, lambda_color, lambda_depth, self.loss)
        return self.loss

    def _tile_done(self):
        if self.tile_done is None:  # [T] flags + [1] count of timed-out waits (include/gs.h)
            self.tile_done = torch.zeros(self.T + 1, dtype=torch.int32, device=self.device)
        return self.tile_done

    def flag_timeouts(self):
        """Host sync: capped tile_done waits of the overlapped backward that
        timed out (0 unless the forward -> backward ordering was broken)."""
        return 0 if self.tile_done is None else int(self.tile_done[self.T].item())

    def forward_l1(self, params: Params, view, tgt_color, tgt_depth, reuse_order=False, refresh_order=True,
                   overlap=False):
        """S1-S3 with the L1 gradient maps fused into the forward
        (gs_render_fwd_l1, scales from loss_scales): self.dL_dcolor /
        self.dL_ddepth hold gs_loss's maps; no loss value.  reuse_order: the
        forward is launched in the previous call's work order (tracking: the
        pose moves little between iterations) and gs_bin_sort skips its own
        launch order; refresh_order=False keeps the previous work order for
        the backward too; launch orders never change results.  overlap: the
        next backward(overlap=True) starts while this forward finishes, tile
        by tile (per-tile flags + programmatic dependent launch)."""
        self.project(params, view)
        if reuse_order:  # no launch order for the sort: the forward reuses the previous work order
            gs_bin_sort(self.proj, self.n, self.cam, self.sort_ws, self.capacity, self.sorted_idx, self.tile_range,
                        self.n_pairs, self.counters, tile_order=None)
        else:
            self.bin_sort()
        gs_render_fwd_l1(self.proj, self.sorted_idx, self.tile_range, self.cam, self.frame, tgt_color, tgt_depth,
                         self.scales, self.dL_dcolor, self.dL_ddepth,
                         tile_order=self.bwd_order if reuse_order else self.tile_order, tile_work=self.tile_work,
                         tile_done=self._tile_done() if overlap else None)
        if refresh_order or not reuse_order:
            gs_tile_order(self.tile_work, self.T, self.bwd_order)
        return self.frame

    def compute_loss(self, tgt_color, tgt_depth, weight=None, lambda_color=1.0, lambda_depth=1.0, ssim=0.0):
        """Eq. 12 with the L1 colour term (ssim = 0, BJ.configs) or Eq. 10's
        (1 - ssim) L1 + ssim (1 - SSIM) colour loss (ssim = 0.2 in the paper).
        self.loss = (total, L1 colour, L1 depth, SSIM)."""
        gs_loss(self.cam, self.frame.color, self.frame.depth, tgt_color, tgt_depth, weight,
                lambda_color * (1.0 - ssim), lambda_depth, self.loss_ws, self.loss, self.dL_dcolor, self.dL_ddepth)
        if ssim > 0.0:
            if self.ssim_ws is None:
                self.ssim_ws = torch.empty((lib().gs_ssim_workspace_bytes(self.cam) + 15) // 16 * 4,
                                           dtype=torch.float32, device=self.device)
            gs_ssim(self.cam, self.frame.color, tgt_color, lambda_color * ssim, self.ssim_ws, self.loss,
                    self.dL_dcolor)
        return self.loss

    def compute_tracking_loss(self, tgt_color, tgt_depth, lambda_c=0.5, inlier_mult=50.0):
        """Eq. 15 masked tracking loss into self.tl_loss = (L, med_c, med_d,
        inliers) and the gradient maps used by backward()."""
        if self.tl_ws is None:
            L = lib()
            self.tl_ws = torch.empty((L.gs_tracking_loss_workspace_bytes(self.cam) + 15) // 16 * 4,
                                     dtype=torch.float32, device=self.device)
            self.tl_loss = torch.zeros(4, dtype=torch.float32, device=self.device)
        gs_tracking_loss(self.cam, self.frame.color, self.frame.depth, self.frame.alpha, tgt_color, tgt_depth,
                         lambda_c, inlier_mult, self.tl_ws, self.tl_loss, self.dL_dcolor, self.dL_ddepth)
        return self.tl_loss

    def backward(self, params: Params, view, flags=GS_GRAD_PARAMS, grads: Grads = None, dL_dcolor=None,
                 dL_ddepth=None, dL_dalpha=None, event_pair=None, overlap=False):
        """overlap: right after forward_l1(overlap=True) (see there)."""
        gs_render_bwd(params, view, self.cam, self.proj, self.sorted_idx, self.tile_range, self.frame.T_final,
                      self.frame.n_contrib, self.dL_dcolor if dL_dcolor is None else dL_dcolor,
                      self.dL_ddepth if dL_ddepth is None else dL_ddepth, dL_dalpha, flags, self.bwd_ws, grads,
                      self.pose_partials if flags & GS_GRAD_POSE else None, event_pair=event_pair,
                      tile_order=self.bwd_order, tile_done=self._tile_done() if overlap else None)

    def backward_gauss_range(self, params: Params, view, grads: Grads, i0, i1, flags=GS_GRAD_PARAMS):
        """S6 (GS_BWD_GAUSS_ONLY) for the Gaussians [i0, i1) only: the same C-ABI
        call on sub-array views (parameters, projection, grad2d scratch and
        gradients offset by i0), so a caller can start reducing the finished
        part of the gradient buffer while the rest is chained."""
        sl = lambda t: t[i0:i1]
        P = Params(sl(params.mean_opa), sl(params.quat), sl(params.logscale), sl(params.rgb))
        pr = Proj.__new__(Proj)
        pr.n = i1 - i0
        for name in ("uv", "conic_o", "coef", "rgbz", "depth", "rect", "tiles_touched"):
            setattr(pr, name, sl(getattr(self.proj, name)))
        g = Grads(grads.buf[:, i0:i1])
        gs_render_bwd(P, view, self.cam, pr, self.sorted_idx, self.tile_range, self.frame.T_final,
                      self.frame.n_contrib, self.dL_dcolor, self.dL_ddepth, None, flags | GS_BWD_GAUSS_ONLY,
                      self.bwd_ws[i0 * 12:i1 * 12], _GradView(g), None)

    def pose_grad(self, view, step=None, adam_state=None, dL_dview=None, dL_dtwist=None, dL_dqt=None):
        gs_pose_grad(view, self.pose_partials, self.n_partials, step, adam_state, dL_dview, dL_dtwist, dL_dqt)
