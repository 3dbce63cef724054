"""B200-native differentiable Gaussian-splatting rasterizer — the hot path of
Gaussian-SLAM (arXiv 2312.10070).

The product is the C-ABI library ``libgs.so`` (include/gs.h, CUDA sources in
``csrc/``); ``raster`` is its thin torch binding with the same entry-point
names.  The CUDA extension is required: there is no CPU fallback.
"""
from .raster import (GS_GRAD_PARAMS, GS_GRAD_POSE, Frame, Grads, GsError, Params, Proj, Rasterizer, camera,
                     device_check, gs_bin_sort, gs_loss, gs_pose_grad, gs_project, gs_render_bwd, gs_render_fwd)

__all__ = ["GS_GRAD_PARAMS", "GS_GRAD_POSE", "Frame", "Grads", "GsError", "Params", "Proj", "Rasterizer", "camera",
           "device_check", "gs_bin_sort", "gs_loss", "gs_pose_grad", "gs_project", "gs_render_bwd", "gs_render_fwd"]
