"""ctypes declarations of include/gs.h (argument marshalling only).

The library is loaded from this package directory (built in-tree by
``__graft_entry__.build()``).  There is no fallback: if ``libgs.so`` is
missing, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
# GS_LIB_DEBUG=1: the debug build with device-side bounds checks (tests only)
LIB_PATH = os.path.join(PKG, "libgs_debug.so" if os.environ.get("GS_LIB_DEBUG", "0") == "1" else "libgs.so")
HEADER = os.path.join(os.path.dirname(PKG), "include", "gs.h")

GS_OK = 0
GS_ERR_INVALID_ARG = -1
GS_ERR_WORKSPACE = -2
GS_ERR_CUDA = -3
GS_ERR_UNSUPPORTED = -4
GS_GRAD_PARAMS = 1
GS_GRAD_POSE = 2
GS_BWD_PIXELS_ONLY = 4
GS_BWD_GAUSS_ONLY = 8
GS_BWD_ATOMIC_ACC = 16


class GsCamera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("z_near", C.c_float), ("z_far", C.c_float)]


class GsParams(C.Structure):
    _fields_ = [("mean_opa", C.c_void_p), ("quat", C.c_void_p), ("logscale", C.c_void_p),
                ("rgb", C.c_void_p), ("n", C.c_int32)]


class GsProj(C.Structure):
    _fields_ = [("uv", C.c_void_p), ("conic_o", C.c_void_p), ("coef", C.c_void_p), ("rgbz", C.c_void_p),
                ("depth", C.c_void_p), ("rect", C.c_void_p), ("tiles_touched", C.c_void_p)]


class GsPoseStep(C.Structure):
    _fields_ = [("lr_trans", C.c_float), ("lr_rot", C.c_float), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double)]


class GsView(C.Structure):
    _fields_ = [("R", C.c_float * 9), ("t", C.c_float * 3)]


class GsAdamCfg(C.Structure):
    _fields_ = [("lr_mean", C.c_float), ("lr_quat", C.c_float), ("lr_logscale", C.c_float),
                ("lr_opacity", C.c_float), ("lr_rgb", C.c_float), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("step", C.c_int32)]


class GsError(RuntimeError):
    pass


_VP, _I32, _I64, _U32, _SZ, _F = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_size_t, C.c_float

_PROTOS = {
    "gs_version": (C.c_int, []),
    "gs_last_error": (C.c_char_p, []),
    "gs_check_device": (C.c_int, [C.c_int, C.POINTER(C.c_int)]),
    "gs_num_tiles": (_I32, [GsCamera]),
    "gs_binsort_workspace_bytes": (_SZ, [_I32, _I64, GsCamera]),
    "gs_loss_workspace_bytes": (_SZ, [GsCamera]),
    "gs_bwd_workspace_bytes": (_SZ, [_I32]),
    "gs_pose_partials_count": (_I32, [_I32]),
    "gs_project": (C.c_int, [GsParams, _VP, GsCamera, GsProj, _VP, _VP]),
    "gs_bin_sort": (C.c_int, [GsProj, _I32, GsCamera, _VP, _SZ, _I64, _VP, _VP, _VP, _VP, _VP, _VP]),
    "gs_render_fwd": (C.c_int, [GsProj, _VP, _VP, _VP, GsCamera, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "gs_tile_order": (C.c_int, [_VP, _I32, _VP, _VP]),
    "gs_loss": (C.c_int, [GsCamera, _VP, _VP, _VP, _VP, _VP, _F, _F, _VP, _SZ, _VP, _VP, _VP, _VP]),
    "gs_loss_scales": (C.c_int, [GsCamera, _VP, _F, _F, _VP, _SZ, _VP, _VP]),
    "gs_render_fwd_l1": (C.c_int, [GsProj, _VP, _VP, _VP, GsCamera, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP,
                                   _VP, _VP, _VP, _VP]),
    "gs_loss_from_tiles": (C.c_int, [GsCamera, _VP, _VP, _F, _F, _VP, _VP]),
    "gs_tracking_loss_workspace_bytes": (_SZ, [GsCamera]),
    "gs_ssim_workspace_bytes": (_SZ, [GsCamera]),
    "gs_opt_workspace_bytes": (_SZ, [_I32]),
    "gs_seed_workspace_bytes": (_SZ, [GsCamera, _I32, _I32]),
    "gs_seed": (C.c_int, [GsCamera, _VP, _VP, _VP, _VP, _F, _F, _I32, _U32, GsParams, _I32, _VP, _SZ, _VP, _VP]),
    "gs_unpack_rgbd": (C.c_int, [GsCamera, _VP, _VP, _F, _VP, _VP, _VP, _F, _F, _VP]),
    "gs_gradient_mask_workspace_bytes": (_SZ, [GsCamera]),
    "gs_gradient_mask": (C.c_int, [GsCamera, _VP, _VP, C.c_double, _VP, _VP, _VP, _SZ, _VP]),
    "gs_iso_reg": (C.c_int, [GsParams, _F, _VP, _VP, _SZ, _VP, _VP]),
    "gs_adam_step": (C.c_int, [GsParams, _VP, _VP, _VP, _VP, _VP, C.POINTER(GsAdamCfg), _VP, _VP]),
    "gs_prune": (C.c_int, [GsParams, _VP, _F, GsParams, _VP, _VP, _SZ, _VP, _VP]),
    "gs_ssim": (C.c_int, [GsCamera, _VP, _VP, _F, _VP, _SZ, _VP, _VP, _VP]),
    "gs_tracking_loss": (C.c_int, [GsCamera, _VP, _VP, _VP, _VP, _VP, _F, _F, _VP, _SZ, _VP, _VP, _VP, _VP]),
    "gs_render_bwd": (C.c_int, [GsParams, _VP, GsCamera, GsProj, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _U32, _VP,
                                _SZ, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "gs_pose_grad": (C.c_int, [_VP, _VP, _I32, C.POINTER(GsPoseStep), _VP, _VP, _VP, _VP, _VP]),
}

_lib = None


def lib():
    """Load libgs.so (raises if the CUDA extension was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise GsError(f"CUDA extension missing: {LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _PROTOS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def header_symbols():
    """Function names declared in include/gs.h."""
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(gs_[a-z_0-9]+)\s*\(", src, flags=re.M)))


def check(rc, what):
    if rc != GS_OK:
        raise GsError(f"{what} failed ({rc}): {lib().gs_last_error().decode()}")
