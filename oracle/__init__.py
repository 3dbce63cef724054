"""fp64 CPU oracle of the Gaussian-SLAM rasterizer — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  It wraps ``gs_oracle.c``
(plain fp64 C, built by ``__graft_entry__.build()`` into ``liboracle.so``) with
numpy marshalling, and shares nothing with the CUDA path.

Every function cites the passage it follows (P:n = PAPER.md line n, S:n =
SPEC.md line n, R# = DESIGN.md §3 readings).  Pins: tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gs_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_dp = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_fp = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")


def build(force=False):
    """Compile the oracle: gcc -O2 -fopenmp -ffp-contract=off (R1)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        L.or_num_tiles.restype = C.c_int
        L.or_count_pairs.restype = C.c_int64
        L.or_num_threads.restype = C.c_int
        _lib = L
    return _lib


def _ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(C.c_void_p)


def _cam(cam):
    """(W, H, fx, fy, cx, cy, z_near, z_far): the camera is an fp32 gs_camera in
    the C-ABI, so the float fields are promoted from their fp32 values."""
    c = list(cam.as_tuple() if hasattr(cam, "as_tuple") else cam)
    c = c[:2] + [float(np.float32(x)) for x in c[2:]]
    return np.ascontiguousarray(np.array(c, np.float64))


def _view(view):
    v = np.asarray(view, np.float64).reshape(12)
    return np.ascontiguousarray(v[:9]), np.ascontiguousarray(v[9:])


def num_threads():
    return lib().or_num_threads()


def params64(mean_opa, quat, logscale, rgb):
    """Exact fp32 -> fp64 promotion of the gs_params float4 records."""
    mo = np.asarray(mean_opa, np.float64)
    return dict(mean=np.ascontiguousarray(mo[:, :3]), quat=np.ascontiguousarray(np.asarray(quat, np.float64)),
                logscale=np.ascontiguousarray(np.asarray(logscale, np.float64)[:, :3]),
                logit=np.ascontiguousarray(mo[:, 3]),
                rgb=np.ascontiguousarray(np.asarray(rgb, np.float64)[:, :3]))


def quat_to_rot(q):
    """R(q) of a unit quaternion (w, x, y, z)."""
    out = np.zeros(9)
    lib().or_quat_to_rot(_ptr(np.ascontiguousarray(q, np.float64)), _ptr(out))
    return out.reshape(3, 3)


def covariance(q, logscale):
    """Sigma = R S S^T R^T."""
    out = np.zeros(9)
    lib().or_covariance(_ptr(np.ascontiguousarray(q, np.float64)),
                        _ptr(np.ascontiguousarray(logscale, np.float64)), _ptr(out))
    return out.reshape(3, 3)


def project(p64, view, cam):
    """S1, Eqs. 1-2. Returns a dict of per-Gaussian arrays."""
    n = p64["mean"].shape[0]
    R, t = _view(view)
    out = dict(uv=np.zeros((n, 2)), conic=np.zeros((n, 3)), opac=np.zeros(n), pz=np.zeros(n),
               depth_key=np.zeros(n, np.float32), hxy=np.zeros((n, 2)),
               rect=np.zeros((n, 4), np.int32), culled=np.zeros(n, np.int32),
               cov2d=np.zeros((n, 3)))
    lib().or_project(C.c_int(n), _ptr(p64["mean"]), _ptr(p64["quat"]), _ptr(p64["logscale"]),
                     _ptr(p64["logit"]), _ptr(R), _ptr(t), _ptr(_cam(cam)),
                     _ptr(out["uv"]), _ptr(out["conic"]), _ptr(out["opac"]), _ptr(out["pz"]),
                     _ptr(out["depth_key"]), _ptr(out["hxy"]), _ptr(out["rect"]),
                     _ptr(out["culled"]), _ptr(out["cov2d"]))
    return out


def bin_sort(rect, culled, depth_key, cam):
    """S2 (R10): (sorted_idx[P], tile_range[T,2])."""
    rect = np.ascontiguousarray(rect, np.int32)
    culled = np.ascontiguousarray(culled, np.int32)
    depth_key = np.ascontiguousarray(depth_key, np.float32)
    n = rect.shape[0]
    P = lib().or_count_pairs(C.c_int(n), _ptr(rect), _ptr(culled))
    T = lib().or_num_tiles(_ptr(_cam(cam)))
    idx = np.zeros(max(P, 1), np.int32)
    rng = np.zeros((T, 2), np.int32)
    lib().or_bin(C.c_int(n), _ptr(_cam(cam)), _ptr(rect), _ptr(culled), _ptr(depth_key),
                 _ptr(idx), _ptr(rng))
    return idx[:P], rng


def render(proj, rgb, sorted_idx, tile_range, cam, tile_mask=None):
    """S3, Eqs. 3, 4, 6: per-pixel front-to-back loop."""
    c = cam
    H, W = c.height, c.width
    n = proj["uv"].shape[0]
    o = dict(color=np.zeros((3, H, W)), depth=np.zeros((H, W)), alpha=np.zeros((H, W)),
             T_final=np.zeros((H, W)), n_contrib=np.zeros((H, W), np.int32),
             scanned=np.zeros((H, W), np.int32), contrib=np.zeros((H, W), np.int32),
             margin=np.full((H, W), np.inf), sig=np.zeros((H, W), np.uint64))
    tm = None if tile_mask is None else np.ascontiguousarray(tile_mask, np.uint8)
    lib().or_render(C.c_int(n), _ptr(_cam(cam)), _ptr(np.ascontiguousarray(proj["uv"])),
                    _ptr(np.ascontiguousarray(proj["conic"])), _ptr(np.ascontiguousarray(proj["opac"])),
                    _ptr(np.ascontiguousarray(proj["pz"])), _ptr(np.ascontiguousarray(rgb, np.float64)),
                    _ptr(np.ascontiguousarray(sorted_idx, np.int32)),
                    _ptr(np.ascontiguousarray(tile_range, np.int32)), _ptr(tm),
                    _ptr(o["color"]), _ptr(o["depth"]), _ptr(o["alpha"]), _ptr(o["T_final"]),
                    _ptr(o["n_contrib"]), _ptr(o["scanned"]), _ptr(o["contrib"]),
                    _ptr(o["margin"]), _ptr(o["sig"]))
    return o


def forward(p64, view, cam, tile_mask=None):
    """project -> bin_sort -> render, fp64 end to end."""
    pr = project(p64, view, cam)
    idx, rng = bin_sort(pr["rect"], pr["culled"], pr["depth_key"], cam)
    fr = render(pr, p64["rgb"], idx, rng, cam, tile_mask)
    fr.update(proj=pr, sorted_idx=idx, tile_range=rng)
    return fr


def loss(cam, color, depth, tgt_color, tgt_depth, weight=None, lambda_color=1.0,
         lambda_depth=1.0):
    """S4: L1 colour + L1 depth (Eqs. 9, 10 L1 part, 12; R20, R21)."""
    H, W = cam.height, cam.width
    out = np.zeros(3)
    gc = np.zeros((3, H, W))
    gd = np.zeros((H, W))
    f = lambda a: np.ascontiguousarray(a, np.float64)
    lib().or_loss(_ptr(_cam(cam)), _ptr(f(color)), _ptr(f(depth)), _ptr(f(tgt_color)),
                  _ptr(f(tgt_depth)), _ptr(None if weight is None else f(weight)),
                  C.c_double(lambda_color), C.c_double(lambda_depth), _ptr(out), _ptr(gc), _ptr(gd))
    return out, gc, gd


def backward(p64, view, cam, sorted_idx, tile_range, gC, gD, gA=None, tile_mask=None):
    """S5+S6 (Eqs. 7-8): analytic gradients and magnitude scales.

    Returns g2/m2 [n,10] (u, v, A, B, C, logit, r, g, b, p_z), g3/m3 [n,16] in
    the gs_params float4 layout, pose/mpose [12] = (dL/dR 9, dL/dt 3)."""
    n = p64["mean"].shape[0]
    R, t = _view(view)
    P = int(len(sorted_idx))
    o = dict(g2=np.zeros((n, 10)), m2=np.zeros((n, 10)), g3=np.zeros((n, 16)),
             m3=np.zeros((n, 16)), pose=np.zeros(12), mpose=np.zeros(12))
    f = lambda a: np.ascontiguousarray(a, np.float64)
    tm = None if tile_mask is None else np.ascontiguousarray(tile_mask, np.uint8)
    idx = np.ascontiguousarray(sorted_idx, np.int32)
    if P == 0:
        idx = np.zeros(1, np.int32)
    lib().or_backward(C.c_int(n), _ptr(p64["mean"]), _ptr(p64["quat"]), _ptr(p64["logscale"]),
                      _ptr(p64["logit"]), _ptr(p64["rgb"]), _ptr(R), _ptr(t), _ptr(_cam(cam)),
                      _ptr(idx), _ptr(np.ascontiguousarray(tile_range, np.int32)),
                      C.c_int64(P), _ptr(tm), _ptr(f(gC)), _ptr(f(gD)),
                      _ptr(None if gA is None else f(gA)), _ptr(o["g2"]), _ptr(o["m2"]),
                      _ptr(o["g3"]), _ptr(o["m3"]), _ptr(o["pose"]), _ptr(o["mpose"]))
    return o


def pose_twist(pose12, view):
    """dL/d(v, w) of the left perturbation T <- exp(xi^) T (R22)."""
    R, t = _view(view)
    out = np.zeros(6)
    p = np.ascontiguousarray(pose12, np.float64)
    lib().or_pose_twist(_ptr(np.ascontiguousarray(p[:9])), _ptr(np.ascontiguousarray(p[9:])),
                        _ptr(R), _ptr(t), _ptr(out))
    return out


def pose_qt(pose12, q):
    """dL/dq of T_wc's unit quaternion q (w, x, y, z) (R22); dL/dt is pose12[9:]."""
    out = np.zeros(4)
    p = np.ascontiguousarray(pose12, np.float64)
    lib().or_pose_qt(_ptr(np.ascontiguousarray(p[:9])), _ptr(np.ascontiguousarray(q, np.float64)),
                     _ptr(out))
    return out


def se3_exp(xi):
    R = np.zeros(9)
    t = np.zeros(3)
    lib().or_se3_exp(_ptr(np.ascontiguousarray(xi, np.float64)), _ptr(R), _ptr(t))
    return R.reshape(3, 3), t


def pose_adam(view, twist_grad, state, lr=(2e-3, 1e-3), hyp=(0.9, 0.999, 1e-8)):
    """One Adam step on the twist; returns the new view (12) and state (13)."""
    R, t = _view(view)
    R = R.copy()
    t = t.copy()
    st = np.ascontiguousarray(state, np.float64).copy()
    lib().or_pose_adam(_ptr(R), _ptr(t), _ptr(np.ascontiguousarray(twist_grad, np.float64)),
                       _ptr(st), _ptr(np.array(lr, np.float64)), _ptr(np.array(hyp, np.float64)))
    return np.concatenate([R, t]), st
