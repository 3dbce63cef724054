"""Build libgs.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2312_10070_b200._build      # or __graft_entry__.build()

project.cu is compiled with --fmad=false: its fp64 decision path must keep the
documented rounding order (DESIGN.md §3 R1).  Everything else is compiled with
contraction on; the alpha evaluation uses explicit _rn intrinsics so that
forward and backward agree bit for bit (H5).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
# GS_DEBUG=1: the debug build (device-side bounds checks, gs_internal.cuh
# GS_ASSERT) into libgs_debug.so / build_debug/, loaded by _lib when GS_LIB_DEBUG=1
DEBUG = os.environ.get("GS_DEBUG", "0") == "1"
BUILD = os.path.join(PKG, "build_debug" if DEBUG else "build")
LIB = os.path.join(PKG, "libgs_debug.so" if DEBUG else "libgs.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC,
              "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
PER_FILE = {"project.cu": ["--fmad=false"]}
SOURCES = ["abi.cpp", "project.cu", "binsort.cu", "render_fwd.cu", "loss.cu", "tracking_loss.cu", "ssim.cu", "optim.cu", "seed.cu", "rgbd.cu", "render_bwd.cu",
           "pose.cu"]
HEADERS = ["gs_internal.cuh", "raster_common.cuh"]


def nvcc():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose=False, force=False):
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "gs.h"), __file__]
    objs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src + ".o")
        objs.append(obj)
        if force or _stale(obj, [path] + hdrs):
            cmd = ([nvcc()] + ARCH + NVCC_FLAGS + PER_FILE.get(src, []) + (["-DGS_DEBUG"] if DEBUG else []) +
                   os.environ.get("GS_EXTRA_NVCC", "").split())
            if src.endswith(".cpp"):
                cmd += ["-x", "cu"]
            cmd += ["-c", path, "-o", obj]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.check_call(cmd)
    if force or _stale(LIB, objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
