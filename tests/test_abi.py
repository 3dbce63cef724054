"""C-ABI host-side checks that run without a GPU: the library loads, exports
every symbol include/gs.h declares, answers size queries, and rejects invalid
arguments before touching the device."""
import ctypes as C
import re

import pytest

from paper_2312_10070_b200 import _lib, inputs
from paper_2312_10070_b200.raster import camera


def test_library_exports_every_header_symbol():
    names = _lib.header_symbols()
    assert len(names) >= 14
    L = _lib.lib()
    for n in names:
        assert hasattr(L, n), n
    for n in ["gs_project", "gs_bin_sort", "gs_render_fwd", "gs_loss", "gs_render_bwd", "gs_pose_grad"]:
        assert n in names  # the six north-star calls


def test_header_constants_match_oracle():
    """The oracle carries its own copies of the rasterizer constants; they must agree."""
    hdr = open(_lib.HEADER).read()
    src = open(__import__("oracle").__file__.replace("__init__.py", "gs_oracle.c")).read()
    assert re.search(r"#define GS_TILE 16\b", hdr) and re.search(r"#define OR_TILE 16\b", src)
    for h, o in [("GS_DILATION 0.3f", "OR_DILATION = (double)0.3f"), ("GS_ALPHA_MAX 0.999f", "OR_ALPHA_MAX = (double)0.999f"),
                 ("GS_ALPHA_MIN (1.0f / 255.0f)", "OR_ALPHA_MIN = (double)(1.0f / 255.0f)"),
                 ("GS_T_EPS 1e-4f", "OR_T_EPS = (double)1e-4f")]:
        assert h in hdr and o in src, (h, o)


def test_header_and_binding_constants_agree():
    hdr = open(_lib.HEADER).read()
    for name in ("GS_GRAD_PARAMS", "GS_GRAD_POSE", "GS_BWD_PIXELS_ONLY", "GS_BWD_GAUSS_ONLY", "GS_BWD_ATOMIC_ACC"):
        m = re.search(r"#define %s (\d+)u?" % name, hdr)
        assert m and int(m.group(1)) == getattr(_lib, name), name


def test_version_and_queries():
    L = _lib.lib()
    assert L.gs_version() == 2
    cam = camera(inputs.Camera(1200, 680, 600.0, 600.0, 599.5, 339.5))
    assert L.gs_num_tiles(cam) == 75 * 43
    assert L.gs_binsort_workspace_bytes(500_000, 6_000_000, cam) >= 12 * 6_000_000  # chunked-sort scratch
    assert L.gs_bwd_workspace_bytes(1000) == 1000 * 12 * 4
    assert L.gs_pose_partials_count(1000) == 8
    assert L.gs_loss_workspace_bytes(cam) > 0
    bad = camera(inputs.Camera(0, 10, 1.0, 1.0, 0.0, 0.0))
    assert L.gs_num_tiles(bad) == 0 and L.gs_binsort_workspace_bytes(10, 10, bad) == 0


def test_invalid_arguments_rejected_on_host():
    L = _lib.lib()
    cam = camera(inputs.Camera(64, 48, 60.0, 60.0, 32.0, 24.0))
    p = _lib.GsParams(None, None, None, None, -1)
    pr = _lib.GsProj()
    assert L.gs_project(p, None, cam, pr, None, None) == _lib.GS_ERR_INVALID_ARG
    assert b"invalid" in L.gs_last_error()
    p = _lib.GsParams(None, None, None, None, 10)
    assert L.gs_project(p, C.c_void_p(16), cam, pr, None, None) == _lib.GS_ERR_INVALID_ARG
    badcam = camera(inputs.Camera(64, 48, -1.0, 60.0, 32.0, 24.0))
    assert L.gs_render_fwd(pr, None, None, None, badcam, None, None, None, None, None, None, None,
                           None) == _lib.GS_ERR_INVALID_ARG
    assert L.gs_tile_order(None, 10, None, None) == _lib.GS_ERR_INVALID_ARG
    assert L.gs_bin_sort(pr, 10, cam, None, 0, 100, C.c_void_p(16), C.c_void_p(16), None, C.c_void_p(16), None,
                         None, None, None) == _lib.GS_ERR_INVALID_ARG  # null projection arrays
    assert L.gs_loss(cam, None, None, None, None, None, 1.0, 1.0, None, 0, None, None, None, None) == _lib.GS_ERR_INVALID_ARG
    assert L.gs_render_bwd(p, C.c_void_p(16), cam, pr, None, C.c_void_p(16), None, C.c_void_p(16), C.c_void_p(16),
                           C.c_void_p(16), C.c_void_p(16), None, 0, None, 0, None, None, None, None, None,
                           None, None) == _lib.GS_ERR_INVALID_ARG  # flags = 0
    assert L.gs_pose_grad(None, None, 0, None, None, None, None, None, None) == _lib.GS_ERR_INVALID_ARG


def test_no_device_reports_error():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    L = _lib.lib()
    sm = C.c_int(0)
    assert L.gs_check_device(0, C.byref(sm)) == _lib.GS_ERR_CUDA
