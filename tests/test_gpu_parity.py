"""Parity of the CUDA path (through the C-ABI) with the fp64 oracle on the same
seeded inputs.

Bars (BASELINE.json north_star): tile and sort indices bit-exact; colour,
depth, alpha <= 1e-4 absolute; gradients <= 1e-3 relative or 1e-6 x the
component's magnitude scale m* (R23).  Pixels whose fp64 decision margin is
below 1e-4 relative are "ambiguous" (R2): excluded from value checks and, for
gradient parity, their upstream maps are zeroed on both sides.
"""
import json
import os

import numpy as np
import pytest
import torch

from gpu_helpers import (AMBIG, GS_GRAD_PARAMS, GS_GRAD_POSE, gpu_backward, gpu_forward, gpu_frame, gpu_proj,
                         gpu_sort, grad_check, oracle, oracle_view, to_np)
from paper_2312_10070_b200 import inputs

pytestmark = pytest.mark.gpu

LOG = os.environ.get("GS_PARITY_LOG")


def log(name, **kw):
    if LOG:
        with open(LOG, "a") as f:
            f.write(json.dumps(dict(test=name, **kw), default=float) + "\n")


def _tilted(seed):
    """A random non-identity camera pose for the small scenes."""
    from scipy.spatial.transform import Rotation
    rng = np.random.default_rng(seed)
    R = Rotation.from_rotvec(rng.normal(0, 0.08, 3)).as_matrix()
    t = rng.normal(0, 0.05, 3)
    return np.concatenate([R.reshape(9), t]).astype(np.float32)


SCENES = {
    "tiny": lambda: inputs.config0(),
    "ragged37x29": lambda: inputs.random_scene(21, 300, 37, 29, spread=1.4, ls=(-2.0, 0.5)),
    "dense96x80": lambda: inputs.random_scene(22, 3000, 96, 80, spread=1.2, ls=(-2.6, 0.5), lo=(0.5, 1.5)),
    "tilted160x120": lambda: _with_view(inputs.random_scene(23, 4000, 160, 120, spread=1.3, ls=(-3.0, 0.6)), _tilted(1)),
}


def _with_view(s, v):
    s.views = v[None]
    return s


@pytest.fixture(scope="module", params=sorted(SCENES))
def case(request):
    s = SCENES[request.param]()
    r, P, v = gpu_forward(s)
    p64 = oracle.params64(*s.params())
    fr = oracle.forward(p64, oracle_view(s), s.cam)
    return dict(name=request.param, s=s, r=r, P=P, v=v, p64=p64, fr=fr)


# ---------------------------------------------------------------------------
# S1 projection

def test_project_parity(case):
    s, fr = case["s"], case["fr"]
    g = gpu_proj(case["r"])
    o = fr["proj"]
    vis = o["culled"] == 0
    assert np.array_equal(g["tiles_touched"] > 0, vis)
    assert np.array_equal(g["rect"][vis], o["rect"][vis])                     # bit-exact
    assert np.array_equal(g["depth"][vis], o["depth_key"][vis])               # bit-exact fp32 key
    assert np.all(np.isinf(g["depth"][~vis]))
    area = (o["rect"][:, 2] - o["rect"][:, 0] + 1) * (o["rect"][:, 3] - o["rect"][:, 1] + 1)
    assert np.array_equal(g["tiles_touched"][vis], area[vis])
    assert np.allclose(g["uv"][vis], o["uv"][vis], rtol=1e-14, atol=1e-12)
    assert np.allclose(g["conic_o"][vis, :3], o["conic"][vis], rtol=2e-7, atol=0)
    assert np.allclose(g["conic_o"][vis, 3], o["opac"][vis], rtol=2e-7)
    assert np.allclose(g["rgbz"][vis, 3], o["pz"][vis], rtol=1e-7)
    log("project", case=case["name"], n=int(s.n), visible=int(vis.sum()))


# ---------------------------------------------------------------------------
# S2 binning and depth order

def test_sort_parity(case):
    s, fr = case["s"], case["fr"]
    idx, rng = gpu_sort(case["r"])
    # (i) conditional: the oracle bins the GPU's own rects / keys -> must be identical
    g = gpu_proj(case["r"])
    culled = (g["tiles_touched"] == 0).astype(np.int32)
    oi, orng = oracle.bin_sort(g["rect"], culled, g["depth"], s.cam)
    assert np.array_equal(rng, orng)
    assert np.array_equal(idx, oi)
    # (ii) end to end against the oracle's own projection
    assert np.array_equal(rng, fr["tile_range"]) and np.array_equal(idx, fr["sorted_idx"])
    log("sort", case=case["name"], pairs=int(len(idx)))


def test_sort_without_order_matches(case):
    """gs_bin_sort without a launch order (tile_order = NULL, what the
    pipelines request) takes the one-CTA-per-tile-row counts step: the same
    tile ranges, sorted ids and pair count as with the order, and the same
    overflow outcome at a capacity one pair short."""
    r = case["r"]
    from paper_2312_10070_b200.raster import gs_bin_sort
    P = int(r.n_pairs.item())
    ref_idx, ref_rng = gpu_sort(r)
    for cap, over in ((r.capacity, False), (P - 1, True)):
        idx = torch.full_like(r.sorted_idx, -7)
        rng = torch.empty_like(r.tile_range)
        n_pairs = torch.zeros_like(r.n_pairs)
        cnt = torch.zeros_like(r.counters)
        gs_bin_sort(r.proj, r.n, r.cam, r.sort_ws, cap, idx, rng, n_pairs, cnt, tile_order=None)
        torch.cuda.synchronize()
        assert int(n_pairs.item()) == P
        if over:  # every range empty, the overflow counted (gs_counters.n_overflow)
            assert not to_np(rng).any() and int(to_np(cnt)[2]) == 1  # gs_counters: (nonfinite, culled, overflow, reserved)
        else:
            assert np.array_equal(to_np(rng), ref_rng)
            assert np.array_equal(to_np(idx)[:P], ref_idx)


def test_sort_without_order_wide_image():
    """The no-order counts step on an image wider than 128 tiles (its
    column chunks and carries): same ranges and ids as the ordered path and
    as the oracle's binning of the GPU projection."""
    s = inputs.random_scene(37, 3000, 2600, 40, spread=1.0)
    r, _, _ = gpu_forward(s)
    assert (s.cam.width + 15) // 16 > 128
    from paper_2312_10070_b200.raster import gs_bin_sort
    P = int(r.n_pairs.item())
    ref_idx, ref_rng = gpu_sort(r)
    idx = torch.full_like(r.sorted_idx, -7)
    rng = torch.empty_like(r.tile_range)
    n_pairs = torch.zeros_like(r.n_pairs)
    gs_bin_sort(r.proj, r.n, r.cam, r.sort_ws, r.capacity, idx, rng, n_pairs, None, tile_order=None)
    torch.cuda.synchronize()
    assert int(n_pairs.item()) == P
    assert np.array_equal(to_np(rng), ref_rng) and np.array_equal(to_np(idx)[:P], ref_idx)
    g = gpu_proj(r)
    oi, orng = oracle.bin_sort(g["rect"], (g["tiles_touched"] == 0).astype(np.int32), g["depth"], s.cam)
    assert np.array_equal(to_np(rng), orng) and np.array_equal(to_np(idx)[:P], oi)


def test_sort_ties_by_index():
    """R10: exact fp32 depth ties are ordered by Gaussian id (duplicates)."""
    s = inputs.random_scene(31, 400, 64, 48, spread=1.0)
    for arr in (s.mean_opa, s.quat, s.logscale, s.rgb):
        arr[1::2] = arr[0::2]
    r, _, _ = gpu_forward(s)
    idx, rng = gpu_sort(r)
    g = gpu_proj(r)
    for t in range(len(rng)):
        seg = idx[rng[t, 0]:rng[t, 1]]
        keys = g["depth"][seg]
        assert np.all((keys[1:] > keys[:-1]) | ((keys[1:] == keys[:-1]) & (seg[1:] > seg[:-1])))


def _conditional_sort_check(s):
    """The oracle bins the GPU's own rects / depth keys: bit-identical lists."""
    r, _, _ = gpu_forward(s, stats=False)
    idx, rng = gpu_sort(r)
    g = gpu_proj(r)
    culled = (g["tiles_touched"] == 0).astype(np.int32)
    oi, orng = oracle.bin_sort(g["rect"], culled, g["depth"], s.cam)
    assert np.array_equal(rng, orng) and np.array_equal(idx, oi)
    return rng


def test_sort_long_tiles():
    """Tile lists longer than one shared-memory chunk (4096 entries) take the
    chunked two-key path of gs_bin_sort."""
    s = inputs.random_scene(32, 9000, 40, 40, spread=0.6, ls=(-1.2, 0.2), lo=(2.0, 0.5))
    rng = _conditional_sort_check(s)
    assert (rng[:, 1] - rng[:, 0]).max() > 4096


def test_sort_dense_depth_cluster():
    """A tight cluster of depths next to one far outlier (the counting sort's
    buckets overflow) and long runs of exactly equal depths: both take the
    exact two-key path and must still equal the (depth, id) order."""
    s = inputs.random_scene(33, 3000, 48, 48, spread=0.9, ls=(-2.0, 0.3), lo=(2.0, 0.5))
    z = s.mean_opa[:, 2].astype(np.float64)
    z = 2.0 + (z - 1.0) * 1e-5                       # ~400 ulps of depth for 2999 Gaussians
    z[0] = 90.0                                      # far outlier covering the image
    s.mean_opa[:, 0] *= (z / s.mean_opa[:, 2]).astype(np.float32)
    s.mean_opa[:, 1] *= (z / s.mean_opa[:, 2]).astype(np.float32)
    s.mean_opa[:, 2] = z.astype(np.float32)
    s.logscale[0, :3] = 1.5
    s.mean_opa[1500:1700, 2] = np.float32(2.0)       # a run of 200 equal depths
    _conditional_sort_check(s)


# ---------------------------------------------------------------------------
# S3 compositing

def test_render_parity(case):
    s, fr = case["s"], case["fr"]
    g = gpu_frame(case["r"])
    ok = fr["margin"] > AMBIG
    amb = 1.0 - ok.mean()
    for key in ("depth", "alpha", "T_final"):
        err = np.abs(g[key] - fr[key])[ok]
        assert err.max(initial=0) <= 1e-4, (key, err.max())
    errc = np.abs(g["color"] - fr["color"])[:, ok]
    assert errc.max(initial=0) <= 1e-4
    for key in ("n_contrib", "scanned", "contrib"):
        assert np.array_equal(g[key][ok], fr[key][ok]), key
    assert amb < 0.02
    log("render", case=case["name"], ambiguous=amb, max_color_err=float(errc.max(initial=0)),
        max_depth_err=float(np.abs(g["depth"] - fr["depth"])[ok].max(initial=0)),
        mean_scanned=float(fr["scanned"].mean()), mean_contrib=float(fr["contrib"].mean()))


def test_render_deterministic(case):
    r = case["r"]
    a = gpu_frame(r)
    idx_a, _ = gpu_sort(r)
    r.forward(case["P"], case["v"], stats=True)
    torch.cuda.synchronize()
    b = gpu_frame(r)
    idx_b, _ = gpu_sort(r)
    assert np.array_equal(idx_a, idx_b)
    for k in a:
        assert np.array_equal(a[k], b[k]), k


# ---------------------------------------------------------------------------
# S4 loss

def test_loss_parity():
    s = inputs.config1()
    H, W = s.cam.height, s.cam.width
    rng = np.random.default_rng(5)
    color = rng.uniform(0, 1, (3, H, W)).astype(np.float32)
    depth = rng.uniform(0.5, 5, (H, W)).astype(np.float32)
    tc, td = s.extra["tgt_color"][0], s.extra["tgt_depth"][0].copy()
    td[::7] = 0.0
    w = rng.uniform(0.5, 1.5, (H, W)).astype(np.float32)
    from paper_2312_10070_b200 import Rasterizer
    r = Rasterizer(s.n, s.cam, device="cuda")
    d = torch.device("cuda")
    r.frame.color.copy_(torch.as_tensor(color))
    r.frame.depth.copy_(torch.as_tensor(depth))
    T = lambda a: torch.as_tensor(a, device=d)
    for weight in (None, w):
        r.compute_loss(T(tc), T(td), None if weight is None else T(weight), 0.7, 1.3)
        L, gc, gd = oracle.loss(s.cam, color, depth, tc, td, weight, 0.7, 1.3)
        assert np.allclose(to_np(r.loss)[:3], L, rtol=1e-6)
        assert np.allclose(to_np(r.dL_dcolor), gc, rtol=1e-6, atol=0)
        assert np.allclose(to_np(r.dL_ddepth), gd, rtol=1e-6, atol=0)
        l2 = to_np(r.compute_loss(T(tc), T(td), None if weight is None else T(weight), 0.7, 1.3)).copy()
        assert np.array_equal(l2, to_np(r.loss))  # bit-deterministic


# ---------------------------------------------------------------------------
# S5 + S6 backward, S7 pose

def _upstream(s, fr, seed=0):
    gc, gd, ga = inputs.upstream_maps(seed, s.cam)
    amb = fr["margin"] <= AMBIG
    gc = gc.copy()
    gd = gd.copy()
    ga = ga.copy()
    gc[:, amb] = 0
    gd[amb] = 0
    ga[amb] = 0
    return gc, gd, ga


def test_backward_parity(case):
    s, fr, r, P, v = case["s"], case["fr"], case["r"], case["P"], case["v"]
    gc, gd, ga = _upstream(s, fr)
    gb = gpu_backward(r, P, v, gc, gd, ga, GS_GRAD_PARAMS | GS_GRAD_POSE)
    ob = oracle.backward(case["p64"], oracle_view(s), s.cam, fr["sorted_idx"], fr["tile_range"], gc, gd, ga)
    ok2, st2 = grad_check(gb["g2"], ob["g2"], ob["m2"])
    ok3, st3 = grad_check(gb["g3"], ob["g3"], ob["m3"])
    log("backward", case=case["name"], g2=st2, g3=st3)
    assert ok2.all(), st2
    assert ok3.all(), st3


def test_pose_parity(case):
    s, fr, r, P, v = case["s"], case["fr"], case["r"], case["P"], case["v"]
    gc, gd, ga = _upstream(s, fr, seed=1)
    gpu_backward(r, P, v, gc, gd, ga, GS_GRAD_POSE)
    d = torch.device("cuda")
    dview = torch.zeros(12, device=d)
    dtw = torch.zeros(6, device=d)
    dqt = torch.zeros(7, device=d)
    r.pose_grad(v, dL_dview=dview, dL_dtwist=dtw, dL_dqt=dqt)
    torch.cuda.synchronize()
    ob = oracle.backward(case["p64"], oracle_view(s), s.cam, fr["sorted_idx"], fr["tile_range"], gc, gd, ga)
    ok, st = grad_check(to_np(dview), ob["pose"], ob["mpose"])
    log("pose", case=case["name"], view=st)
    assert ok.all(), (st, to_np(dview), ob["pose"])
    tw = oracle.pose_twist(ob["pose"], oracle_view(s))
    ok, st = grad_check(to_np(dtw), tw, twist_magnitude(ob["mpose"], oracle_view(s)))
    assert ok.all(), (st, to_np(dtw), tw)
    q = _quat_wxyz(oracle_view(s))  # (q, t) of T_wc (R22)
    ok, st = grad_check(to_np(dqt)[:4], oracle.pose_qt(ob["pose"], q), qt_magnitude(ob["mpose"][:9], q))
    assert ok.all(), (st, to_np(dqt)[:4])
    ok, st = grad_check(to_np(dqt)[4:], ob["pose"][9:], ob["mpose"][9:])
    assert ok.all(), st


def _quat_wxyz(view):
    """Unit quaternion (w, x, y, z), w >= 0, of the view's rotation (scipy,
    the nearest rotation of the fp32 matrix)."""
    from scipy.spatial.transform import Rotation
    x, y, z, w = Rotation.from_matrix(np.asarray(view[:9], np.float64).reshape(3, 3)).as_quat()
    q = np.array([w, x, y, z])
    return -q if q[0] < 0 else q


def qt_magnitude(mR, q):
    """|.|-propagation of the dL/dR magnitudes through dL/dq = (I - q q^T)
    sum_i dL/dR_i dR_i/dq (R22): m_k = sum_i |dR_i/dq_k| m_i +
    |q_k| sum_l |q_l| sum_i |dR_i/dq_l| m_i."""
    w, x, y, z = q
    D = np.array([[0, -2 * z, 2 * y, 2 * z, 0, -2 * x, -2 * y, 2 * x, 0],
                  [0, 2 * y, 2 * z, 2 * y, -4 * x, -2 * w, 2 * z, 2 * w, -4 * x],
                  [-4 * y, 2 * x, 2 * w, 2 * x, 0, 2 * z, -2 * w, 2 * z, -4 * y],
                  [-4 * z, -2 * w, 2 * x, 2 * w, -4 * z, 2 * y, 2 * x, 2 * y, 0]])
    raw = np.abs(D) @ mR
    return raw + np.abs(q) * (np.abs(q) @ raw)


def test_pose_qt_and_device_adam_steps_match_oracle():
    """S7 (R22, R28): gs_pose_grad's dL/d(q, t) of T_wc against oracle.pose_qt
    and three device Adam steps with the exp-map retraction (view and fp64 Adam
    state) against oracle.pose_adam, on fixed synthetic pose partials.  Both
    sides follow their own trajectory (the oracle never sees a GPU value); the
    GPU stores the view in fp32 (and re-orthonormalises R), so the views agree
    to ~1e-7 and the twists (linear in R, t) to ~1e-7 relative."""
    from paper_2312_10070_b200.raster import gs_pose_grad
    rng = np.random.default_rng(17)
    n_part = 37
    parts = rng.normal(0.0, 1.0, (n_part, 12)).astype(np.float32)
    view0 = _tilted(4)
    step = (2e-3, 1e-3, 0.9, 0.999, 1e-8)
    d = torch.device("cuda")
    v = torch.as_tensor(view0, device=d).contiguous()
    tparts = torch.as_tensor(parts, device=d)
    adam = torch.zeros(13, dtype=torch.float64, device=d)
    pose = parts.astype(np.float64).sum(0)                       # the fp64 reduction of the partials
    mpose = np.abs(parts.astype(np.float64)).sum(0)
    vo, st = view0.astype(np.float64), np.zeros(13)
    for k in range(3):
        dview = torch.zeros(12, device=d)
        dtw = torch.zeros(6, device=d)
        dqt = torch.zeros(7, device=d)
        gs_pose_grad(v, tparts, n_part, step, adam, dL_dview=dview, dL_dtwist=dtw, dL_dqt=dqt)
        torch.cuda.synchronize()
        # gradients at the view before the step
        assert np.allclose(to_np(dview), pose, rtol=1e-6, atol=1e-6 * mpose.max())
        tw = oracle.pose_twist(pose, vo)
        ok, st_tw = grad_check(to_np(dtw), tw, twist_magnitude(mpose, vo))
        assert ok.all(), (k, st_tw, to_np(dtw), tw)
        q = _quat_wxyz(vo)
        gq = oracle.pose_qt(pose, q)
        ok, st_q = grad_check(to_np(dqt)[:4], gq, qt_magnitude(mpose[:9], q))
        assert ok.all(), (k, st_q, to_np(dqt)[:4], gq)
        assert np.array_equal(to_np(dqt)[4:], to_np(dview)[9:])   # dL/dt of (q, t) = dL/dt
        vo, st = oracle.pose_adam(vo, tw, st, lr=step[:2], hyp=step[2:])
        gv, ga = to_np(v).astype(np.float64), to_np(adam)
        assert np.abs(gv - vo).max() <= 2e-6, (k, gv, vo)
        assert ga[12] == st[12] == k + 1
        assert np.allclose(ga[:6], st[:6], rtol=1e-5, atol=1e-9 * np.abs(st[:6]).max())
        assert np.allclose(ga[6:12], st[6:12], rtol=1e-5, atol=0)
        log("pose_adam", step=k, view_err=float(np.abs(gv - vo).max()), qt=st_q, twist=st_tw)


def twist_magnitude(mpose, view):
    """|.|-propagation of the (dR, dt) magnitudes through the linear map to the
    twist: m_v = m_t; m_w_k = sum |[e_k]x R| m_R + sum |e_k x t| m_t."""
    R = view[:9].reshape(3, 3)
    t = view[9:]
    mR = mpose[:9].reshape(3, 3)
    mt = mpose[9:]
    out = list(mt)
    for k in range(3):
        e = np.zeros(3)
        e[k] = 1.0
        E = np.array([[0, -e[2], e[1]], [e[2], 0, -e[0]], [-e[1], e[0], 0]])
        out.append((np.abs(E @ R) * mR).sum() + (np.abs(np.cross(e, t)) * mt).sum())
    return np.array(out)


def test_zero_gradient_for_non_contributors():
    """culled Gaussians get exact zeros (bit-exact on the GPU)."""
    s = inputs.random_scene(41, 200, 64, 48, spread=1.2)
    s.mean_opa[:20, 2] = -1.0  # behind the camera
    r, P, v = gpu_forward(s)
    gc, gd, ga = inputs.upstream_maps(2, s.cam)
    gb = gpu_backward(r, P, v, gc, gd, ga)
    assert np.array_equal(gb["g3"][:20], np.zeros((20, 16), np.float32))
    assert np.abs(gb["g3"][20:]).sum() > 0


# ---------------------------------------------------------------------------
# Edge cases

def test_empty_and_all_culled():
    for n in (0, 50):
        s = inputs.random_scene(51, n, 48, 40)
        if n:
            s.mean_opa[:, 2] = 200.0  # beyond z_far
        r, P, v = gpu_forward(s, capacity=16)
        g = gpu_frame(r)
        assert not g["color"].any() and not g["alpha"].any() and (g["T_final"] == 1).all()
        assert int(r.n_pairs.item()) == 0
        if n:
            assert int(r.counters[1].item()) == n
            gb = gpu_backward(r, P, v, *inputs.upstream_maps(0, s.cam))
            assert not gb["g3"].any()


def test_capacity_overflow_reports_and_renders_empty():
    s = inputs.random_scene(52, 500, 64, 48, spread=1.2)
    r, P, v = gpu_forward(s, capacity=10)
    assert int(r.counters[2].item()) == 1 and int(r.n_pairs.item()) > 10
    assert not to_np(r.tile_range).any()
    assert not gpu_frame(r)["alpha"].any()


def test_large_splat_covers_image():
    """One near, wide Gaussian whose rect is clamped to the whole image."""
    cam = inputs.Camera(100, 70, 90.0, 90.0, 49.5, 34.5)
    s = inputs.Scene("wide", cam, np.array([[0.0, 0.0, 1.0, 2.0]], np.float32), np.array([[1, 0, 0, 0]], np.float32),
                     np.array([[-0.5, -0.7, -0.6, 0]], np.float32), np.array([[0.3, 0.6, 0.9, 0]], np.float32),
                     inputs.identity_view()[None], 0)
    r, P, v = gpu_forward(s)
    fr = oracle.forward(oracle.params64(*s.params()), oracle_view(s), cam)
    g = gpu_frame(r)
    assert to_np(r.proj.tiles_touched)[0] == 7 * 5
    ok = fr["margin"] > AMBIG
    assert np.abs(g["color"] - fr["color"])[:, ok].max() <= 1e-4


@pytest.mark.parametrize("T", [1, 5, 1200, 3225, 8160, 20000])
def test_tile_orders_are_heaviest_first_permutations(T):
    """gs_tile_order (and gs_bin_sort's tile_order): a permutation of the
    tiles, bucket-major by 64 buckets of max / 64, heaviest bucket first."""
    import torch
    from paper_2312_10070_b200.raster import gs_tile_order
    rng = np.random.default_rng(T)
    work = rng.integers(0, 5000, T).astype(np.int32)
    work[rng.uniform(size=T) < 0.1] = 0
    w = torch.as_tensor(work, device="cuda")
    order = torch.full((T,), -1, dtype=torch.int32, device="cuda")
    gs_tile_order(w, T, order)
    torch.cuda.synchronize()
    o = order.cpu().numpy()
    assert np.array_equal(np.sort(o), np.arange(T))
    b = 63 - (work[o].astype(np.int64) * 64) // (int(work.max()) + 1)
    assert (np.diff(b) >= 0).all()


def test_bin_sort_tile_order_by_list_length():
    s = inputs.config1()
    r, P, v = gpu_forward(s)
    import torch
    torch.cuda.synchronize()
    o = r.tile_order.cpu().numpy()
    rng_ = r.tile_range.cpu().numpy().reshape(-1, 2)
    L = (rng_[:, 1] - rng_[:, 0]).astype(np.int64)
    assert np.array_equal(np.sort(o), np.arange(len(L)))
    b = 63 - (L[o] * 64) // (int(L.max()) + 1)
    assert (np.diff(b) >= 0).all()
