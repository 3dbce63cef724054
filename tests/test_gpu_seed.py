"""Parity of gs_seed (NEXT(4) sub-map seeding) with the oracle on the same
inputs: the sampled pixels and their order, the accepted set and the new
Gaussians' means and colours bit-exact (integer and fp64 decisions, R38-R40),
log-scales within 1e-6 (fp64 log, rounded to fp32)."""
import numpy as np
import pytest
import torch

from oracle import seed as S
from paper_2312_10070_b200 import Params, Rasterizer, inputs
from paper_2312_10070_b200.raster import camera, gs_seed, lib

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def _run(color, depth, alpha, view, cam_py, means, max_new, seed, rho=0.01, alpha_n=0.6):
    n = len(means)
    cap = n + max_new
    arr = np.zeros((max(cap, 1), 4), np.float32)
    mo = arr.copy()
    mo[:n] = means
    P = Params.from_numpy(mo, arr.copy(), arr.copy(), arr.copy(), device=DEV)
    cam = camera(cam_py)
    ws = torch.empty((lib().gs_seed_workspace_bytes(cam, n, max_new) + 15) // 16 * 4, dtype=torch.float32, device=DEV)
    n_new = torch.zeros(1, dtype=torch.int32, device=DEV)
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a, np.float32), device=DEV)
    gs_seed(cam, view, t(color), t(depth), t(alpha), alpha_n, rho, max_new, seed, P, n, ws, n_new)
    torch.cuda.synchronize()
    k = int(n_new.item())
    return k, {name: getattr(P, name).cpu().numpy()[n:n + k] for name in ("mean_opa", "quat", "logscale", "rgb")}


def _check(color, depth, alpha, view, cam, means, max_new=100000, seed=0, rho=0.01):
    o = S.seed(color, depth, alpha, view, cam, means, rho=rho, max_new=max_new, seed_=seed)
    k, g = _run(color, depth, alpha, view, cam, means, max_new, seed, rho)
    assert k == int(o["accepted"].sum())
    assert np.array_equal(g["mean_opa"], o["mean_opa"])
    assert np.array_equal(g["quat"], o["quat"])
    assert np.array_equal(g["rgb"], o["rgb"])
    np.testing.assert_allclose(g["logscale"], o["logscale"], rtol=1e-6, atol=1e-7)
    return o


def test_seed_parity_wall_with_submap():
    H, W = 60, 80
    rng = np.random.default_rng(0)
    color = rng.uniform(0, 1, (3, H, W)).astype(np.float32)
    depth = (2.0 + 0.05 * rng.standard_normal((H, W))).astype(np.float32)
    depth[rng.uniform(size=(H, W)) < 0.05] = 0.0
    alpha = rng.uniform(0, 1, (H, W)).astype(np.float32)
    cam = inputs.Camera(W, H, 400.0, 400.0, (W - 1) / 2, (H - 1) / 2)
    ex = np.concatenate([rng.uniform(-0.2, 0.2, (3000, 2)), 2.0 + 0.05 * rng.standard_normal((3000, 1)),
                         np.zeros((3000, 1))], axis=1).astype(np.float32)
    view = np.array([0.98, -0.2, 0, 0.2, 0.98, 0, 0, 0, 1, 0.01, -0.02, 0.03], np.float32)
    o = _check(color, depth, alpha, view, cam, ex, max_new=1500, seed=11)
    assert 0 < o["accepted"].sum() < len(o["idx"]) == 1500


@pytest.mark.parametrize("max_new", [0, 1, 10, 100000])
def test_seed_parity_empty_submap(max_new):
    H, W = 33, 47
    rng = np.random.default_rng(1)
    color = rng.uniform(0, 1, (3, H, W)).astype(np.float32)
    depth = rng.uniform(0.5, 4.0, (H, W)).astype(np.float32)
    alpha = rng.uniform(0, 1, (H, W)).astype(np.float32)
    cam = inputs.Camera(W, H, 40.0, 40.0, 23.0, 16.0)
    view = np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0], np.float32)
    _check(color, depth, alpha, view, cam, np.zeros((0, 4), np.float32), max_new=max_new, seed=5)


def test_seed_from_rendered_alpha_full_size():
    """BJ.configs[1] (640x480): the rendered alpha of the scene gates the
    candidates of a synthetic RGB-D frame (depth = the render's depth
    normalised by alpha, 2 cm noise); the volume-filling scene is opaque, so
    an unmapped 200 x 150 window (alpha 0, depth 3 m) supplies the seeds."""
    s = inputs.config1()
    P = Params.from_numpy(*s.params(), device=DEV)
    v = torch.as_tensor(s.views[0], device=DEV)
    r = Rasterizer(s.n, s.cam, device=DEV)
    r.size_for(P, v)
    r.forward(P, v)
    a = r.frame.alpha.cpu().numpy()
    d = np.where(a > 0, r.frame.depth.cpu().numpy() / np.maximum(a, 1e-6), 0).astype(np.float32)
    rng = np.random.default_rng(3)
    d = np.where(d > 0, d + 0.02 * rng.standard_normal(d.shape), 0).astype(np.float32)
    a = a.copy()
    a[100:250, 200:400] = 0.0
    d[100:250, 200:400] = 3.0
    c = r.frame.color.cpu().numpy()
    o = _check(c, d, a, s.views[0], s.cam, s.params()[0][:20000], max_new=4000, seed=7)
    assert o["accepted"].sum() > 0


@pytest.mark.parametrize("W,H,q", [(37, 23, 0.95), (64, 48, 0.9), (2, 2, 0.95), (1200, 680, 0.95)])
def test_gradient_mask_parity(W, H, q):
    """R43: the high-colour-gradient set and its nearest-rank threshold,
    bit-exact (fp64 Sobel in the oracle's order, exact radix select)."""
    from paper_2312_10070_b200.raster import gs_gradient_mask
    rng = np.random.default_rng(W + H)
    color = rng.uniform(0, 1, (3, H, W)).astype(np.float32)
    color[:, :, W // 2:] *= 0.3
    color[:, ::7] = 0.5  # ties in m2
    depth = rng.uniform(0.5, 4.0, (H, W)).astype(np.float32)
    depth[rng.uniform(size=(H, W)) < 0.1] = 0.0
    cam = camera(inputs.Camera(W, H, 100.0, 100.0, W / 2, H / 2))
    ws = torch.empty((lib().gs_gradient_mask_workspace_bytes(cam) + 15) // 16 * 4, dtype=torch.float32, device=DEV)
    pa = torch.full((H, W), -1.0, device=DEV)
    thr = torch.zeros(1, dtype=torch.float64, device=DEV)
    t = lambda a: torch.as_tensor(a, device=DEV)
    gs_gradient_mask(cam, t(color), t(depth), q, pa, ws, threshold_m2=thr)
    torch.cuda.synchronize()
    m2 = S.gradient_m2(color)
    assert thr.item() == S.gradient_threshold(m2, q)
    mask = S.gradient_mask(color, depth, q)
    assert np.array_equal(pa.cpu().numpy(), np.where(mask, 0.0, 1.0).astype(np.float32))


def test_first_keyframe_parity():
    """P:156 / R43: the M_u uniform batch, then the M_c gradient batch against
    it, equal to the oracle's two batches (counts, means, colours, rotations
    bit-exact; log-scales within 1e-6)."""
    from paper_2312_10070_b200.raster import seed_first_keyframe
    H, W = 60, 80
    rng = np.random.default_rng(9)
    color = rng.uniform(0, 1, (3, H, W)).astype(np.float32)
    color[:, 20:40, 30:50] = 0.9  # a bright square: strong edges
    depth = (2.0 + 0.05 * rng.standard_normal((H, W))).astype(np.float32)
    depth[rng.uniform(size=(H, W)) < 0.05] = 0.0
    cam_py = inputs.Camera(W, H, 400.0, 400.0, (W - 1) / 2, (H - 1) / 2)
    view = np.array([0.98, -0.2, 0, 0.2, 0.98, 0, 0, 0, 1, 0.01, -0.02, 0.03], np.float32)
    M_u, M_c = 1200, 300
    r1, r2 = S.first_keyframe(color, depth, view, cam_py, M_u, M_c, seed_=4)
    cap = M_u + M_c
    z = np.zeros((cap, 4), np.float32)
    P = Params.from_numpy(z, z, z, z, device=DEV)
    t = lambda a: torch.as_tensor(a, device=DEV)
    n_u, n_c = seed_first_keyframe(camera(cam_py), view, t(color), t(depth), P, 0, M_u, M_c, 4)
    torch.cuda.synchronize()
    assert n_u == int(r1["accepted"].sum()) and n_c == int(r2["accepted"].sum()) and n_c > 0
    for name, k0, k1, o in (("mean_opa", 0, n_u, r1), ("mean_opa", n_u, n_u + n_c, r2)):
        assert np.array_equal(P.mean_opa.cpu().numpy()[k0:k1], o["mean_opa"])
    got = {k: getattr(P, k).cpu().numpy() for k in ("quat", "rgb", "logscale")}
    for k0, k1, o in ((0, n_u, r1), (n_u, n_u + n_c, r2)):
        assert np.array_equal(got["quat"][k0:k1], o["quat"])
        assert np.array_equal(got["rgb"][k0:k1], o["rgb"])
        np.testing.assert_allclose(got["logscale"][k0:k1], o["logscale"], rtol=1e-6, atol=1e-7)
