"""Parity of gs_tracking_loss (Eq. 15 masked tracking loss, NEXT(1)) with the
oracle on identical fp32 maps: medians and masks bit-exact (R31), loss within
1e-6 relative, gradient maps within 1e-6 relative (fp32 weights vs fp64)."""
import numpy as np
import pytest
import torch

from oracle import tracking as T
from paper_2312_10070_b200 import Params, Rasterizer, inputs
from paper_2312_10070_b200.raster import camera, gs_tracking_loss, lib

pytestmark = pytest.mark.gpu


def _gpu(c, d, a, tc, td, lam, mult):
    dev = torch.device("cuda:0")
    H, W = d.shape
    cam = camera(inputs.Camera(W, H, 1.0, 1.0, 0.0, 0.0))
    t = lambda x: torch.as_tensor(np.ascontiguousarray(x, np.float32), device=dev)
    ws = torch.empty((lib().gs_tracking_loss_workspace_bytes(cam) + 15) // 16 * 4, dtype=torch.float32, device=dev)
    loss = torch.zeros(4, dtype=torch.float32, device=dev)
    gc = torch.full((3, H, W), np.nan, dtype=torch.float32, device=dev)
    gd = torch.full((H, W), np.nan, dtype=torch.float32, device=dev)
    gs_tracking_loss(cam, t(c), t(d), t(a), t(tc), t(td), lam, mult, ws, loss, gc, gd)
    torch.cuda.synchronize()
    return loss.cpu().numpy(), gc.cpu().numpy(), gd.cpu().numpy()


def _check(c, d, a, tc, td, lam=0.5, mult=50.0):
    o = T.tracking_loss(c, d, a, tc, td, lam, mult)
    loss, gc, gd = _gpu(c, d, a, tc, td, lam, mult)
    assert loss[1] == o["med_c"] and loss[2] == o["med_d"]          # exact order statistics
    assert int(loss[3]) == int(o["inlier"].sum())
    assert abs(loss[0] - o["loss"]) <= 1e-6 * max(abs(o["loss"]), 1e-30)
    w = o["inlier"] * o["m_alpha"]
    if lam < 1:  # the mask, bit for bit
        assert np.array_equal(gd != 0, (w > 0) & (np.float32(d) != np.float32(td)))
    if lam > 0:
        assert np.array_equal((gc != 0).any(0), (w > 0) & (np.float32(c) != np.float32(tc)).any(0))
    np.testing.assert_allclose(gc, o["g_color"], rtol=1e-6, atol=1e-12)
    np.testing.assert_allclose(gd, o["g_depth"], rtol=1e-6, atol=1e-12)
    return o


def _maps(seed, H, W, invalid=0.1, quant=None):
    rng = np.random.default_rng(seed)
    c = rng.uniform(0, 1, (3, H, W)).astype(np.float32)
    tc = rng.uniform(0, 1, (3, H, W)).astype(np.float32)
    d = rng.uniform(0.5, 4, (H, W)).astype(np.float32)
    td = (d + rng.laplace(0, 0.02, (H, W))).astype(np.float32)
    if quant:  # many exactly equal errors (ties at the median)
        c = (np.round(c * quant) / quant).astype(np.float32)
        tc = (np.round(tc * quant) / quant).astype(np.float32)
        td = (d + np.round(rng.laplace(0, 0.02, (H, W)) * 100) / 100).astype(np.float32)
    td[rng.uniform(size=(H, W)) < invalid] = 0.0
    a = rng.uniform(0, 1, (H, W)).astype(np.float32)
    return c, d, a, tc, td


@pytest.mark.parametrize("shape", [(48, 64), (37, 29), (480, 640)])
def test_tracking_loss_parity(shape):
    H, W = shape
    o = _check(*_maps(1, H, W), lam=0.5)
    assert 0 < o["inlier"].sum() < (H * W)


def test_tracking_loss_ties_and_outliers():
    c, d, a, tc, td = _maps(2, 96, 128, quant=8)
    d[10:20, 10:20] += 3.0  # a block of gross depth outliers
    o = _check(c, d, a, tc, td, lam=0.9, mult=50.0)
    assert not o["inlier"][10:20, 10:20].any()
    _check(c, d, a, tc, td, lam=0.0, mult=2.0)
    _check(c, d, a, tc, td, lam=1.0, mult=1.0)


def test_tracking_loss_degenerate():
    c, d, a, tc, td = _maps(3, 32, 32)
    td0 = np.zeros_like(td)
    loss, gc, gd = _gpu(c, d, a, tc, td0, 0.5, 50.0)
    assert loss.tolist() == [0.0, 0.0, 0.0, 0.0] and not gc.any() and not gd.any()
    # zero error everywhere: median 0, only exact matches are inliers
    _check(c, d, a, c.copy(), d.copy(), 0.5, 50.0)
    # a single valid pixel
    td1 = np.zeros_like(td)
    td1[5, 7] = 2.0
    _check(c, d, a, tc, td1)


def test_tracking_loss_full_size_rendered():
    """BJ.configs[2] sizes: maps rendered by this path at the perturbed start
    pose against the GT render; the oracle runs on the same fp32 maps."""
    s = inputs.config2()
    dev = torch.device("cuda:0")
    P = Params.from_numpy(*s.params(), device=dev)
    r = Rasterizer(s.n, s.cam, device=dev)
    gt = torch.as_tensor(s.extra["gt_view"], device=dev)
    r.size_for(P, gt)
    r.forward(P, gt)
    tc, td = r.frame.color.clone(), r.frame.depth.clone()
    r.forward(P, torch.as_tensor(s.extra["start_view"], device=dev))
    torch.cuda.synchronize()
    f = r.frame
    _check(f.color.cpu().numpy(), f.depth.cpu().numpy(), f.alpha.cpu().numpy(), tc.cpu().numpy(), td.cpu().numpy(),
           lam=0.5)


def test_masked_tracking_loop_converges():
    """The 100-iteration tracking graph with the Eq. 15 loss recovers the
    2 deg / 5 cm perturbation of BJ.configs[2] (sanity, not parity)."""
    from paper_2312_10070_b200.pipeline import TrackingLoop
    s = inputs.config2()
    dev = torch.device("cuda:0")
    P = Params.from_numpy(*s.params(), device=dev)
    r = Rasterizer(s.n, s.cam, device=dev)
    gt = torch.as_tensor(s.extra["gt_view"], device=dev)
    r.size_for(P, gt)
    r.forward(P, gt)
    tc, td = r.frame.color.clone(), r.frame.depth.clone()
    loop = TrackingLoop(P, s.cam, tc, td, torch.as_tensor(s.extra["start_view"], device=dev), iters=100,
                        masked=(0.5, 50.0))
    loop.size()
    loop.capture()
    loop.run()
    torch.cuda.synchronize()
    v = loop.view.cpu().numpy().astype(np.float64)
    R, t = v[:9].reshape(3, 3), v[9:]
    rot = np.degrees(np.arccos(np.clip((np.trace(R) - 1) / 2, -1, 1)))
    assert rot < 0.5 and np.linalg.norm(t) < 0.01
