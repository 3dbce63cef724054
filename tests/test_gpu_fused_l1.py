"""gs_render_fwd_l1 (S3 with S4's gradient fused, tracking) against the
separate calls: the frame is bit-identical to gs_render_fwd's and the
gradient maps to gs_loss's (weight 1); gs_loss_scales gives gs_loss's
scales; the fused tracking loop follows the unfused one."""
import numpy as np
import pytest
import torch

from paper_2312_10070_b200 import Params, Rasterizer, inputs

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


@pytest.mark.parametrize("cfg,lc,ld,holes", [(0, 1.0, 0.0, False), (1, 1.0, 1.0, True), (1, 0.5, 2.0, False)])
def test_fwd_l1_equals_fwd_then_loss(cfg, lc, ld, holes):
    s = inputs.CONFIGS[cfg]()
    P = Params.from_numpy(*s.params(), device=DEV)
    v = torch.as_tensor(s.views[0], device=DEV)
    r = Rasterizer(s.n, s.cam, device=DEV)
    r.size_for(P, v)
    rng = np.random.default_rng(cfg)
    H, W = s.cam.height, s.cam.width
    tc = torch.as_tensor(rng.uniform(0, 1, (3, H, W)).astype(np.float32), device=DEV)
    tdn = rng.uniform(0.5, 5, (H, W)).astype(np.float32)
    if holes:
        tdn[rng.uniform(size=(H, W)) < 0.2] = 0.0  # invalid target depths
    td = torch.as_tensor(tdn, device=DEV)
    r.forward(P, v)
    r.compute_loss(tc, td, None, lc, ld)
    ref = {k: getattr(r.frame, k).clone() for k in ("color", "depth", "alpha", "T_final", "n_contrib")}
    gc, gd = r.dL_dcolor.clone(), r.dL_ddepth.clone()
    r.dL_dcolor.fill_(7.0)
    r.dL_ddepth.fill_(7.0)
    sc = r.loss_scales(td, lc, ld)
    r.forward_l1(P, v, tc, td)
    torch.cuda.synchronize()
    nv = int((tdn > 0).sum())
    assert sc[0].item() == np.float32(lc / (3.0 * H * W))
    assert sc[1].item() == (np.float32(ld / nv) if nv else 0.0)
    for k, t in ref.items():
        assert torch.equal(getattr(r.frame, k), t), k
    assert torch.equal(r.dL_dcolor, gc)
    assert torch.equal(r.dL_ddepth, gd)


def test_fused_tracking_follows_unfused():
    from paper_2312_10070_b200.pipeline import TrackingLoop
    s = inputs.config2(n=40_000)
    P = Params.from_numpy(*s.params(), device=DEV)
    gt = torch.as_tensor(s.extra["gt_view"], device=DEV)
    r = Rasterizer(s.n, s.cam, device=DEV)
    r.size_for(P, gt)
    r.forward(P, gt)
    tc, td = r.frame.color.clone(), r.frame.depth.clone()
    views = []
    for fused in (True, False):
        loop = TrackingLoop(P, s.cam, tc, td, torch.as_tensor(s.extra["start_view"], device=DEV), iters=10,
                            fused_loss=fused)
        loop.size()
        loop.run()
        torch.cuda.synchronize()
        views.append(loop.view.cpu().numpy())
    # same gradient maps; only the fp32 atomic order of the backward differs
    assert np.allclose(views[0], views[1], rtol=0, atol=2e-5), views
