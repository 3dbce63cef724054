"""gs_unpack_rgbd vs the oracle: bit-exact (IEEE fp32 division / product),
vector path (HW % 4 == 0) and scalar path (ragged), incl. a full-size frame."""
import numpy as np
import pytest
import torch

from oracle import rgbd
from paper_2312_10070_b200 import inputs
from paper_2312_10070_b200.raster import camera, gs_unpack_rgbd

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


@pytest.mark.parametrize("W,H,scale", [(64, 48, 1 / 5000), (33, 17, 1 / 6553.5), (1, 1, 0.001), (1200, 680, 1 / 5000)])
def test_unpack_parity(W, H, scale):
    rng = np.random.default_rng(W * H)
    rgb = rng.integers(0, 256, (H, W, 3), dtype=np.uint8)
    d = rng.integers(0, 65536, (H, W), dtype=np.uint16)
    d[rng.uniform(size=(H, W)) < 0.1] = 0
    cam = camera(inputs.Camera(W, H, 100.0, 100.0, W / 2, H / 2))
    c = torch.full((3, H, W), -1.0, device=DEV)
    z = torch.full((H, W), -1.0, device=DEV)
    gs_unpack_rgbd(cam, torch.as_tensor(rgb, device=DEV), torch.as_tensor(d.view(np.int16), device=DEV), scale, c, z)
    torch.cuda.synchronize()
    oc, oz = rgbd.unpack(rgb, d, scale)
    assert np.array_equal(c.cpu().numpy(), oc)
    assert np.array_equal(z.cpu().numpy(), oz)


@pytest.mark.parametrize("W,H,lc,ld", [(64, 48, 1.0, 1.0), (33, 17, 0.5, 2.0), (1200, 680, 1.0, 1.0)])
def test_unpack_scales_equal_gs_loss_scales(W, H, lc, ld):
    """gs_unpack_rgbd(scales): the frame's gs_loss_scales from the unpacking
    pass, bit-identical to the separate call (incl. frames without valid depth)."""
    from paper_2312_10070_b200.raster import gs_loss_scales, lib
    rng = np.random.default_rng(W)
    rgb = rng.integers(0, 256, (H, W, 3), dtype=np.uint8)
    for frac in (0.3, 1.0):
        d = rng.integers(1, 65536, (H, W), dtype=np.uint16)
        d[rng.uniform(size=(H, W)) < frac] = 0
        cam = camera(inputs.Camera(W, H, 100.0, 100.0, W / 2, H / 2))
        c = torch.empty((3, H, W), device=DEV)
        z = torch.empty((H, W), device=DEV)
        sc = torch.full((4,), 7.0, device=DEV)
        gs_unpack_rgbd(cam, torch.as_tensor(rgb, device=DEV), torch.as_tensor(d.view(np.int16), device=DEV),
                       1 / 5000, c, z, scales=sc, lambda_color=lc, lambda_depth=ld)
        ws = torch.empty((lib().gs_loss_workspace_bytes(cam) + 15) // 16 * 4, dtype=torch.float32, device=DEV)
        ref = torch.zeros(4, device=DEV)
        gs_loss_scales(cam, z, lc, ld, ws, ref)
        torch.cuda.synchronize()
        assert torch.equal(sc, ref), (sc, ref)
        assert int(sc[2].item()) == int((d > 0).sum())
