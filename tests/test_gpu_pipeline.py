"""The pipelined multi-view mapping step (pipeline.MapStep): gradients are the
sum of the single-view backward calls, independent of the number of stream
lanes, and the CUDA path's sharded sum equals the unsharded one."""
import numpy as np
import pytest
import torch

from paper_2312_10070_b200 import GS_GRAD_PARAMS, Grads, Params, Rasterizer, inputs
from paper_2312_10070_b200.pipeline import MapStep, shard_views

pytestmark = pytest.mark.gpu


def _small_submap(seed=5, n=40_000, V=4):
    s = inputs.config3(seed=seed, n=n, n_views=V)
    s.cam = inputs.Camera(320, 184, 160.0, 160.0, 159.5, 91.5)
    return s


def _targets(s, d):
    Pt = Params.from_numpy(*s.extra["target_params"], device=d)
    r = Rasterizer(s.n, s.cam, device=d)
    tc, td = {}, {}
    for v in range(s.views.shape[0]):
        vv = torch.as_tensor(s.views[v], device=d)
        r.size_for(Pt, vv)
        r.forward(Pt, vv)
        tc[v], td[v] = r.frame.color.clone(), r.frame.depth.clone()
    return tc, td


def test_mapstep_equals_sum_of_views_for_any_lanes():
    d = torch.device("cuda")
    s = _small_submap()
    P = Params.from_numpy(*s.params(), device=d)
    views = torch.as_tensor(s.views, device=d)
    tc, td = _targets(s, d)
    V = views.shape[0]
    # reference: one view at a time, same lambdas (1/V)
    ref = Grads.zeros(s.n, d)
    r = Rasterizer(s.n, s.cam, device=d)
    losses = []
    for v in range(V):
        r.size_for(P, views[v])
        r.forward(P, views[v])
        r.compute_loss(tc[v], td[v], None, 1.0 / V, 1.0 / V)
        losses.append(r.loss.clone())
        r.backward(P, views[v], GS_GRAD_PARAMS, ref)
    torch.cuda.synchronize()
    ref_np = ref.buf.cpu().numpy()
    scale = np.abs(ref_np).max()
    # atomic: per-view Gaussian phases add atomically (GS_BWD_ATOMIC_ACC,
    # unordered); else serialised in view order by events
    for lanes, atomic in ((1, True), (2, True), (3, True), (4, True), (4, False), (2, False), (8, True)):
        # the fused L1 loss (default) everywhere but the 2-lane serialised case
        ms = MapStep(P, views, s.cam, tc, td, lanes=lanes, device=d, atomic_gauss=atomic,
                     fused_loss=(lanes, atomic) != (2, False))
        ms.size()
        g = ms.step()
        torch.cuda.synchronize()
        got = g.buf.cpu().numpy()
        assert np.allclose(got, ref_np, rtol=1e-4, atol=1e-5 * scale), (lanes, atomic)
        assert np.allclose(ms.losses.cpu().numpy(), torch.stack(losses).cpu().numpy(), rtol=1e-6)
        g2 = ms.step()  # the grad2d scratches were left zeroed: a second step gives the same
        torch.cuda.synchronize()
        assert np.allclose(g2.buf.cpu().numpy(), got, rtol=1e-5, atol=1e-6 * scale), (lanes, atomic)


def test_sharded_sum_equals_unsharded():
    """Strong-scaling shards (round robin) summed = the 1-rank gradient."""
    d = torch.device("cuda")
    s = _small_submap(seed=6)
    P = Params.from_numpy(*s.params(), device=d)
    views = torch.as_tensor(s.views, device=d)
    tc, td = _targets(s, d)
    full = MapStep(P, views, s.cam, tc, td, device=d)
    full.size()
    g1 = full.step().buf.clone()
    acc = torch.zeros_like(g1)
    for rank in range(2):
        ms = MapStep(P, views, s.cam, tc, td, rank=rank, world=2, device=d, allreduce=lambda buf: None)
        assert ms.mine == shard_views(views.shape[0], rank, 2)
        ms.size()
        acc += ms.step().buf  # stands in for the NCCL SUM
    torch.cuda.synchronize()
    scale = g1.abs().max().item()
    assert torch.allclose(acc, g1, rtol=1e-4, atol=1e-5 * scale)


@pytest.mark.parametrize("frames", ["f32", "rgbd16"])
def test_mapstep_with_host_inputs(frames):
    """MapStep.step(host=HostInputs): inputs uploaded from pinned host memory
    inside the step (parameters in two parts, the frames view by view, as
    8-bit RGB + 16-bit depth unpacked by gs_unpack_rgbd for "rgbd16") give
    the step of device-resident inputs holding the same values; the per-view
    losses are read back into host.loss."""
    from oracle import rgbd
    from paper_2312_10070_b200.pipeline import HostInputs
    d = torch.device("cuda")
    s = _small_submap(seed=6)
    P = Params.from_numpy(*s.params(), device=d)
    views = torch.as_tensor(s.views, device=d)
    tc, td = _targets(s, d)
    V = views.shape[0]
    if frames == "rgbd16":  # the device-resident reference holds the unpacked sensor frames
        for v in range(V):
            r8, d16 = inputs.quantize_rgbd(tc[v].cpu().numpy(), td[v].cpu().numpy())
            c, z = rgbd.unpack(r8, d16, inputs.DEPTH_SCALE)
            tc[v], td[v] = torch.as_tensor(c, device=d), torch.as_tensor(z, device=d)
    ms = MapStep(P, views, s.cam, tc, td, lanes=4, device=d)
    ms.size()
    ref = ms.step().buf.clone()
    ref_loss = ms.losses.clone()
    torch.cuda.synchronize()
    host = HostInputs(ms.params, ms.views, ms.tgt_color, ms.tgt_depth, ms.mine, ms.losses.shape[0], frames=frames)
    # scribble over the device copies: the step must bring everything from the host
    for name in ("mean_opa", "quat", "logscale", "rgb"):
        getattr(ms.params, name).fill_(float("nan"))
    ms.views.zero_()
    for v in range(V):
        ms.tgt_color[v].fill_(-1.0)
        ms.tgt_depth[v].fill_(-1.0)
    for _ in range(2):
        g = ms.step(host=host)
    torch.cuda.synchronize()
    scale = ref.abs().max()
    assert torch.allclose(g.buf, ref, rtol=1e-4, atol=1e-5 * scale)
    assert torch.allclose(host.loss, ref_loss.cpu(), rtol=1e-6, atol=0)
    assert host.h2d_bytes() == 4 * s.n * 16 + V * 48 + (
        V * s.cam.width * s.cam.height * (5 if frames == "rgbd16" else 16))


def test_step_checked_resizes_on_overflow():
    """Gaussians that grow after sizing overflow the pair capacity (the view
    renders empty and n_overflow counts it); step_checked re-sizes and
    repeats the step, matching a step sized for the grown Gaussians."""
    d = torch.device("cuda")
    s = _small_submap(seed=7)
    P = Params.from_numpy(*s.params(), device=d)
    views = torch.as_tensor(s.views, device=d)
    tc, td = _targets(s, d)
    ms = MapStep(P, views, s.cam, tc, td, lanes=2, device=d)
    ms.size(slack=1.0)
    P.logscale[:, :3] += 0.7  # ~2x larger splats: many more (tile, Gaussian) pairs
    ms.step()
    torch.cuda.synchronize()
    assert ms.overflowed() > 0  # the unchecked step lost views
    g = ms.step_checked().buf.clone()
    torch.cuda.synchronize()
    ref_ms = MapStep(P, views, s.cam, tc, td, lanes=2, device=d)
    ref_ms.size()
    ref = ref_ms.step().buf.clone()
    torch.cuda.synchronize()
    assert ms.overflowed() == 0 and ref_ms.overflowed() == 0
    assert np.allclose(g.cpu().numpy(), ref.cpu().numpy(), rtol=1e-4, atol=1e-5 * ref.abs().max().item())


def test_mapstep_matches_oracle():
    """The benched mapping step (fused L1 loss in the compositing kernel, one
    lane per view, atomic per-view S6) against the fp64 oracle's mapping
    iteration (Eq. 12 summed over the keyframes) on BJ.configs[3]
    reduced to 40k Gaussians and 4 views of 320x184: the summed gradient per
    component under R23, the per-view losses at rtol 1e-6.  The oracle's
    ambiguous pixels (R2, R21) get zero upstream on both sides (a bwd-stage hook
    masks the GPU's fused gradient maps; everything else is the step as benched)."""
    from gpu_helpers import grad_check, grads_as_g3, oracle_mapping_reference, small_submap, zero_upstream_hook
    d = torch.device("cuda")
    s = small_submap(seed=8)
    ref = oracle_mapping_reference(s)
    P = Params.from_numpy(*s.params(), device=d)
    views = torch.as_tensor(s.views, device=d)
    V = views.shape[0]
    tc = {v: torch.as_tensor(ref["tc"][v], device=d) for v in range(V)}
    td = {v: torch.as_tensor(ref["td"][v], device=d) for v in range(V)}
    amb = {v: torch.as_tensor(ref["amb"][v], device=d) for v in range(V)}
    ms = MapStep(P, views, s.cam, tc, td, device=d)  # benched defaults: 8 lanes, fused L1, atomic S6
    assert ms.fused_loss and ms.atomic_gauss and len(ms.lanes) == V
    ms.size()
    # step 1: stream-ordered stages; step 2 on: each view's per-pixel backward
    # overlaps its forward tile by tile (MapStep.overlap, previous work order)
    ms.overlap = True
    for it in range(2):
        g = ms.step(hooks={"bwd": zero_upstream_hook(ms, amb)})
        torch.cuda.synchronize()
        ok, st = grad_check(grads_as_g3(g), ref["g3"], ref["m3"])
        assert ok.all(), (it, st)
        loss = ms.losses.cpu().numpy()[:, :3].astype(np.float64)
        assert np.allclose(loss, ref["loss"], rtol=1e-6, atol=0), (it, loss, ref["loss"])
        assert all(r.flag_timeouts() == 0 for r in ms.lanes)
    amb_frac = float(np.mean([ref["amb"][v].mean() for v in range(V)]))
    assert amb_frac < 0.02


def test_mapstep_graph_replay_equals_eager():
    """MapStep.capture / replay (the bench's timed path): the same summed
    gradient and per-view losses as the eager step (atomic accumulation:
    up to float rounding of the sum order)."""
    from gpu_helpers import oracle_mapping_reference, small_submap
    s = small_submap(seed=5)
    d = torch.device("cuda")
    P = Params.from_numpy(*s.params(), device=d)
    views = torch.as_tensor(s.views, device=d)
    ref = oracle_mapping_reference(s)
    V = s.views.shape[0]
    tc = {v: torch.as_tensor(ref["tc"][v], device=d) for v in range(V)}
    td = {v: torch.as_tensor(ref["td"][v], device=d) for v in range(V)}
    ms = MapStep(P, views, s.cam, tc, td, device=d)
    ms.overlap = True
    ms.size()
    for _ in range(3):
        ms.step()
    eager = ms.step().buf.clone()
    eager_loss = ms.losses.clone()
    ms.capture()
    for _ in range(2):
        got = ms.replay().buf
    torch.cuda.synchronize()
    scale = eager.abs().max().item()
    assert torch.allclose(got, eager, rtol=1e-5, atol=1e-6 * scale)
    assert torch.allclose(ms.losses, eager_loss, rtol=1e-6, atol=0)
