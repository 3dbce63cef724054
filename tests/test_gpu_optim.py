"""Parity of the mapping epilogue (NEXT(3)) with the fp64 oracle: Eq. 11
regulariser (loss within 1e-6 relative, gradient within 1e-5), Adam steps
(parameters / moments within fp32 rounding), opacity pruning (bit-exact
compaction); plus a mapping loop that lowers the loss."""
import numpy as np
import pytest
import torch

from oracle import optim as O
from paper_2312_10070_b200 import Grads, Params, inputs
from paper_2312_10070_b200.raster import Optimizer

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def _params(n, seed):
    rng = np.random.default_rng(seed)
    mo = rng.normal(size=(n, 4)).astype(np.float32)
    q = rng.normal(size=(n, 4))
    q = (q / np.linalg.norm(q, axis=1, keepdims=True)).astype(np.float32)
    ls = rng.normal(-3.0, 0.6, (n, 4)).astype(np.float32)
    rgb = rng.uniform(0, 1, (n, 4)).astype(np.float32)
    return mo, q, ls, rgb


def _np(P: Params):
    return {k: getattr(P, k).cpu().numpy().astype(np.float64) for k in O.NAMES}


@pytest.mark.parametrize("n", [1, 1000, 10007])
def test_iso_reg_parity(n):
    P = Params.from_numpy(*_params(n, n), device=DEV)
    g = Grads.zeros(n, DEV)
    g.logscale.normal_()
    g0 = g.logscale.cpu().numpy().astype(np.float64)
    opt = Optimizer(n, DEV)
    reg = opt.regularize(P, g, 0.7).cpu().numpy()
    L, gl = O.iso_reg(P.logscale.cpu().numpy())
    assert abs(reg[1] - L) <= 1e-6 * L and abs(reg[0] - 0.7 * L) <= 1e-6 * L
    got = g.logscale.cpu().numpy()
    np.testing.assert_allclose(got[:, :3], g0[:, :3] + 0.7 * gl, rtol=1e-5, atol=1e-6 / n)
    assert np.array_equal(got[:, 3], g0[:, 3])


def test_adam_parity():
    n = 5000
    P = Params.from_numpy(*_params(n, 3), device=DEV)
    opt = Optimizer(n, DEV)
    p = _np(P)
    z = {k: np.zeros((n, 4)) for k in O.NAMES}
    m, v = dict(z), dict(z)
    rng = np.random.default_rng(4)
    for t in range(1, 4):
        gn = {k: rng.normal(0, 10 ** rng.uniform(-3, 0), (n, 4)).astype(np.float32) for k in O.NAMES}
        if t == 2:
            gn["quat"][17, 2] = np.inf  # skipped entry
        g = Grads(torch.as_tensor(np.stack([gn[k] for k in O.NAMES]), device=DEV).contiguous())
        cnt = torch.zeros(4, dtype=torch.int64, device=DEV)
        opt.step(P, g, cnt)
        p, m, v, ns = O.adam_step(p, gn, m, v, t, opt.lr)
        assert int(cnt[0].item()) == ns  # n_nonfinite
    got = _np(P)
    for k in O.NAMES:
        np.testing.assert_allclose(got[k], p[k], rtol=2e-5, atol=2e-6)
    mom = opt.moments.cpu().numpy().astype(np.float64)
    for i, k in enumerate(O.NAMES):
        # fp32 moments: cancellation between steps' gradients -> absolute floor at the array's scale
        np.testing.assert_allclose(mom[:, i], m[k], rtol=1e-5, atol=1e-6 * np.abs(m[k]).max())
        np.testing.assert_allclose(mom[:, 4 + i], v[k], rtol=1e-5, atol=1e-6 * np.abs(v[k]).max())


@pytest.mark.parametrize("n", [0, 1, 257, 20000])
def test_prune_parity(n):
    arrs = _params(max(n, 1), 5)
    mo = arrs[0]
    rng = np.random.default_rng(6)
    o = rng.uniform(0.0, 0.3, max(n, 1))
    mo[:, 3] = np.log(o / (1 - o)).astype(np.float32)
    arrs = tuple(a[:n] for a in arrs)
    P = Params.from_numpy(*arrs, device=DEV) if n else Params.from_numpy(*[np.zeros((0, 4), np.float32)] * 4,
                                                                          device=DEV)
    opt = Optimizer(n, DEV)
    opt.moments.normal_()
    out = Params.from_numpy(*[np.zeros((max(n, 1), 4), np.float32)] * 4, device=DEV)
    mout = torch.zeros_like(opt.moments)
    k = int(opt.prune(P, 0.1, out, mout).item())
    keep = O.prune_keep(arrs[0][:, 3], 0.1) if n else np.zeros(0, bool)
    assert k == int(keep.sum())
    for name, a in zip(O.NAMES, arrs):
        assert np.array_equal(getattr(out, name).cpu().numpy()[:k], a[keep])
    if n:
        assert np.array_equal(mout.cpu().numpy()[:k], opt.moments.cpu().numpy()[:n][keep])


def test_mapping_loop_lowers_the_loss():
    """BJ.configs[1]-sized scene: 15 iterations of render -> L1 + SSIM loss ->
    backward -> Eq. 11 -> Adam lower the loss against the targets of a
    perturbed copy (sanity, not parity)."""
    from paper_2312_10070_b200 import Rasterizer
    from paper_2312_10070_b200.pipeline import MapStep
    s = inputs.config1()
    rng = np.random.default_rng(0)
    P = Params.from_numpy(*s.params(), device=DEV)
    views = torch.as_tensor(s.views, device=DEV)
    r = Rasterizer(s.n, s.cam, device=DEV)
    r.size_for(P, views[0])
    r.forward(P, views[0])
    tc, td = {0: r.frame.color.clone()}, {0: r.frame.depth.clone()}
    noisy = [a.copy() for a in s.params()]
    noisy[3][:, :3] = np.clip(noisy[3][:, :3] + rng.normal(0, 0.1, noisy[3][:, :3].shape), 0, 1)  # colours
    Pn = Params.from_numpy(*noisy, device=DEV)
    ms = MapStep(Pn, views, s.cam, tc, td, device=DEV, lanes=1, ssim=0.2)
    ms.size()
    opt = Optimizer(s.n, DEV, lr_rgb=1e-2)
    losses = []
    for _ in range(15):
        g = ms.step()
        opt.regularize(Pn, g, 1.0)
        opt.step(Pn, g)
        losses.append(float(ms.losses[0, 0].item()))
    assert losses[-1] < 0.8 * losses[0], losses
