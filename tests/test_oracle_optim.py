"""Pins of the mapping-epilogue oracle (NEXT(3): Eq. 11, Adam, pruning) against
closed forms, worked examples of the spec and finite differences (CPU)."""
import numpy as np

from oracle import optim as O

LR = dict(lr_mean=1e-4, lr_quat=1e-3, lr_logscale=1e-3, lr_opacity=5e-2, lr_rgb=2.5e-3)


def test_iso_reg_worked_example_and_invariants():
    # one Gaussian with scales (2, 1, 1): s^bar = 4/3, L = 4/3
    L, _ = O.iso_reg(np.log([[2.0, 1.0, 1.0]]))
    assert abs(L - 4.0 / 3.0) < 1e-14
    # isotropic Gaussians -> 0, zero gradient
    L, g = O.iso_reg(np.log(np.full((5, 3), 0.7)))
    assert L < 1e-15 and np.abs(g).max() < 1e-15  # up to the rounding of the mean
    # replicating the sub-map leaves the mean-normalised loss unchanged
    l = np.random.default_rng(0).normal(-3, 0.5, (7, 3))
    assert abs(O.iso_reg(l)[0] - O.iso_reg(np.concatenate([l, l, l]))[0]) < 1e-15


def test_iso_reg_gradient_finite_differences():
    l = np.random.default_rng(1).normal(-3, 0.5, (9, 3))
    L, g = O.iso_reg(l)
    h = 1e-7
    for i in range(9):
        for j in range(3):
            e = np.zeros_like(l)
            e[i, j] = h
            fd = (O.iso_reg(l + e)[0] - O.iso_reg(l - e)[0]) / (2 * h)
            assert abs(fd - g[i, j]) <= 1e-7 * max(1.0, abs(fd))


def _state(n, seed):
    rng = np.random.default_rng(seed)
    p = {k: rng.normal(size=(n, 4)) for k in O.NAMES}
    p["quat"] /= np.linalg.norm(p["quat"], axis=1, keepdims=True)
    g = {k: rng.normal(size=(n, 4)) for k in O.NAMES}
    z = {k: np.zeros((n, 4)) for k in O.NAMES}
    return p, g, z


def test_adam_first_step_closed_form():
    """g = 1, lr = 0.1: the first bias-corrected step moves by -0.1
    (m^ = g, v^ = g^2, up to eps)."""
    p, _, z = _state(3, 0)
    g = {k: np.ones((3, 4)) for k in O.NAMES}
    lr = {k: 0.1 for k in LR}
    p2, m, v, ns = O.adam_step(p, g, z, z, 1, lr)
    d = p2["mean_opa"] - p["mean_opa"]
    assert np.allclose(d, -0.1 / (1 + 1e-8), rtol=1e-12) and ns == 0
    assert np.allclose(p2["logscale"][:, 3], p["logscale"][:, 3])  # unused component: rate 0
    assert np.allclose(np.linalg.norm(p2["quat"], axis=1), 1.0)     # renormalised


def test_adam_zero_gradient_and_nonfinite_skip():
    p, g, z = _state(4, 1)
    zero = {k: np.zeros((4, 4)) for k in O.NAMES}
    p2, m, v, ns = O.adam_step(p, zero, z, z, 1, LR)
    for k in O.NAMES:
        assert np.allclose(p2[k], p[k] if k != "quat" else p[k] / np.linalg.norm(p[k], axis=1, keepdims=True))
    g["rgb"][2, 1] = np.nan
    p3, m3, v3, ns = O.adam_step(p, g, z, z, 1, LR)
    assert ns == 1
    for k in O.NAMES:
        assert np.array_equal(p3[k][2], p[k][2]) and not m3[k][2].any()


def test_adam_converges_on_a_quadratic():
    """on a convex quadratic the iterates reach the optimum."""
    rng = np.random.default_rng(2)
    target = rng.normal(size=(1, 4))
    p = {k: np.zeros((1, 4)) for k in O.NAMES}
    p["quat"][0, 0] = 1.0
    z = {k: np.zeros((1, 4)) for k in O.NAMES}
    m, v = z, z
    lr = {k: 1e-2 for k in LR}
    for t in range(1, 3001):
        g = {k: np.zeros((1, 4)) for k in O.NAMES}
        g["mean_opa"] = 2 * (p["mean_opa"] - target)
        p, m, v, _ = O.adam_step(p, g, m, v, t, lr)
    assert np.abs(p["mean_opa"] - target).max() < 1e-3


def test_prune_rule():
    """logit(0.01) with o_thre = 0.1 is removed; 0.5 (the initial
    opacity) is kept; the order of the kept Gaussians is preserved."""
    logit = np.log(np.array([0.01, 0.5, 0.2, 0.05, 0.9]) / (1 - np.array([0.01, 0.5, 0.2, 0.05, 0.9])))
    keep = O.prune_keep(logit, 0.1)
    assert keep.tolist() == [False, True, True, False, True]
