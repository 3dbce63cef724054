"""Pins of the seeding oracle (NEXT(4); DESIGN.md
R37-R41): the sampling permutation, the alpha gate, the back-projection, the
rho rejection and the nearest-neighbour scales, by closed forms and brute
force (CPU)."""
import numpy as np

from oracle import seed as S
from paper_2312_10070_b200 import inputs


def test_permutation_is_a_seeded_bijection():
    for n in (1, 2, 7, 1000, 4096, 30000):
        p = S.permutation(n, 3)
        assert np.array_equal(np.sort(p), np.arange(n))
    a, b = S.permutation(5000, 1), S.permutation(5000, 2)
    assert not np.array_equal(a, b) and np.array_equal(a, S.permutation(5000, 1))
    # roughly uniform: the first 10% of the order covers the image evenly
    first = S.permutation(10000, 7)[:1000]
    assert abs(np.mean(first < 5000) - 0.5) < 0.06


def _frame(H=24, W=32, seed=0, z=2.0):
    rng = np.random.default_rng(seed)
    color = rng.uniform(0, 1, (3, H, W)).astype(np.float32)
    depth = (z + rng.uniform(-0.5, 0.5, (H, W))).astype(np.float32)
    alpha = rng.uniform(0, 1, (H, W)).astype(np.float32)
    return color, depth, alpha


def _cam(H=24, W=32):
    return inputs.Camera(W, H, 30.0, 30.0, (W - 1) / 2, (H - 1) / 2)


I12 = np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0], np.float32)


def test_alpha_gate_and_valid_depth():
    color, depth, alpha = _frame()
    alpha[:] = 1.0  # fully covered frame: nothing to add
    r = S.seed(color, depth, alpha, I12, _cam(), np.zeros((0, 4)))
    assert len(r["idx"]) == 0 and r["mean_opa"].shape == (0, 4)
    color, depth, alpha = _frame()
    depth[:, :16] = 0.0  # invalid depth never seeds
    r = S.seed(color, depth, alpha, I12, _cam(), np.zeros((0, 4)))
    assert (r["idx"] % 32 >= 16).all()
    assert (alpha.ravel()[r["idx"]] < 0.6).all()
    assert len(r["idx"]) == int(((depth > 0) & (alpha < 0.6)).sum())


def test_backprojection_closed_form():
    H, W = 24, 32
    color, depth, alpha = _frame(H, W)
    alpha[:] = 0.0
    cam = _cam(H, W)
    # a pose with rotation about z by 90 degrees and a translation
    v = np.array([0, -1, 0, 1, 0, 0, 0, 0, 1, 0.1, 0.2, 0.3], np.float32)
    r = S.seed(color, depth, alpha, v, cam, np.zeros((0, 4)), max_new=50)
    R, t = v[:9].reshape(3, 3).astype(np.float64), v[9:].astype(np.float64)
    for k, p in enumerate(r["idx"]):
        i, j = p % W, p // W
        D = float(depth.ravel()[p])
        pc = np.array([(i - cam.cx) * D / cam.fx, (j - cam.cy) * D / cam.fy, D])
        assert np.allclose(r["points"][k], np.linalg.solve(R, pc - t), rtol=0, atol=1e-6)


def test_accepted_points_are_rho_apart_and_off_the_submap():
    """every accepted point is >= rho from every other accepted point
    and from every existing mean (brute force)."""
    H, W = 40, 48
    color, depth, alpha = _frame(H, W, 1)
    depth[:] = 2.0  # a fronto-parallel wall: neighbouring pixels ~7 cm apart at f = 30
    alpha[:] = 0.0
    cam = inputs.Camera(W, H, 300.0, 300.0, (W - 1) / 2, (H - 1) / 2)  # ~7 mm pixel pitch: rejections happen
    rng = np.random.default_rng(2)
    ex = np.concatenate([rng.uniform(-0.1, 0.1, (200, 2)), np.full((200, 1), 2.0), np.zeros((200, 1))], axis=1)
    r = S.seed(color, depth, alpha, I12, cam, ex.astype(np.float32), rho=0.01)
    A = r["mean_opa"][:, :3].astype(np.float64)
    assert 0 < len(A) < len(r["idx"])
    d = np.sqrt(((A[:, None] - A[None]) ** 2).sum(-1)) + np.eye(len(A))
    assert d.min() >= 0.01 - 1e-9
    de = np.sqrt(((A[:, None] - ex[None, :, :3]) ** 2).sum(-1))
    assert de.min() >= 0.01 - 1e-9


def test_new_gaussian_init():
    """P:624 / R41: opacity 0.5, identity rotation, isotropic NN-distance scale
    clamped to [rho / 2, 0.1 m], the pixel's colour."""
    H, W = 8, 8
    color, depth, alpha = _frame(H, W, 3)
    alpha[:] = 1.0
    alpha[2, 3] = 0.0  # a single candidate
    cam = _cam(H, W)
    r = S.seed(color, depth, alpha, I12, cam, np.zeros((0, 4)))
    assert len(r["mean_opa"]) == 1
    assert r["mean_opa"][0, 3] == 0.0 and np.array_equal(r["quat"][0], [1, 0, 0, 0])
    assert np.allclose(r["logscale"][0, :3], np.log(0.1))  # alone: clamped at 0.1 m
    assert np.array_equal(r["rgb"][0, :3], color[:, 2, 3])
    # an existing mean 3 cm away sets the scale
    p = r["mean_opa"][0, :3].astype(np.float64)
    ex = np.array([[p[0] + 0.03, p[1], p[2], 0.0]], np.float32)
    r2 = S.seed(color, depth, alpha, I12, cam, ex)
    assert abs(np.exp(r2["logscale"][0, 0]) - 0.03) < 1e-6


def test_sobel_step_edge_and_border():
    """A vertical step of height d in grey: gx = 4 d on the two columns next
    to the edge, gy = 0; the border is 0 (R43)."""
    H, W = 6, 8
    c = np.zeros((3, H, W), np.float32)
    c[:, :, 4:] = 0.5  # grey = 0.5 (0.299 + 0.587 + 0.114 = 1)
    m2 = S.gradient_m2(c)
    g = (0.299 * 0.5 + 0.587 * 0.5) + 0.114 * 0.5
    assert np.allclose(m2[1:-1, 3], (4 * g) ** 2) and np.allclose(m2[1:-1, 4], (4 * g) ** 2)
    assert (m2[1:-1, [1, 2, 5, 6]] == 0).all()
    assert (m2[0] == 0).all() and (m2[-1] == 0).all() and (m2[:, 0] == 0).all() and (m2[:, -1] == 0).all()
    # a horizontal ramp of slope s: gx = 8 s everywhere inside, gy = 0
    r = np.tile(np.arange(W, dtype=np.float32) * 0.01, (H, 1))
    m2 = S.gradient_m2(np.stack([r, r, r]))
    assert np.allclose(m2[1:-1, 1:-1], (8 * 0.01) ** 2, rtol=1e-9)


def test_grey_weights_and_sobel_brute_force():
    rng = np.random.default_rng(4)
    c = rng.uniform(0, 1, (3, 7, 9)).astype(np.float32)
    m2 = S.gradient_m2(c)
    g = c.astype(np.float64)
    grey = 0.299 * g[0] + 0.587 * g[1] + 0.114 * g[2]
    kx = np.array([[-1, 0, 1], [-2, 0, 2], [-1, 0, 1]], np.float64)
    for j in range(1, 6):
        for i in range(1, 8):
            win = grey[j - 1:j + 2, i - 1:i + 2]
            gx, gy = (win * kx).sum(), (win * kx.T).sum()
            assert abs(m2[j, i] - (gx * gx + gy * gy)) < 1e-12


def test_percentile_nearest_rank():
    v = np.arange(1, 101, dtype=np.float64)  # 1..100
    assert S.gradient_threshold(v, 0.95) == 95.0
    assert S.gradient_threshold(v, 0.951) == 96.0
    assert S.gradient_threshold(np.array([3.0]), 0.95) == 3.0
    m = np.zeros(100)
    m[:7] = 5.0  # ties: 93 zeros, 7 fives -> threshold 5, nothing strictly above
    assert S.gradient_threshold(m, 0.95) == 5.0


def test_first_keyframe_batches():
    """Uniform batch, then the gradient batch against it: the gradient
    candidates all come from the high-gradient set, and the union stays
    rho-separated (R40, R43)."""
    H, W = 40, 48
    rng = np.random.default_rng(5)
    color = rng.uniform(0, 1, (3, H, W)).astype(np.float32)
    color[:, :, 24:] *= 0.2  # a strong edge
    depth = (2.0 + 0.1 * rng.uniform(size=(H, W))).astype(np.float32)
    cam = inputs.Camera(W, H, 300.0, 300.0, (W - 1) / 2, (H - 1) / 2)
    r1, r2 = S.first_keyframe(color, depth, I12, cam, M_u=200, M_c=60, seed_=3)
    mask = S.gradient_mask(color, depth)
    assert mask.sum() <= int(np.ceil(0.05 * H * W)) + 1 and mask.sum() > 0
    assert mask.ravel()[r2["idx"]].all()
    A = np.concatenate([r1["mean_opa"][:, :3], r2["mean_opa"][:, :3]]).astype(np.float64)
    d = np.sqrt(((A[:, None] - A[None]) ** 2).sum(-1)) + np.eye(len(A))
    assert d.min() >= 0.01 - 1e-9
