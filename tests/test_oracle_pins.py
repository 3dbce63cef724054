"""Pins of the fp64 oracle against what the paper and the mathematics fix.

Each test names the passage it pins (P:n = PAPER.md line, S:n = SPEC.md line)
and checks the oracle against something other than itself: closed forms,
invariants, library routines (scipy / numpy.linalg), brute force on tiny
inputs, and central finite differences.  CPU only.
"""
import numpy as np
import pytest
from scipy.linalg import expm
from scipy.spatial.transform import Rotation

from paper_2312_10070_b200 import inputs


def _cam(w, h, f, cx=None, cy=None, zn=0.2, zf=100.0):
    return inputs.Camera(w, h, f, f, (w - 1) / 2 if cx is None else cx,
                         (h - 1) / 2 if cy is None else cy, zn, zf)


def _params(means, logscales, logits, rgbs, quats=None):
    n = len(means)
    q = np.tile([1.0, 0, 0, 0], (n, 1)) if quats is None else np.asarray(quats, float)
    return dict(mean=np.ascontiguousarray(means, float), quat=np.ascontiguousarray(q),
                logscale=np.ascontiguousarray(logscales, float),
                logit=np.ascontiguousarray(logits, float), rgb=np.ascontiguousarray(rgbs, float))


IDV = inputs.identity_view().astype(np.float64)


# --------------------------------------------------------------------------
# Geometry: R(q) and Sigma = R S S^T R^T

def test_quat_to_rot_examples(orc):
    assert np.allclose(orc.quat_to_rot([1, 0, 0, 0]), np.eye(3), atol=0)
    R = orc.quat_to_rot([np.sqrt(0.5), 0, 0, np.sqrt(0.5)])
    assert np.allclose(R @ [1, 0, 0], [0, 1, 0], atol=1e-15)


def test_quat_to_rot_matches_scipy(orc):
    rng = np.random.default_rng(0)
    for _ in range(50):
        q = rng.standard_normal(4)
        q /= np.linalg.norm(q)
        ref = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()  # scipy: scalar-last
        R = orc.quat_to_rot(q)
        assert np.allclose(R, ref, atol=1e-14)
        assert np.allclose(R.T @ R, np.eye(3), atol=1e-14)
        assert abs(np.linalg.det(R) - 1) < 1e-14


def test_covariance_examples(orc):
    assert np.allclose(orc.covariance([1, 0, 0, 0], [0, 0, 0]), np.eye(3))
    assert np.allclose(orc.covariance([1, 0, 0, 0], [np.log(2), 0, 0]), np.diag([4, 1, 1]))
    qz = [np.sqrt(0.5), 0, 0, np.sqrt(0.5)]
    assert np.allclose(orc.covariance(qz, [np.log(2), 0, 0]), np.diag([1, 4, 1]), atol=1e-14)


def test_covariance_spectrum(orc):
    """Eigenvalues of Sigma are s^2 and its eigenvectors the columns of R(q)."""
    rng = np.random.default_rng(1)
    for _ in range(20):
        q = rng.standard_normal(4) * 3.0          # unnormalised input is legal (R18)
        ls = rng.normal(-1, 0.5, 3)
        S = orc.covariance(q, ls)
        ev = np.sort(np.linalg.eigvalsh(S))
        assert np.allclose(ev, np.sort(np.exp(2 * ls)), rtol=1e-12)
        assert np.allclose(S, S.T, atol=1e-15)


# --------------------------------------------------------------------------
# Projection (Eqs. 1-2)

def test_projection_on_axis(orc):
    """on-axis point -> (cx, cy); identity Sigma at z=1 -> diag(fx^2, fy^2) + 0.3."""
    cam = inputs.Camera(128, 128, 100.0, 100.0, 64.0, 64.0)
    p = _params([[0, 0, 1.0]], [[0, 0, 0]], [0.0], [[1, 1, 1]])
    pr = orc.project(p, IDV, cam)
    assert pr["culled"][0] == 0
    assert np.array_equal(pr["uv"][0], [64.0, 64.0])
    assert pr["pz"][0] == 1.0
    d = np.float64(np.float32(0.3))
    assert np.allclose(pr["cov2d"][0], [1e4 + d, 0.0, 1e4 + d], rtol=1e-15)
    assert pr["opac"][0] == 0.5


def test_projection_near_far_cull(orc):
    """z = z_near/2 is culled; R5 keeps z_near <= z <= z_far (the camera is
    fp32 in the C-ABI, so the boundary is fp32(0.2))."""
    cam = _cam(64, 64, 60.0)
    zn = float(np.float32(0.2))
    p = _params([[0, 0, 0.1], [0, 0, 150.0], [0, 0, zn], [0, 0, 100.0], [0, 0, -1.0]],
                [[-3, -3, -3]] * 5, [0.0] * 5, [[1, 1, 1]] * 5)
    pr = orc.project(p, IDV, cam)
    assert list(pr["culled"]) == [1, 1, 0, 0, 1]
    assert np.isinf(pr["depth_key"][0]) and pr["depth_key"][2] == np.float32(0.2)


def _pinhole(p, cam):
    return np.array([cam.fx * p[0] / p[2] + cam.cx, cam.fy * p[1] / p[2] + cam.cy])


def test_projection_matches_numeric_jacobian(orc):
    """Eq. 2: Sigma^I - 0.3 I = J R Sigma R^T J^T with J the Jacobian of the
    pinhole map (central differences here, not the oracle's closed form), and
    conic = inverse(Sigma^I), and the alpha >= 1/255 box half-widths against the
    extreme points of the ellipse sampled on its boundary (R8')."""
    rng = np.random.default_rng(2)
    cam = _cam(320, 240, 300.0)
    n = 40
    R = Rotation.from_rotvec(rng.normal(0, 0.3, 3)).as_matrix()
    t = rng.normal(0, 0.2, 3)
    view = np.concatenate([R.reshape(9), t])
    pc = np.stack([rng.uniform(-1, 1, n), rng.uniform(-0.8, 0.8, n), rng.uniform(1.5, 5, n)], 1)
    mu = (pc - t) @ R          # world points whose camera coordinates are pc
    q = rng.standard_normal((n, 4))
    ls = rng.normal(-2.5, 0.4, (n, 3))
    p = _params(mu, ls, rng.normal(0, 1, n), rng.uniform(0, 1, (n, 3)), q)
    pr = orc.project(p, view, cam)
    d = np.float64(np.float32(0.3))
    for i in range(n):
        pcam = R @ mu[i] + t
        assert np.allclose(pr["uv"][i], _pinhole(pcam, cam), rtol=1e-13)
        h = 1e-6
        Jn = np.stack([(_pinhole(pcam + h * e, cam) - _pinhole(pcam - h * e, cam)) / (2 * h)
                       for e in np.eye(3)], 1)
        qq = q[i] / np.linalg.norm(q[i])
        Rq = Rotation.from_quat([qq[1], qq[2], qq[3], qq[0]]).as_matrix()
        Sig = Rq @ np.diag(np.exp(2 * ls[i])) @ Rq.T
        S2 = Jn @ R @ Sig @ R.T @ Jn.T + d * np.eye(2)
        a, b, c = pr["cov2d"][i]
        assert np.allclose([a, b, c], [S2[0, 0], S2[0, 1], S2[1, 1]], rtol=1e-6, atol=1e-9)
        if pr["culled"][i] == 0:
            Ci = np.linalg.inv(np.array([[a, b], [b, c]]))
            assert np.allclose(pr["conic"][i], [Ci[0, 0], Ci[0, 1], Ci[1, 1]], rtol=1e-12)
            # boundary of {Delta : Delta^T conic Delta = 2 tau}, tau = ln(o / alpha_min)
            tau = np.log(pr["opac"][i] / np.float64(np.float32(1 / 255)))
            L = np.linalg.cholesky(np.array([[a, b], [b, c]]))
            th = np.linspace(0, 2 * np.pi, 20001)
            pts = np.sqrt(2 * tau) * (L @ np.stack([np.cos(th), np.sin(th)]))
            assert np.allclose(pr["hxy"][i], np.abs(pts).max(1), rtol=1e-6)


def test_rect_brute_force(orc):
    """R8'/R9: the rect is exactly the set of tiles whose pixel square meets the
    box [u-hx, u+hx] x [v-hy, v+hy] (brute force over all tiles)."""
    s = inputs.random_scene(7, 300, 100, 70, spread=1.6, ls=(-2.0, 0.6))
    p = s.params64()
    pr = orc.project(p, s.views[0], s.cam)
    TX, TY = (s.cam.width + 15) // 16, (s.cam.height + 15) // 16
    for i in range(s.n):
        if pr["culled"][i] in (1, 2):
            continue
        u, v = pr["uv"][i]
        hx, hy = pr["hxy"][i]
        hit = [(tx, ty) for ty in range(TY) for tx in range(TX)
               if 16 * tx <= u + hx and u - hx < 16 * (tx + 1) and 16 * ty <= v + hy and v - hy < 16 * (ty + 1)]
        if pr["culled"][i] == 3:
            assert hit == [] or hx == 0.0
            continue
        x0, y0, x1, y1 = pr["rect"][i]
        exp = [(tx, ty) for ty in range(y0, y1 + 1) for tx in range(x0, x1 + 1)]
        assert sorted(hit) == sorted(exp)


def test_rect_covers_every_pixel_with_alpha_over_threshold(orc):
    """Eq. 4 + R8': wherever alpha~ = o exp(-sigma) >= 1/255, the pixel's tile is
    in the Gaussian's rect (brute force over every pixel; opaque Gaussians reach
    ~3.33 sigma, beyond a 3-sigma square)."""
    s = inputs.random_scene(8, 120, 96, 80, spread=1.2, ls=(-2.2, 0.6), lo=(2.0, 2.0))
    p = s.params64()
    pr = orc.project(p, s.views[0], s.cam)
    ys, xs = np.mgrid[0:80, 0:96]
    amin = np.float64(np.float32(1 / 255))
    for i in np.nonzero(pr["culled"] == 0)[0]:
        A, B, C = pr["conic"][i]
        dx, dy = pr["uv"][i, 0] - xs, pr["uv"][i, 1] - ys
        al = pr["opac"][i] * np.exp(-0.5 * (A * dx * dx + 2 * B * dx * dy + C * dy * dy))
        tx, ty = xs[al >= amin] // 16, ys[al >= amin] // 16
        x0, y0, x1, y1 = pr["rect"][i]
        assert ((tx >= x0) & (tx <= x1) & (ty >= y0) & (ty <= y1)).all()


# --------------------------------------------------------------------------
# Binning (R10)

def test_bin_sort_brute_force(orc):
    s = inputs.random_scene(3, 400, 96, 64, spread=1.3)
    p = s.params64()
    # force exact fp32 depth ties: duplicate some Gaussians
    for k in range(0, 40, 2):
        for key in p:
            p[key][k + 1] = p[key][k]
    pr = orc.project(p, s.views[0], s.cam)
    idx, rng = orc.bin_sort(pr["rect"], pr["culled"], pr["depth_key"], s.cam)
    TX = (s.cam.width + 15) // 16
    T = TX * ((s.cam.height + 15) // 16)
    assert rng.shape == (T, 2)
    start = 0
    for t in range(T):
        tx, ty = t % TX, t // TX
        mem = [i for i in range(s.n) if pr["culled"][i] == 0
               and pr["rect"][i, 0] <= tx <= pr["rect"][i, 2] and pr["rect"][i, 1] <= ty <= pr["rect"][i, 3]]
        mem = np.array(mem, dtype=np.int64)
        order = mem[np.lexsort((mem, pr["depth_key"][mem]))] if len(mem) else mem
        assert rng[t, 0] == start and rng[t, 1] == start + len(mem)
        assert np.array_equal(idx[rng[t, 0]:rng[t, 1]], order)
        start += len(mem)


# --------------------------------------------------------------------------
# Forward compositing (Eqs. 3, 4, 6)

def _iso_at_pixel(cam, i, j, z, s_px):
    """Isotropic Gaussian whose mean projects onto pixel (i, j) at depth z,
    with screen-space std s_px before dilation."""
    x = (i - cam.cx) * z / cam.fx
    y = (j - cam.cy) * z / cam.fy
    return [x, y, z], [np.log(s_px * z / cam.fx)] * 3


def test_render_empty(orc):
    cam = _cam(40, 24, 30.0)
    p = _params(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros(0), np.zeros((0, 3)))
    fr = orc.forward(p, IDV, cam)
    assert not fr["color"].any() and not fr["depth"].any() and not fr["alpha"].any()
    assert (fr["T_final"] == 1).all() and not fr["n_contrib"].any()


def test_render_single_centered(orc):
    """North-star closed form: one isotropic Gaussian centred on pixel (i, j)
    gives alpha = min(o, 0.999), C = alpha c, D = alpha z, A = alpha (R24)."""
    cam = _cam(64, 48, 60.0, cx=32.0, cy=24.0)
    for o in (0.3, 0.9, 0.9995):
        m, ls = _iso_at_pixel(cam, 20, 17, 2.0, 1.5)
        logit = np.log(o / (1 - o))
        p = _params([m], [ls], [logit], [[0.2, 0.5, 0.9]])
        fr = orc.forward(p, IDV, cam)
        a = min(o, np.float32(0.999))
        assert np.allclose(fr["color"][:, 17, 20], a * np.array([0.2, 0.5, 0.9]), rtol=1e-12)
        assert np.isclose(fr["depth"][17, 20], a * 2.0, rtol=1e-12)
        assert np.isclose(fr["alpha"][17, 20], a, rtol=1e-12)
        assert fr["n_contrib"][17, 20] == 1


def test_render_two_splats_spec_example(orc):
    """two pixel-centred splats at depths 1 m and 2 m with alpha = 0.5
    -> D = 0.5*1 + 0.5*0.5*2 = 1.0, A = 0.75; C = c1 a1 + c2 a2 (1 - a1)."""
    cam = _cam(64, 48, 60.0, cx=32.0, cy=24.0)
    m1, l1 = _iso_at_pixel(cam, 10, 10, 1.0, 1.0)
    m2, l2 = _iso_at_pixel(cam, 10, 10, 2.0, 1.0)
    p = _params([m2, m1], [l2, l1], [0.0, 0.0], [[0, 1, 0], [1, 0, 0]])  # far one first in the input
    fr = orc.forward(p, IDV, cam)
    assert np.isclose(fr["depth"][10, 10], 1.0, rtol=1e-12)
    assert np.isclose(fr["alpha"][10, 10], 0.75, rtol=1e-12)
    assert np.allclose(fr["color"][:, 10, 10], [0.5, 0.25, 0.0], rtol=1e-12)


def test_render_eq4_unit_conic(orc):
    """Delta = (1, 0), Sigma^I = I, o = 1 -> alpha = exp(-1/2) (here o
    is held below the clamp: alpha = o exp(-1/2))."""
    cam = _cam(64, 48, 60.0, cx=32.0, cy=24.0)
    d = float(np.float32(0.3))
    m, ls = _iso_at_pixel(cam, 32, 24, 2.0, np.sqrt(1 - d))   # on axis -> J S J^T = (1-d) I
    o = 0.8
    p = _params([m], [ls], [np.log(o / (1 - o))], [[1, 1, 1]])
    fr = orc.forward(p, IDV, cam)
    assert np.allclose(fr["proj"]["cov2d"][0], [1, 0, 1], atol=1e-12)
    assert np.isclose(fr["alpha"][24, 33], o * np.exp(-0.5), rtol=1e-12)
    assert np.isclose(fr["alpha"][23, 32], o * np.exp(-0.5), rtol=1e-12)


def test_render_stop_and_skip_rules(orc):
    """R11: alpha < 1/255 is skipped; compositing stops after the entry that
    leaves T < 1e-4 (include, then stop).  R8': a Gaussian whose alpha never
    reaches 1/255 (o < 1/255) is in no tile list."""
    cam = _cam(32, 32, 30.0)
    ms, lss = [], []
    for z, (i, j) in zip((1.0, 1.5, 2.0, 2.5), ((15, 8), (8, 8), (8, 8), (8, 8))):
        m, ls = _iso_at_pixel(cam, i, j, z, 2.0)
        ms.append(m)
        lss.append(ls)
    m, ls = _iso_at_pixel(cam, 8, 8, 0.5, 2.0)  # o = 1/300 < 1/255: culled
    ms.append(m)
    lss.append(ls)
    o_hi = 0.99995
    lo = np.log(o_hi / (1 - o_hi))
    faint = 1.0 / 300.0
    p = _params(ms, lss, [0.0, lo, lo, lo, np.log(faint / (1 - faint))],
                [[1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 1, 1], [1, 1, 1]])
    fr = orc.forward(p, IDV, cam)
    assert fr["proj"]["culled"][4] == 3
    # entry 0 (o = 0.5, 7 px away: alpha = 0.5 e^-5.7 < 1/255 but its box meets the
    # tile) is scanned and skipped; entries 1 and 2 composite (T = 1e-6 < 1e-4);
    # entry 3 is not reached
    assert fr["tile_range"][0, 1] - fr["tile_range"][0, 0] == 4
    assert fr["contrib"][8, 8] == 2 and fr["n_contrib"][8, 8] == 3 and fr["scanned"][8, 8] == 3
    a = np.float64(np.float32(0.999))
    assert np.isclose(fr["T_final"][8, 8], (1 - a) ** 2, rtol=1e-12)
    assert np.allclose(fr["color"][:, 8, 8], [0, a, a * (1 - a)], rtol=1e-12)


def test_render_invariants_random(orc):
    """Telescoping of Eq. 3: sum alpha_j T_j + T_final = 1; alpha in [0, 1];
    colour within [0, 1] for rgb in [0, 1]; bit-identical repeat."""
    for seed in range(20):
        s = inputs.random_scene(100 + seed, 150, 48, 40, spread=1.2, lo=(1.0, 1.5))
        p = s.params64()
        fr = orc.forward(p, s.views[0], s.cam)
        assert np.max(np.abs(fr["alpha"] + fr["T_final"] - 1)) < 1e-12
        assert fr["alpha"].min() >= 0 and fr["alpha"].max() <= 1
        assert fr["color"].min() >= 0 and fr["color"].max() <= 1 + 1e-12
        fr2 = orc.forward(p, s.views[0], s.cam)
        assert np.array_equal(fr["color"], fr2["color"]) and np.array_equal(fr["depth"], fr2["depth"])
        assert (fr["contrib"] <= fr["scanned"]).all()


def test_render_permutation_invariance(orc):
    """permuting the input leaves the frame bit-identical (distinct depths, R25)."""
    s = inputs.random_scene(5, 200, 48, 40, spread=1.2)
    p = s.params64()
    fr = orc.forward(p, s.views[0], s.cam)
    perm = np.random.default_rng(0).permutation(s.n)
    pp = {k: np.ascontiguousarray(v[perm]) for k, v in p.items()}
    fr2 = orc.forward(pp, s.views[0], s.cam)
    for key in ("color", "depth", "alpha", "T_final", "n_contrib"):
        assert np.array_equal(fr[key], fr2[key])


# --------------------------------------------------------------------------
# Loss (Eqs. 9-10, 12)

def test_loss_closed_forms(orc):
    cam = _cam(8, 6, 8.0)
    H, W = 6, 8
    rng = np.random.default_rng(0)
    c = rng.uniform(0, 1, (3, H, W))
    d = rng.uniform(1, 2, (H, W))
    L, gc, gd = orc.loss(cam, c, d, c, d)
    assert np.array_equal(L, [0, 0, 0]) and not gc.any() and not gd.any()
    L, _, gd = orc.loss(cam, c, d + 0.5, c, d)
    assert np.isclose(L[2], 0.5) and np.allclose(gd, 1.0 / (H * W))
    td = d.copy()
    td[: H // 2] = 0.0                                                           # invalid half
    dd = d + 1.0
    L, _, gd = orc.loss(cam, c, dd, c, td)
    assert np.isclose(L[2], 1.0) and not gd[: H // 2].any()
    L, gc, _ = orc.loss(cam, c + 0.25, d, c, d, lambda_color=2.0)
    assert np.isclose(L[1], 0.25) and np.isclose(L[0], 0.5) and np.allclose(gc, 2.0 / (3 * H * W))


def test_loss_gradient_fd(orc):
    cam = _cam(6, 5, 6.0)
    rng = np.random.default_rng(1)
    c, tc = rng.uniform(0, 1, (2, 3, 5, 6))
    d, td = rng.uniform(1, 2, (2, 5, 6))
    td[0, :3] = 0
    w = rng.uniform(0.5, 1.5, (5, 6))
    L, gc, gd = orc.loss(cam, c, d, tc, td, w, 0.7, 1.3)
    h = 1e-7
    for idx in [(0, 1, 2), (2, 4, 5), (1, 0, 0)]:
        e = np.zeros_like(c)
        e[idx] = h
        fd = (orc.loss(cam, c + e, d, tc, td, w, 0.7, 1.3)[0][0] - orc.loss(cam, c - e, d, tc, td, w, 0.7, 1.3)[0][0]) / (2 * h)
        assert np.isclose(fd, gc[idx], rtol=1e-6)
    for idx in [(1, 2), (4, 5), (0, 4)]:
        e = np.zeros_like(d)
        e[idx] = h
        fd = (orc.loss(cam, c, d + e, tc, td, w, 0.7, 1.3)[0][0] - orc.loss(cam, c, d - e, tc, td, w, 0.7, 1.3)[0][0]) / (2 * h)
        assert np.isclose(fd, gd[idx], rtol=1e-6, atol=1e-12)


# --------------------------------------------------------------------------
# Backward (Eqs. 7-8) — central finite differences

def _objective(orc, p, view, cam, G):
    fr = orc.forward(p, view, cam)
    L = (G[0] * fr["color"]).sum() + (G[1] * fr["depth"]).sum() + (G[2] * fr["alpha"]).sum()
    return L, (fr["sig"].copy(), fr["n_contrib"].copy(), fr["proj"]["rect"].copy())


def _same(a, b):
    return all(np.array_equal(x, y) for x, y in zip(a, b))


def _fd_check(orc, s, h=1e-5, rtol=1e-4, seed=0):
    p = s.params64()
    cam, view = s.cam, s.views[0].astype(np.float64)
    rng = np.random.default_rng(seed)
    G = (rng.standard_normal((3, cam.height, cam.width)), rng.standard_normal((cam.height, cam.width)),
         rng.standard_normal((cam.height, cam.width)))
    fr = orc.forward(p, view, cam)
    b = orc.backward(p, view, cam, fr["sorted_idx"], fr["tile_range"], G[0], G[1], G[2])
    _, sig0 = _objective(orc, p, view, cam, G)
    fields = [("mean", 3, 0), ("logit", None, 3), ("quat", 4, 4), ("logscale", 3, 8), ("rgb", 3, 12)]
    checked = skipped = 0
    worst = 0.0
    scale = np.abs(b["g3"]).max()
    for i in range(s.n):
        for name, width, off in fields:
            for c in range(width or 1):
                pp = {k: v.copy() for k, v in p.items()}
                pm = {k: v.copy() for k, v in p.items()}
                if width is None:
                    pp[name][i] += h
                    pm[name][i] -= h
                else:
                    pp[name][i, c] += h
                    pm[name][i, c] -= h
                Lp, sp = _objective(orc, pp, view, cam, G)
                Lm, sm = _objective(orc, pm, view, cam, G)
                if not (_same(sp, sig0) and _same(sm, sig0)):
                    skipped += 1
                    continue
                fd = (Lp - Lm) / (2 * h)
                an = b["g3"][i, off + c]
                err = abs(fd - an) / (abs(an) + 1e-6 * scale)
                worst = max(worst, err)
                assert err < rtol, (i, name, c, fd, an)
                checked += 1
    return checked, skipped, worst, b


@pytest.mark.parametrize("seed", range(6))
def test_backward_fd_small_scenes(orc, seed):
    """every parameter gradient matches central finite
    differences (h = 1e-5, fp64) within relative error 1e-4 on random
    <=20-Gaussian 32x32 scenes; components whose decision signature changes
    between theta +- h are skipped and counted (H8)."""
    s = inputs.random_scene(seed, 12 + seed, 32, 32, spread=0.9, ls=(-2.2, 0.3), lo=(0.5, 1.0))
    checked, skipped, worst, _ = _fd_check(orc, s)
    assert checked > 0.9 * (checked + skipped)


def test_backward_fd_tiny_config(orc):
    """BJ.configs[0] geometry (64x48), first 24 Gaussians."""
    s = inputs.config0()
    for arr in ("mean_opa", "quat", "logscale", "rgb"):
        setattr(s, arr, getattr(s, arr)[:24].copy())
    checked, skipped, worst, _ = _fd_check(orc, s)
    assert checked > 0.9 * (checked + skipped)


def _twist_apply(view, xi):
    """T <- exp(xi^) T with scipy's matrix exponential (independent of the oracle)."""
    v, w = xi[:3], xi[3:]
    X = np.zeros((4, 4))
    X[:3, :3] = [[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]]
    X[:3, 3] = v
    T = np.eye(4)
    T[:3, :3] = view[:9].reshape(3, 3)
    T[:3, 3] = view[9:]
    T2 = expm(X) @ T
    return np.concatenate([T2[:3, :3].reshape(9), T2[:3, 3]])


def test_pose_gradient_fd_and_translation_identity(orc):
    """Eq. 14 gradient w.r.t. the 6-DoF pose: twist FD (scipy expm); and the
    identity dL/dt = R sum_g dL/dmu_g, since mu enters only through p = R mu + t."""
    s = inputs.random_scene(11, 15, 32, 32, spread=0.9, ls=(-2.2, 0.3), lo=(0.5, 1.0))
    p = s.params64()
    cam = s.cam
    R0 = Rotation.from_rotvec([0.05, -0.03, 0.02]).as_matrix()
    view = np.concatenate([R0.reshape(9), [0.02, -0.01, 0.05]])
    rng = np.random.default_rng(3)
    G = (rng.standard_normal((3, 32, 32)), rng.standard_normal((32, 32)), rng.standard_normal((32, 32)))
    fr = orc.forward(p, view, cam)
    b = orc.backward(p, view, cam, fr["sorted_idx"], fr["tile_range"], *G)
    gR, gt = b["pose"][:9], b["pose"][9:]
    assert np.allclose(gt, R0 @ b["g3"][:, 0:3].sum(0), rtol=1e-10, atol=1e-12)
    tw = orc.pose_twist(b["pose"], view)
    _, sig0 = _objective(orc, p, view, cam, G)
    h = 1e-6
    ok = 0
    for k in range(6):
        e = np.zeros(6)
        e[k] = h
        Lp, sp = _objective(orc, p, _twist_apply(view, e), cam, G)
        Lm, sm = _objective(orc, p, _twist_apply(view, -e), cam, G)
        if not (_same(sp, sig0) and _same(sm, sig0)):
            continue
        fd = (Lp - Lm) / (2 * h)
        assert abs(fd - tw[k]) <= 1e-4 * abs(tw[k]) + 1e-7 * np.abs(tw).max(), (k, fd, tw[k])
        ok += 1
    assert ok >= 5
    # (q, t) parameterisation: FD on the quaternion of R (scipy for q -> R)
    qs = Rotation.from_matrix(R0).as_quat()
    q = np.array([qs[3], qs[0], qs[1], qs[2]])
    gq = orc.pose_qt(b["pose"], q)
    for k in range(4):
        dq = np.zeros(4)
        dq[k] = h

        def L_of(qq):
            qq = qq / np.linalg.norm(qq)
            Rm = Rotation.from_quat([qq[1], qq[2], qq[3], qq[0]]).as_matrix()
            return _objective(orc, p, np.concatenate([Rm.reshape(9), view[9:]]), cam, G)[0]

        fd = (L_of(q + dq) - L_of(q - dq)) / (2 * h)
        assert abs(fd - gq[k]) <= 1e-4 * abs(gq[k]) + 1e-7 * np.abs(gq).max()


def test_backward_linearity_and_zero_gradients(orc):
    """linearity in the upstream maps; Gaussians that never
    composite (culled, or hidden behind an opaque splat) get exact zeros."""
    cam = _cam(32, 32, 30.0)
    m1, l1 = _iso_at_pixel(cam, 16, 16, 1.0, 30.0)
    m2, l2 = _iso_at_pixel(cam, 16, 16, 3.0, 1.0)
    m3 = [0, 0, 0.05]
    hi = np.log(0.99999 / 0.00001)
    p = _params([m1, m1, m1, m2, m3], [l1, l1, l1, l2, l2], [hi, hi, hi, 0.0, 0.0], [[1, 0, 0]] * 5)
    fr = orc.forward(p, IDV, cam)
    rng = np.random.default_rng(0)
    G1 = [rng.standard_normal(x) for x in ((3, 32, 32), (32, 32), (32, 32))]
    G2 = [rng.standard_normal(x) for x in ((3, 32, 32), (32, 32), (32, 32))]
    b1 = orc.backward(p, IDV, cam, fr["sorted_idx"], fr["tile_range"], *G1)
    b2 = orc.backward(p, IDV, cam, fr["sorted_idx"], fr["tile_range"], *G2)
    b12 = orc.backward(p, IDV, cam, fr["sorted_idx"], fr["tile_range"], *[2 * a - 3 * b for a, b in zip(G1, G2)])
    assert np.allclose(b12["g3"], 2 * b1["g3"] - 3 * b2["g3"], rtol=1e-10, atol=1e-10)
    # Gaussian 3 sits behind three near-opaque splats (T < 1e-4 before it) wherever
    # its alpha >= 1/255: exact zero; Gaussian 4 is culled (z < z_near)
    assert np.array_equal(b1["g3"][3], np.zeros(16))
    assert np.array_equal(b1["g3"][4], np.zeros(16))
    assert np.abs(b1["g3"][0]).sum() > 0


# --------------------------------------------------------------------------
# Pose utilities (R22) and the Adam step

def test_se3_exp_matches_expm(orc):
    rng = np.random.default_rng(4)
    for _ in range(10):
        xi = rng.normal(0, 0.5, 6)
        R, t = orc.se3_exp(xi)
        ref = _twist_apply(np.concatenate([np.eye(3).reshape(9), np.zeros(3)]), xi)
        assert np.allclose(R.reshape(9), ref[:9], atol=1e-12) and np.allclose(t, ref[9:], atol=1e-12)


def test_adam_first_step(orc):
    """bias-corrected first step moves by lr * sign(g)."""
    g = np.array([0.3, -2.0, 1e-3, 5.0, -0.1, 0.7])
    view, st = orc.pose_adam(IDV, g, np.zeros(13), lr=(2e-3, 1e-3))
    xi = -np.concatenate([2e-3 * np.sign(g[:3]), 1e-3 * np.sign(g[3:])]) * (1 / (1 + 1e-8 / np.abs(g)))
    ref = _twist_apply(IDV, xi)
    assert np.allclose(view, ref, atol=1e-12) and st[12] == 1


# --------------------------------------------------------------------------
# R23 magnitude scales m2, m3, mpose and the R2 decision margin: they set the
# slack of every GPU parity check, so they are pinned here against definitions
# computed independently of the oracle's backward.

G2_FIELDS = ("u", "v", "A", "B", "C", "logit", "r", "g", "b", "pz")


@pytest.mark.parametrize("seed", range(4))
def test_magnitude_scales_bound_the_gradients(orc, seed):
    """R23: m* >= |g*| componentwise (2-D, 3-D and pose) on random scenes
    (every inner sum of m* is a sum of absolute values of g*'s terms)."""
    s = inputs.random_scene(100 + seed, 30, 40, 32, spread=1.0, ls=(-2.2, 0.4), lo=(0.5, 1.0))
    p = s.params64()
    view = np.concatenate([Rotation.from_rotvec([0.04, -0.02, 0.03]).as_matrix().reshape(9), [0.01, 0.02, -0.03]])
    fr = orc.forward(p, view, s.cam)
    rng = np.random.default_rng(seed)
    G = (rng.standard_normal((3, 32, 40)), rng.standard_normal((32, 40)), rng.standard_normal((32, 40)))
    b = orc.backward(p, view, s.cam, fr["sorted_idx"], fr["tile_range"], *G)
    for g, m in (("g2", "m2"), ("g3", "m3"), ("pose", "mpose")):
        assert (b[m] >= np.abs(b[g]) * (1 - 1e-12)).all(), g
        assert (b[m] > np.abs(b[g]) * 1.01).any(), g  # and not merely |g*| (cancellation is counted)


def _one_gaussian(cam, z=2.0, dy_px=1.3, logit=1.2, ls=-2.0):
    """One isotropic Gaussian at camera x = 0 (so Sigma^I is diagonal: B = 0),
    dy_px pixels below the principal point."""
    return _params([[0.0, dy_px * z / cam.fy, z]], [[ls, ls, ls]], [logit], [[0.8, 0.5, 0.3]])


def test_magnitude_scale_equals_gradient_on_single_pixel(orc):
    """R23 on a 1-Gaussian, 1-pixel scene with same-sign upstream terms: every
    absolute-value sum of m2 has one term, so m2 == |g2| exactly (dx = 0 here:
    the u and A components vanish on both sides)."""
    cam = _cam(1, 1, 50.0, cx=0.0, cy=0.0)
    p = _one_gaussian(cam, dy_px=0.7)
    fr = orc.forward(p, IDV, cam)
    G = (np.full((3, 1, 1), 0.6), np.full((1, 1), 0.4), np.full((1, 1), 0.9))
    b = orc.backward(p, IDV, cam, fr["sorted_idx"], fr["tile_range"], *G)
    assert fr["n_contrib"][0, 0] == 1
    assert np.allclose(b["m2"], np.abs(b["g2"]), rtol=1e-13, atol=0)
    assert (np.abs(b["g2"][0, [1, 4, 5, 6, 7, 8, 9]]) > 0).all()


def test_magnitude_scale_is_sum_of_per_pixel_fd_gradients(orc):
    """R23's m2 = sum over pixels of |per-pixel contribution|: one Gaussian
    (B = 0, same-sign upstream and colours, so every inner sum is one-signed),
    each pixel's contribution to dL/d(u, v, A, B, C, logit, rgb, p_z) by central
    finite differences of that pixel's value through orc.render with the 2-D
    quantities perturbed directly (no backward code involved)."""
    cam = _cam(24, 20, 60.0)
    p = _one_gaussian(cam, dy_px=1.6, ls=-2.6)
    fr = orc.forward(p, IDV, cam)
    pr, idx, rng_ = fr["proj"], fr["sorted_idx"], fr["tile_range"]
    assert abs(pr["conic"][0, 1]) < 1e-18
    rgen = np.random.default_rng(9)
    G = (rgen.uniform(0.2, 1.0, (3, 20, 24)), rgen.uniform(0.2, 1.0, (20, 24)), rgen.uniform(0.2, 1.0, (20, 24)))
    b = orc.backward(p, IDV, cam, idx, rng_, *G)

    def per_px(prx, rgb):
        o = orc.render(prx, rgb, idx, rng_, cam)
        return (G[0] * o["color"]).sum(0) + G[1] * o["depth"] + G[2] * o["alpha"], o["sig"]

    base_sig = per_px(pr, p["rgb"])[1]
    h = 1e-6
    for j, name in enumerate(G2_FIELDS):
        vals = []
        for sgn in (1.0, -1.0):
            q = {k: v.copy() for k, v in pr.items()}
            rgb = p["rgb"].copy()
            if name in ("u", "v"):
                q["uv"][0, "uv".index(name)] += sgn * h
            elif name in ("A", "B", "C"):
                q["conic"][0, "ABC".index(name)] += sgn * h
            elif name == "logit":
                q["opac"][0] = 1.0 / (1.0 + np.exp(-(p["logit"][0] + sgn * h)))
            elif name in ("r", "g", "b"):
                rgb[0, "rgb".index(name)] += sgn * h
            else:
                q["pz"][0] += sgn * h
            L, sig = per_px(q, rgb)
            assert np.array_equal(sig, base_sig), name  # no decision flips at this h
            vals.append(L)
        contrib = (vals[0] - vals[1]) / (2 * h)
        # the oracle's conic B term enters sigma as 2 B dx dy: dL/dB there is the
        # coefficient of the symmetric off-diagonal, as g2 defines it
        assert np.isclose(b["g2"][0, j], contrib.sum(), rtol=1e-6, atol=1e-9), name
        assert np.isclose(b["m2"][0, j], np.abs(contrib).sum(), rtol=1e-6, atol=1e-9), name


def _x2d(orc, p, view, cam):
    """The 2-D quantities of every Gaussian (oracle projection): [n, 10] in g2 order."""
    pr = orc.project(p, view, cam)
    return np.concatenate([pr["uv"], pr["conic"], p["logit"][:, None], p["rgb"], pr["pz"][:, None]], 1)


def test_magnitude_scales_3d_and_pose_are_abs_jacobian_of_m2(orc):
    """R23: m3 = |d x2D / d theta|^T m2 per Gaussian and mpose = sum_g
    |d x2D_g / d(R, t)|^T m2_g, with the Jacobian of the 2-D quantities taken by
    central finite differences of orc.project (not the backward's chain)."""
    s = inputs.random_scene(77, 8, 40, 32, spread=0.8, ls=(-2.2, 0.3), lo=(0.5, 1.0))
    p = s.params64()
    view = np.concatenate([Rotation.from_rotvec([0.03, 0.05, -0.02]).as_matrix().reshape(9), [0.02, -0.01, 0.04]])
    fr = orc.forward(p, view, s.cam)
    rng = np.random.default_rng(5)
    G = (rng.standard_normal((3, 32, 40)), rng.standard_normal((32, 40)), rng.standard_normal((32, 40)))
    b = orc.backward(p, view, s.cam, fr["sorted_idx"], fr["tile_range"], *G)
    vis = fr["proj"]["culled"] == 0
    assert vis.sum() >= 6
    h = 1e-6
    fields = [("mean", 3, 0), ("logit", None, 3), ("quat", 4, 4), ("logscale", 3, 8), ("rgb", 3, 12)]
    m3 = np.zeros((s.n, 16))
    for name, width, off in fields:
        for c in range(width or 1):
            pp = {k: v.copy() for k, v in p.items()}
            pm = {k: v.copy() for k, v in p.items()}
            if width is None:
                pp[name] += h
                pm[name] -= h
            else:
                pp[name][:, c] += h
                pm[name][:, c] -= h
            J = (_x2d(orc, pp, view, s.cam) - _x2d(orc, pm, view, s.cam)) / (2 * h)  # [n, 10], per Gaussian
            m3[:, off + c] = (np.abs(J) * b["m2"]).sum(1)
    assert np.allclose(b["m3"][vis], m3[vis], rtol=2e-5, atol=1e-12 * np.abs(m3).max())
    assert (b["m3"][~vis] == 0).all()
    mpose = np.zeros(12)
    for k in range(12):
        vp, vm = view.copy(), view.copy()
        vp[k] += h
        vm[k] -= h
        J = (_x2d(orc, p, vp, s.cam) - _x2d(orc, p, vm, s.cam)) / (2 * h)
        mpose[k] = (np.abs(J[vis]) * b["m2"][vis]).sum()
    assert np.allclose(b["mpose"], mpose, rtol=2e-5)


def test_decision_margin_brute_force(orc):
    """R2: the per-pixel minimum relative decision margin, recomputed by a
    brute-force numpy walk over each pixel's tile list (alpha~ against 1/255
    and 0.999 at every scanned entry, T against 1e-4 after every composited
    entry, stopping where the pixel stops)."""
    s = inputs.random_scene(88, 18, 32, 32, spread=0.9, ls=(-2.0, 0.4), lo=(1.0, 1.5))
    p = s.params64()
    fr = orc.forward(p, IDV, s.cam)
    pr = fr["proj"]
    amin, amax, teps = (np.float64(np.float32(x)) for x in (1 / 255, 0.999, 1e-4))
    TX = (s.cam.width + 15) // 16
    ref = np.full((32, 32), np.inf)
    for j in range(32):
        for i in range(32):
            t = (j // 16) * TX + i // 16
            T, mg = 1.0, np.inf
            for k in range(*fr["tile_range"][t]):
                g = fr["sorted_idx"][k]
                dx, dy = pr["uv"][g, 0] - i, pr["uv"][g, 1] - j
                A, B, C = pr["conic"][g]
                at = pr["opac"][g] * np.exp(-0.5 * (A * dx * dx + 2 * B * dx * dy + C * dy * dy))
                mg = min(mg, abs(at - amin) / amin, abs(at - amax) / amax)
                a = min(at, amax)
                if a < amin:
                    continue
                T = T * (1 - a)
                mg = min(mg, abs(T - teps) / teps)
                if T < teps:
                    break
            ref[j, i] = mg
    assert np.allclose(fr["margin"], ref, rtol=1e-9, atol=0)
    assert np.isfinite(ref).mean() > 0.5 and (ref < 1e-2).any()
