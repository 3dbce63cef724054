"""Pins of the SSIM colour-loss oracle (Eq. 10; R32)
against library routines, closed forms and finite differences (CPU)."""
import numpy as np
from scipy import ndimage

from oracle import ssim as S


def _imgs(seed, H=13, W=17):
    rng = np.random.default_rng(seed)
    return rng.uniform(0, 1, (3, H, W)), rng.uniform(0, 1, (3, H, W))


def test_window_is_the_normalised_gaussian():
    g = S.window1d()
    assert g.shape == (11,) and abs(g.sum() - 1) < 1e-15
    assert np.allclose(g / g[5], np.exp(-np.arange(-5, 6) ** 2 / (2 * 1.5 ** 2)), rtol=1e-14)


def test_blur_matches_scipy_gaussian_filter():
    """Zero-padded 'same' correlation = scipy.ndimage.gaussian_filter(mode='constant')
    with the window truncated at 5 px = (5 / 1.5) sigma."""
    x = np.random.default_rng(0).uniform(size=(19, 23))
    ref = ndimage.gaussian_filter(x, 1.5, mode="constant", cval=0.0, truncate=5 / 1.5)
    assert np.allclose(S.blur(x), ref, rtol=0, atol=1e-14)
    w = np.outer(S.window1d(), S.window1d())
    assert np.allclose(S.blur(x), ndimage.correlate(x, w, mode="constant", cval=0.0), atol=1e-14)


def test_identical_images_ssim_one():
    x, _ = _imgs(1)
    assert abs(S.ssim(x, x) - 1.0) < 1e-14
    loss, l1, s, g = S.color_loss(x, x)
    assert loss == 0.0 or abs(loss) < 1e-15
    assert np.abs(g).max() < 1e-12  # stationary point (sign(0) = 0 for L1)


def test_constant_images_interior_closed_form():
    """Away from the zero padding, constant a vs b has zero variances and
    SSIM = (2ab + C1) / (a^2 + b^2 + C1)."""
    H = W = 31
    a, b = 0.3, 0.8
    x, y = np.full((H, W), a), np.full((H, W), b)
    Smap = S.ssim_terms(x, y)[0]
    want = (2 * a * b + S.C1) / (a * a + b * b + S.C1)
    assert np.allclose(Smap[5:-5, 5:-5], want, rtol=1e-12)
    # constant 0 vs 1: L1 term = 0.8 * 1
    loss, l1, s, _ = S.color_loss(np.zeros((3, H, W)), np.ones((3, H, W)))
    assert l1 == 1.0 and abs(loss - (0.8 + 0.2 * (1 - s))) < 1e-15


def test_ssim_brute_force_pixel():
    """One pixel of the SSIM map from its windowed sums written out."""
    x, y = _imgs(2)
    c, i, j = 1, 6, 8
    g = S.window1d()
    m = {k: 0.0 for k in ("x", "y", "xx", "yy", "xy")}
    for dy in range(-5, 6):
        for dx in range(-5, 6):
            ii, jj = i + dy, j + dx
            if 0 <= ii < x.shape[1] and 0 <= jj < x.shape[2]:
                w = g[dy + 5] * g[dx + 5]
                a, b = x[c, ii, jj], y[c, ii, jj]
                m["x"] += w * a
                m["y"] += w * b
                m["xx"] += w * a * a
                m["yy"] += w * b * b
                m["xy"] += w * a * b
    vx, vy, cxy = m["xx"] - m["x"] ** 2, m["yy"] - m["y"] ** 2, m["xy"] - m["x"] * m["y"]
    want = ((2 * m["x"] * m["y"] + S.C1) * (2 * cxy + S.C2)) / ((m["x"] ** 2 + m["y"] ** 2 + S.C1) * (vx + vy + S.C2))
    assert abs(S.ssim_terms(x[c], y[c])[0][i, j] - want) < 1e-14


def test_ssim_gradient_finite_differences():
    x, y = _imgs(3, 12, 14)
    g = S.ssim_grad(x, y)
    h = 1e-6
    rng = np.random.default_rng(1)
    for _ in range(30):
        c, i, j = rng.integers(3), rng.integers(12), rng.integers(14)
        e = np.zeros_like(x)
        e[c, i, j] = h
        fd = (S.ssim(x + e, y) - S.ssim(x - e, y)) / (2 * h)
        assert abs(fd - g[c, i, j]) <= 1e-7 * max(1.0, abs(fd)) + 1e-10


def test_color_loss_gradient_finite_differences():
    x, y = _imgs(4, 10, 11)
    _, _, _, g = S.color_loss(x, y, 0.2)
    h = 1e-7
    rng = np.random.default_rng(2)
    for _ in range(30):
        c, i, j = rng.integers(3), rng.integers(10), rng.integers(11)
        e = np.zeros_like(x)
        e[c, i, j] = h
        fd = (S.color_loss(x + e, y)[0] - S.color_loss(x - e, y)[0]) / (2 * h)
        assert abs(fd - g[c, i, j]) <= 1e-6 * max(1e-3, abs(fd))


def test_ssim_gradient_magnitude_scale_bounds():
    """R23 magnitude scale of the SSIM gradient (ssim_grad_mag): an upper
    bound of |ssim_grad| elementwise and of sum_p |dSSIM_p / dx_q| / 3HW (the
    per-output-pixel contributions, by central finite differences of the
    SSIM map, not the oracle's chain), and not merely |ssim_grad|."""
    x, y = _imgs(11, 9, 10)
    g = S.ssim_grad(x, y)
    m = S.ssim_grad_mag(x, y)
    assert (m >= np.abs(g) * (1 - 1e-12)).all()
    assert (m > np.abs(g) * 1.01).any()
    C, H, W = x.shape
    h = 1e-6
    rs = np.random.default_rng(3)
    for _ in range(12):
        c, i, j = rs.integers(C), rs.integers(H), rs.integers(W)
        xp, xm = x.copy(), x.copy()
        xp[c, i, j] += h
        xm[c, i, j] -= h
        Sp = S.ssim_terms(xp[c], y[c])[0]
        Sm = S.ssim_terms(xm[c], y[c])[0]
        contrib = np.abs((Sp - Sm) / (2 * h)).sum() / (C * H * W)
        assert contrib <= m[c, i, j] * (1 + 1e-6) + 1e-12
        assert np.isclose(((Sp - Sm) / (2 * h)).sum() / (C * H * W), g[c, i, j], rtol=1e-5, atol=1e-12)
