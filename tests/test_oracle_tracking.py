"""Pins of the masked tracking-loss oracle (Eq. 15; DESIGN.md
R29-R31) against brute force, closed forms and finite differences (CPU)."""
import numpy as np

from oracle import tracking as T


def _maps(seed, H=9, W=13, invalid=0.1):
    rng = np.random.default_rng(seed)
    c = rng.uniform(0, 1, (3, H, W)).astype(np.float32)
    tc = rng.uniform(0, 1, (3, H, W)).astype(np.float32)
    d = rng.uniform(0.5, 4, (H, W)).astype(np.float32)
    td = rng.uniform(0.5, 4, (H, W)).astype(np.float32)
    td[rng.uniform(size=(H, W)) < invalid] = 0.0
    a = rng.uniform(0, 1, (H, W)).astype(np.float32)
    return c, d, a, tc, td


def test_lower_median_brute_force():
    rng = np.random.default_rng(0)
    for n in (1, 2, 3, 10, 11, 64, 257):
        x = rng.normal(size=n).astype(np.float32)
        s = sorted(x.tolist())
        assert T.lower_median(x) == np.float32(s[(n - 1) // 2])
        if n % 2:
            assert T.lower_median(x) == np.float32(np.median(x))
    assert T.lower_median(np.zeros(0)) is None


def test_error_maps_fp32_order():
    """e_c = ((|dr| + |dg|) + |db|) / 3 with fp32 rounding of every step, e_d = |D^ - D|."""
    c, d, a, tc, td = _maps(1)
    e_c, e_d, valid = T.error_maps32(c, d, tc, td)
    H, W = d.shape
    for i in range(H):
        for j in range(W):
            r = [abs(np.float32(c[k, i, j] - tc[k, i, j])) for k in range(3)]
            want = np.float32(np.float32(np.float32(r[0] + r[1]) + r[2]) / np.float32(3))
            assert e_c[i, j] == want
            assert e_d[i, j] == abs(np.float32(d[i, j] - td[i, j]))
            assert valid[i, j] == (td[i, j] > 0)


def test_brute_force_loss_all_inliers():
    """alpha = 1 and a huge multiplier: L = sum over valid pixels of
    lambda_c mean_c |dC| + (1 - lambda_c) |dD| (a plain loop)."""
    c, d, a, tc, td = _maps(2)
    lam = 0.7
    r = T.tracking_loss(c, d, np.ones_like(a), tc, td, lam, 1e30)
    H, W = d.shape
    want = 0.0
    for i in range(H):
        for j in range(W):
            if td[i, j] > 0:
                ec = sum(abs(float(c[k, i, j]) - float(tc[k, i, j])) for k in range(3)) / 3
                want += lam * ec + (1 - lam) * abs(float(d[i, j]) - float(td[i, j]))
    assert abs(r["loss"] - want) <= 1e-12 * abs(want)
    assert r["inlier"].sum() == (td > 0).sum()


def test_uniform_error_all_valid_are_inliers():
    """a uniform nonzero error equals its median, < 50 x median."""
    H, W = 6, 7
    c = np.full((3, H, W), 0.5, np.float32)
    tc = np.full((3, H, W), 0.25, np.float32)
    d = np.full((H, W), 2.0, np.float32)
    td = np.full((H, W), 1.5, np.float32)
    td[0, 0] = 0.0
    r = T.tracking_loss(c, d, np.ones((H, W), np.float32), tc, td)
    assert r["med_c"] == np.float32(0.25) and r["med_d"] == np.float32(0.5)
    assert r["inlier"].sum() == H * W - 1 and not r["inlier"][0, 0]


def test_outliers_rejected_by_frame_relative_threshold():
    """A depth (or colour) error > 50 x the median error is discarded."""
    c, d, a, tc, td = _maps(3, invalid=0.0)
    td[:] = d + np.float32(0.01)                      # uniform depth error 0.01
    tc[:] = c + np.float32(0.002)                     # uniform colour error 0.002
    d[2, 3] = td[2, 3] + np.float32(0.6)              # 60x the median depth error
    c[1, 4, 5] = tc[1, 4, 5] + np.float32(0.5)        # mean colour error ~0.17 > 50x median
    r = T.tracking_loss(c, d, a, tc, td)
    assert not r["inlier"][2, 3] and not r["inlier"][4, 5]
    assert r["inlier"].sum() == d.size - 2
    d[2, 3] = td[2, 3] + np.float32(0.4)              # 40x: kept
    assert T.tracking_loss(c, d, a, tc, td)["inlier"][2, 3]


def test_alpha_cube_weighting():
    """M_alpha = alpha^3 (R29): alpha = 1/2 everywhere scales L by 1/8."""
    c, d, a, tc, td = _maps(4)
    one = T.tracking_loss(c, d, np.ones_like(a), tc, td)["loss"]
    half = T.tracking_loss(c, d, np.full_like(a, 0.5), tc, td)["loss"]
    assert abs(half - one / 8) <= 1e-12 * one


def test_no_valid_pixel_gives_zero():
    c, d, a, tc, td = _maps(5)
    td[:] = 0.0
    r = T.tracking_loss(c, d, a, tc, td)
    assert r["loss"] == 0.0 and not r["inlier"].any()
    assert not r["g_color"].any() and not r["g_depth"].any()


def test_gradient_matches_finite_differences():
    """dL/dC^ and dL/dD^ with the masks held constant (R29), central FD in fp64."""
    c, d, a, tc, td = _maps(6)
    c, d, tc, td = (x.astype(np.float64) for x in (c, d, tc, td))
    lam = 0.4
    r = T.tracking_loss(c, d, a, tc, td, lam)
    inl, w = r["inlier"], r["inlier"] * r["m_alpha"]

    def L(cc, dd):  # the loss with the masks frozen
        ec = np.abs(cc - tc).mean(axis=0)
        return float(np.sum(w * (lam * ec + (1 - lam) * np.abs(dd - td))))

    h = 1e-6
    rng = np.random.default_rng(0)
    for _ in range(40):
        k, i, j = rng.integers(3), rng.integers(d.shape[0]), rng.integers(d.shape[1])
        e = np.zeros_like(c)
        e[k, i, j] = h
        fd = (L(c + e, d) - L(c - e, d)) / (2 * h)
        assert abs(fd - r["g_color"][k, i, j]) <= 1e-6 * max(1.0, abs(fd))
        e = np.zeros_like(d)
        e[i, j] = h
        fd = (L(c, d + e) - L(c, d - e)) / (2 * h)
        assert abs(fd - r["g_depth"][i, j]) <= 1e-6 * max(1.0, abs(fd))
    assert not r["g_depth"][~inl].any()
