"""Oracle of the SSIM colour loss (Eq. 10) — TEST INFRASTRUCTURE ONLY.

Plain numpy fp64, following the definitions step by step; shares nothing
with the CUDA path.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline / ``--impl reference`` leg may import it.

P:184-190 (Eq. 10):  L_color = (1 - lambda) |I^ - I|_1 + lambda (1 - SSIM(I^, I)),
lambda = 0.2; SSIM as in Wang et al. 2004 (P:185 cites [wang2004image]).
Readings:
  R32  SSIM window: 11 x 11 Gaussian, sigma = 1.5, normalised; K1 = 0.01,
       K2 = 0.03, dynamic range 1; local statistics by correlation
       with zero padding ("same" size; the usual splatting-loss form),
       SSIM(I^, I) = the mean of the SSIM map over the 3 channels and all
       pixels; |I^ - I|_1 = the mean absolute error over 3HW (as R20).
  R33  Eq. 12's colour term with SSIM: L = lambda_color L_color +
       lambda_depth L_depth; the depth term is unchanged (R20).
"""
from __future__ import annotations

import numpy as np

SIGMA, RADIUS = 1.5, 5
C1, C2 = 0.01 ** 2, 0.03 ** 2


def window1d():
    k = np.arange(-RADIUS, RADIUS + 1, dtype=np.float64)
    g = np.exp(-(k * k) / (2 * SIGMA * SIGMA))
    return g / g.sum()


def blur(img):
    """Correlation of a [H, W] map with the 11 x 11 window, zero padding, same size
    (the 2-D window written out: w(dy, dx) = g(dy) g(dx))."""
    g = window1d()
    H, W = img.shape
    p = np.pad(np.asarray(img, np.float64), RADIUS)
    out = np.zeros((H, W))
    for dy in range(2 * RADIUS + 1):
        for dx in range(2 * RADIUS + 1):
            out += g[dy] * g[dx] * p[dy:dy + H, dx:dx + W]
    return out


def ssim_terms(x, y):
    """Per-pixel SSIM map of one channel and the partial derivatives of the
    map w.r.t. its local statistics (Wang et al. 2004, Eq. 13)."""
    mx, my = blur(x), blur(y)
    sxx = blur(x * x) - mx * mx
    syy = blur(y * y) - my * my
    sxy = blur(x * y) - mx * my
    n1, n2 = 2 * mx * my + C1, 2 * sxy + C2
    d1, d2 = mx * mx + my * my + C1, sxx + syy + C2
    S = (n1 * n2) / (d1 * d2)
    D = d1 * d2
    dS_dmx = 2 * my * n2 / D - 2 * mx * S / d1
    dS_dsxx = -S / d2
    dS_dsxy = 2 * n1 / D
    return S, dS_dmx, dS_dsxx, dS_dsxy, mx, my


def ssim(img, tgt):
    """Mean SSIM over channels and pixels of [3, H, W] images (R32)."""
    return float(np.mean([ssim_terms(np.asarray(img[c], np.float64), np.asarray(tgt[c], np.float64))[0]
                          for c in range(img.shape[0])]))


def ssim_grad(img, tgt):
    """d mean-SSIM / d img by the chain rule through the local statistics:
    mu_x = G*x, sigma_xx = G*(x^2) - mu_x^2, sigma_xy = G*(x y) - mu_x mu_y, so
    d/dx(q) = sum_p G(p - q) [dS/dmu_x - 2 mu_x dS/dsigma_xx - mu_y dS/dsigma_xy](p)
            + 2 x(q) sum_p G(p - q) dS/dsigma_xx(p) + y(q) sum_p G(p - q) dS/dsigma_xy(p)
    (G symmetric: the sums are the same zero-padded correlation)."""
    img = np.asarray(img, np.float64)
    tgt = np.asarray(tgt, np.float64)
    C, H, W = img.shape
    out = np.zeros_like(img)
    for c in range(C):
        x, y = img[c], tgt[c]
        S, dmx, dsxx, dsxy, mx, my = ssim_terms(x, y)
        A = dmx - 2 * mx * dsxx - my * dsxy
        out[c] = blur(A) + 2 * x * blur(dsxx) + y * blur(dsxy)
    return out / (C * H * W)


def ssim_grad_mag(img, tgt):
    """R23 magnitude scale of ssim_grad: the same chain with every product and
    inner sum expanded in absolute value,
    m(q) = sum_p G(p - q) [|dS/dmu_x| + 2 |mu_x| |dS/dsigma_xx| + |mu_y| |dS/dsigma_xy|](p)
         + 2 |x(q)| sum_p G(p - q) |dS/dsigma_xx(p)| + |y(q)| sum_p G(p - q) |dS/dsigma_xy(p)|,
    divided by 3HW (G >= 0), so m >= |ssim_grad| elementwise."""
    img = np.asarray(img, np.float64)
    tgt = np.asarray(tgt, np.float64)
    C, H, W = img.shape
    out = np.zeros_like(img)
    for c in range(C):
        x, y = img[c], tgt[c]
        S, dmx, dsxx, dsxy, mx, my = ssim_terms(x, y)
        A = np.abs(dmx) + 2 * np.abs(mx) * np.abs(dsxx) + np.abs(my) * np.abs(dsxy)
        out[c] = blur(A) + 2 * np.abs(x) * blur(np.abs(dsxx)) + np.abs(y) * blur(np.abs(dsxy))
    return out / (C * H * W)


def color_loss(img, tgt, lam=0.2):
    """Eq. 10: (1 - lambda) mean|I^ - I| + lambda (1 - SSIM); returns
    (loss, l1, ssim, dL/dI^)."""
    img = np.asarray(img, np.float64)
    tgt = np.asarray(tgt, np.float64)
    n = img.size
    l1 = float(np.mean(np.abs(img - tgt)))
    s = ssim(img, tgt)
    g = (1 - lam) * np.sign(img - tgt) / n - lam * ssim_grad(img, tgt)
    return (1 - lam) * l1 + lam * (1 - s), l1, s, g
