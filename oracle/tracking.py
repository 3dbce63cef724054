"""Oracle of the masked tracking loss (Eq. 15) — TEST INFRASTRUCTURE ONLY.

Plain numpy, following the paper's definition step by step; shares nothing
with the CUDA path.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline / ``--impl reference`` leg may import it.

P:214-221 (Sec. 3.4, Eq. 15):
    L_tracking = sum M_inlier * M_alpha * (lambda_c |I^ - I|_1 + (1 - lambda_c) |D^ - D|_1)
  "Soft alpha mask M_alpha is a polynomial of the alpha map rendered directly
   from the active sub-map.  Error boolean mask M_inlier discards all the
   pixels where the color and depth errors are larger than a frame-relative
   error threshold."
Readings:
  R29  M_alpha = alpha^3 ("M_alpha = alpha^3"); the masks are constants:
       gradients flow to the rendered colour and depth only ("all the 3D
       Gaussian parameters are frozen").
  R30  frame-relative threshold = inlier_mult x the median error over the
       pixels with valid input depth (D > 0; "50 times larger than
       the median"), applied to the colour error (per-pixel mean over the 3
       channels) and to the depth error; median = the LOWER
       median (the order statistic of rank floor((n-1)/2)).
  R31  the two error maps and the threshold products that DECIDE the inlier
       mask are evaluated in fp32, each operation rounded to nearest in the
       documented order (residual, |.|, ((r+g)+b)/3; mult*median), as the
       kernel does, so the masks can be compared bit for bit; the loss value
       and gradients are then the fp64 definition over those masks.
"""
from __future__ import annotations

import numpy as np

F32 = np.float32


def error_maps32(color, depth, tgt_color, tgt_depth):
    """(e_c, e_d, valid) in fp32 (R31): e_c = ((|dr| + |dg|) + |db|) / 3."""
    c, tc = np.asarray(color, F32), np.asarray(tgt_color, F32)
    d, td = np.asarray(depth, F32), np.asarray(tgt_depth, F32)
    r = np.abs(c - tc)  # fp32 subtraction and abs, per channel
    e_c = ((r[0] + r[1]) + r[2]) / F32(3.0)
    e_d = np.abs(d - td)
    return e_c.astype(F32), e_d.astype(F32), td > 0


def lower_median(x):
    """Order statistic of rank floor((n - 1) / 2) (R30); None for n = 0."""
    x = np.asarray(x).ravel()
    if x.size == 0:
        return None
    k = (x.size - 1) // 2
    return np.partition(x, k)[k]


def tracking_loss(color, depth, alpha, tgt_color, tgt_depth, lambda_c=0.5, inlier_mult=50.0):
    """Eq. 15.  Returns dict(loss, med_c, med_d, inlier, m_alpha,
    g_color, g_depth), with the gradients of L w.r.t. the rendered colour and
    depth (masks held constant, R29; sign(0) = 0)."""
    e_c, e_d, valid = error_maps32(color, depth, tgt_color, tgt_depth)
    med_c, med_d = lower_median(e_c[valid]), lower_median(e_d[valid])
    if med_c is None:
        inlier = np.zeros_like(valid)
        med_c = med_d = F32(0.0)
    else:
        thr_c, thr_d = F32(inlier_mult) * med_c, F32(inlier_mult) * med_d  # fp32 products (R31)
        inlier = valid & (e_d <= thr_d) & (e_c <= thr_c)
    a = np.asarray(alpha, np.float64)
    m_alpha = a ** 3                                       # R29
    w = inlier * m_alpha
    c64, tc64 = np.asarray(color, np.float64), np.asarray(tgt_color, np.float64)
    d64, td64 = np.asarray(depth, np.float64), np.asarray(tgt_depth, np.float64)
    ec64 = np.abs(c64 - tc64).mean(axis=0)                 # |I^ - I|_1 per pixel, mean over channels
    ed64 = np.abs(d64 - td64)
    L = float(np.sum(w * (lambda_c * ec64 + (1.0 - lambda_c) * ed64)))
    g_color = w[None] * (lambda_c / 3.0) * np.sign(c64 - tc64)
    g_depth = w * (1.0 - lambda_c) * np.sign(d64 - td64)
    return dict(loss=L, med_c=F32(med_c), med_d=F32(med_d), inlier=inlier, m_alpha=m_alpha, g_color=g_color,
                g_depth=g_depth)
