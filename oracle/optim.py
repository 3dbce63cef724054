"""Oracle of the mapping epilogue (NEXT(3)) — TEST INFRASTRUCTURE ONLY.

Plain numpy fp64; shares nothing with the CUDA path.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / ``--impl
reference`` leg may import it.

* iso_reg: Eq. 11  L_reg = sum_k |s_k - s^bar_k|_1 / |K|, with
  s_k = exp(logscale_k) and s^bar_k the mean of s_k's three components (S:282,
  DESIGN.md R34); its gradient w.r.t. the log-scales (chain through exp).
* adam_step: the Adam update of S:215-228 (bias-corrected moments, per-group
  learning rates, quaternion renormalised after the step, entries with a
  non-finite gradient skipped).  The paper names no optimiser.
* prune: "prune Gaussians having opacity values lower than a threshold
  o_thre": keep sigmoid(logit) >= o_thre (decided in fp64, R35), in order.
"""
from __future__ import annotations

import numpy as np


def iso_reg(logscale):
    """(L_reg, dL_reg/dlogscale [N, 3]) for log-scales [N, >=3]."""
    l = np.asarray(logscale, np.float64)[:, :3]
    n = l.shape[0]
    if n == 0:
        return 0.0, np.zeros((0, 3))
    s = np.exp(l)
    sb = s.mean(axis=1, keepdims=True)
    L = float(np.abs(s - sb).sum() / n)
    d = np.sign(s - sb)
    # d/ds_j sum_i |s_i - mean(s)| = sign_j - mean(sign)
    g = (d - d.mean(axis=1, keepdims=True)) * s / n
    return L, g


# parameter array -> per-component learning-rate key (mean_opa packs mean xyz + opacity logit)
LR_KEYS = {"mean_opa": ["lr_mean"] * 3 + ["lr_opacity"], "quat": ["lr_quat"] * 4,
           "logscale": ["lr_logscale"] * 3 + [None], "rgb": ["lr_rgb"] * 3 + [None]}
NAMES = ("mean_opa", "quat", "logscale", "rgb")


def adam_step(params, grads, m, v, t, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """One step, returning new (params, m, v, n_skipped).  params / grads /
    m / v: dicts of [N, 4] arrays keyed by NAMES; lr: dict of the five rates."""
    params = {k: np.array(params[k], np.float64) for k in NAMES}
    m = {k: np.array(m[k], np.float64) for k in NAMES}
    v = {k: np.array(v[k], np.float64) for k in NAMES}
    g = {k: np.asarray(grads[k], np.float64) for k in NAMES}
    ok = np.ones(params["quat"].shape[0], bool)
    for k in NAMES:
        ok &= np.isfinite(g[k]).all(axis=1)
    for k in NAMES:
        rate = np.array([lr[key] if key else 0.0 for key in LR_KEYS[k]])
        mk = beta1 * m[k] + (1 - beta1) * g[k]
        vk = beta2 * v[k] + (1 - beta2) * g[k] ** 2
        mh = mk / (1 - beta1 ** t)
        vh = vk / (1 - beta2 ** t)
        pk = params[k] - rate * mh / (np.sqrt(vh) + eps)
        if k == "quat":
            with np.errstate(invalid="ignore"):  # rows with a non-finite gradient are dropped below
                pk = pk / np.linalg.norm(pk, axis=1, keepdims=True)
        params[k][ok], m[k][ok], v[k][ok] = pk[ok], mk[ok], vk[ok]
    return params, m, v, int((~ok).sum())


def prune_keep(logit, o_thre):
    """Boolean keep mask: sigmoid(logit) >= o_thre in fp64 (R35)."""
    return 1.0 / (1.0 + np.exp(-np.asarray(logit, np.float64))) >= o_thre
