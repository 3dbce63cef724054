"""Oracle of sub-map seeding (NEXT(4)) — TEST INFRASTRUCTURE ONLY.

Plain numpy (fp64 geometry, brute-force neighbour search); shares nothing
with the CUDA path except the documented integer permutation both sides
implement (a counter-based generator, allowed by the task rules).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import it.

P:156 (Sub-map Building): "For the following keyframes of the sub-map, we
sample M_k points uniformly from the regions with the rendered alpha values
lower than a threshold alpha_n ... New Gaussians are added to the sub-map
using sampled points that have no neighbors within a search radius rho in the
current sub-map ... their scales are defined based on the nearest neighbor
distance within the active sub-map."  P:230: alpha_n = 0.6, rho = 0.01 m;
P:624: opacity initialised to 0.5, initial scales = nearest-neighbour
distances.  Readings R37-R41:
  R37 eligible pixels: valid input depth (D > 0) and rendered alpha < alpha_n.
  R38 uniform sampling without replacement of min(M_k, n_eligible) pixels:
      the first M_k eligible pixels in the order of a seeded bijective
      permutation of the pixel indices (PERMUTATION below).
  R39 back-projection of pixel (i, j) at depth D (R3 pixel centres):
      p_c = ((i - cx) D / fx, (j - cy) D / fy, D), world p = R^T (p_c - t),
      in fp64, rounded to fp32 (the stored mean).
  R40 a candidate is rejected if an existing mean lies within rho
      (squared distance < rho^2, fp64 on the fp32 points) or an earlier
      candidate (sample order) does: accepted points are >= rho apart.
  R41 a new Gaussian: mean = the point, colour = the pixel's RGB, opacity
      logit 0 (o = 0.5), rotation (1, 0, 0, 0), log-scales = ln(clamp(d_nn,
      rho / 2, 0.1 m)) on all three axes, d_nn = distance to the nearest other
      point among the existing means and the accepted new points.
  R43 the first keyframe of a sub-map ("we sample M_u uniformly and M_c
      points from the keyframe point cloud in high color gradient regions"):
      a batch of M_u uniform samples (valid depth; the empty sub-map renders
      alpha 0), then a batch of M_c samples from the high-colour-gradient set
      against the sub-map that now holds the first batch.  High colour
      gradient: grey = (0.299 r + 0.587 g) + 0.114 b, 3x3
      Sobel gx, gy on interior pixels (0 on the border), m2 = gx^2 + gy^2, all
      in fp64 in this order; the set = valid-depth pixels with m2 strictly
      above the nearest-rank percentile (the ceil(q HW)-th smallest m2 over
      all pixels, q = 0.95).
"""
from __future__ import annotations

import numpy as np

M32 = 0xFFFFFFFF
NN_MAX = 0.1  # m: the clamp of R41 (and the neighbour-grid cell size of the CUDA path)


def _bits(n):
    m = 1
    while (1 << m) < n:
        m += 1
    return m


def permutation(n, seed):
    """The seeded bijection of [0, n) of R38, written out: on m-bit words
    (2^m >= n), x -> odd-multiply / xor-shift rounds keyed by the seed (each
    step is a bijection mod 2^m), cycle-walked back into [0, n)."""
    m = _bits(max(n, 2))
    mask = (1 << m) - 1
    s = np.uint64(seed & M32)

    def f(x):
        x = x.astype(np.uint64)
        for r in range(4):
            x = (x ^ ((s + np.uint64(0x9E3779B9 * (r + 1))) & np.uint64(mask))) & np.uint64(mask)
            x = (x * np.uint64(0x2545F491 | 1)) & np.uint64(mask)
            x = x ^ (x >> np.uint64((m + 1) // 2))
        return x

    # position i in [0, n) -> f(i), re-applying f while the value is >= n
    # (cycle-walking: the cycle of f through i returns to [0, n), so this ends
    # and is a bijection of [0, n))
    out = f(np.arange(n, dtype=np.uint64))
    bad = out >= n
    while bad.any():
        out[bad] = f(out[bad])
        bad = out >= n
    return out.astype(np.int64)


def seed(color, depth, alpha, view, cam, means, alpha_n=0.6, rho=0.01, max_new=100000, seed_=0):
    """Returns dict(idx (sampled pixel indices in order), points fp32 [K, 3],
    accepted mask, mean_opa / quat / logscale / rgb of the accepted Gaussians)."""
    H, W = depth.shape
    d = np.asarray(depth, np.float32).ravel()
    a = np.asarray(alpha, np.float32).ravel()
    eligible = (d > 0) & (a < np.float32(alpha_n))
    order = permutation(H * W, seed_)
    cand = order[eligible[order]][:max_new]
    i = (cand % W).astype(np.float64)
    j = (cand // W).astype(np.float64)
    z = d[cand].astype(np.float64)
    fx, fy, cx, cy = (float(np.float32(v)) for v in (cam.fx, cam.fy, cam.cx, cam.cy))
    pc = np.stack([(i - cx) * z / fx, (j - cy) * z / fy, z], axis=1)
    v = np.asarray(view, np.float64)
    R, t = v[:9].reshape(3, 3), v[9:12]
    dd = pc - t
    # R^T (p_c - t) written out: ((d0 R0c + d1 R1c) + d2 R2c), rounded to the stored fp32 mean
    pw = np.stack([(dd[:, 0] * R[0, c] + dd[:, 1] * R[1, c]) + dd[:, 2] * R[2, c] for c in range(3)],
                  axis=1).astype(np.float32)
    P = pw.astype(np.float64)
    E = np.asarray(means, np.float32)[:, :3].astype(np.float64)
    r2 = float(np.float32(rho)) ** 2
    K = len(cand)
    acc = np.ones(K, bool)
    for k in range(K):
        if len(E) and (((E - P[k]) ** 2).sum(axis=1) < r2).any():
            acc[k] = False
        elif k and (((P[:k] - P[k]) ** 2).sum(axis=1) < r2).any():
            acc[k] = False
    A = P[acc]
    pts = np.concatenate([E, A]) if len(E) else A
    nn = np.full(len(A), np.inf)
    for q in range(len(A)):
        d2 = ((pts - A[q]) ** 2).sum(axis=1)
        d2[len(E) + q] = np.inf  # itself
        nn[q] = np.sqrt(d2.min()) if len(d2) else np.inf
    s = np.log(np.clip(nn, float(np.float32(rho)) / 2, NN_MAX))
    cols = np.asarray(color, np.float32).reshape(3, -1)[:, cand[acc]].T
    n = int(acc.sum())
    return dict(idx=cand, points=pw, accepted=acc,
                mean_opa=np.concatenate([pw[acc], np.zeros((n, 1), np.float32)], axis=1),
                quat=np.tile(np.array([1, 0, 0, 0], np.float32), (n, 1)),
                logscale=np.concatenate([np.repeat(s[:, None], 3, axis=1), np.zeros((n, 1))], axis=1),
                rgb=np.concatenate([cols, np.zeros((n, 1), np.float32)], axis=1))


def gradient_m2(color):
    """R43: squared Sobel magnitude of the grey image, fp64 [H, W]."""
    c = np.asarray(color, np.float32).astype(np.float64)
    g = (0.299 * c[0] + 0.587 * c[1]) + 0.114 * c[2]
    H, W = g.shape
    m2 = np.zeros((H, W))
    if H < 3 or W < 3:
        return m2
    up, mid, dn = g[:-2], g[1:-1], g[2:]
    # gx = right column - left column, gy = bottom row - top row, (1, 2, 1) weights, in this order
    gx = ((up[:, 2:] + 2.0 * mid[:, 2:]) + dn[:, 2:]) - ((up[:, :-2] + 2.0 * mid[:, :-2]) + dn[:, :-2])
    gy = ((dn[:, :-2] + 2.0 * dn[:, 1:-1]) + dn[:, 2:]) - ((up[:, :-2] + 2.0 * up[:, 1:-1]) + up[:, 2:])
    m2[1:-1, 1:-1] = gx * gx + gy * gy
    return m2


def gradient_threshold(m2, q=0.95):
    """R43: the nearest-rank q-percentile of m2 over all pixels."""
    v = np.sort(np.asarray(m2, np.float64).ravel())
    k = max(int(np.ceil(q * v.size)), 1)
    return float(v[k - 1])


def gradient_mask(color, depth, q=0.95):
    """R43: the high-colour-gradient candidate set (bool [H, W])."""
    m2 = gradient_m2(color)
    return (m2 > gradient_threshold(m2, q)) & (np.asarray(depth, np.float32) > 0)


def first_keyframe(color, depth, view, cam, M_u, M_c, rho=0.01, seed_=0, q=0.95):
    """R43: the two insertion batches of a new sub-map's first keyframe;
    returns the two seed() results (the second against the first's Gaussians)."""
    H, W = np.asarray(depth).shape
    r1 = seed(color, depth, np.zeros((H, W), np.float32), view, cam, np.zeros((0, 4), np.float32),
              rho=rho, max_new=M_u, seed_=seed_)
    pseudo = np.where(gradient_mask(color, depth, q), 0.0, 1.0).astype(np.float32)
    r2 = seed(color, depth, pseudo, view, cam, r1["mean_opa"], alpha_n=0.5, rho=rho, max_new=M_c,
              seed_=seed_ + 1)
    return r1, r2
