"""Shared helpers of the -m gpu parity tests: run the CUDA path through the
C-ABI binding, run the oracle on the same seeded inputs, compare."""
import numpy as np
import torch

import oracle
from paper_2312_10070_b200 import GS_GRAD_PARAMS, GS_GRAD_POSE, Grads, Params, Rasterizer
from paper_2312_10070_b200.raster import GS_BWD_GAUSS_ONLY, GS_BWD_PIXELS_ONLY

# grad2d columns of the CUDA scratch in the oracle's g2 order
# (u, v, A, B, C, logit, r, g, b, p_z)
G2_FROM_GPU = [0, 1, 2, 3, 4, 6, 8, 9, 10, 5]
AMBIG = 1e-4  # R2: relative decision margin below which a pixel is ambiguous


def dev():
    return torch.device("cuda:0")


def to_np(t):
    return t.detach().cpu().numpy()


def gpu_forward(scene, view=None, capacity=None, stats=True):
    d = dev()
    P = Params.from_numpy(*scene.params(), device=d)
    v = torch.as_tensor(scene.views[0] if view is None else view, dtype=torch.float32, device=d).contiguous()
    r = Rasterizer(scene.n, scene.cam, device=d)
    if capacity is None:
        r.size_for(P, v)
    else:
        r.set_capacity(capacity)
    r.forward(P, v, stats=stats)
    torch.cuda.synchronize()
    return r, P, v


def gpu_frame(r):
    f = r.frame
    return dict(color=to_np(f.color), depth=to_np(f.depth), alpha=to_np(f.alpha), T_final=to_np(f.T_final),
                n_contrib=to_np(f.n_contrib), scanned=to_np(f.stats[0]), contrib=to_np(f.stats[1]))


def gpu_proj(r):
    p = r.proj
    n = r.n
    return dict(uv=to_np(p.uv)[:n], conic_o=to_np(p.conic_o)[:n], coef=to_np(p.coef)[:n], rgbz=to_np(p.rgbz)[:n],
                depth=to_np(p.depth)[:n], rect=to_np(p.rect)[:n].astype(np.int32),
                tiles_touched=to_np(p.tiles_touched)[:n])


def gpu_sort(r):
    P = int(r.n_pairs.item())
    return to_np(r.sorted_idx)[:P], to_np(r.tile_range)


def oracle_view(scene, view=None):
    return np.asarray(scene.views[0] if view is None else view, np.float64)


def grad_check(g, gstar, mstar, rtol=1e-3, atol_rel=1e-6):
    """R23: |g - g*| <= rtol |g*| + atol_rel m*  per component."""
    err = np.abs(np.asarray(g, np.float64) - gstar)
    bound = rtol * np.abs(gstar) + atol_rel * mstar
    ok = err <= bound
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(mstar > 0, err / np.maximum(mstar, 1e-300), np.where(err > 0, np.inf, 0.0))
    return ok, dict(n=int(ok.size), bad=int((~ok).sum()), worst_err_over_m=float(np.max(r)) if r.size else 0.0)


def gpu_backward(r, P, v, gC, gD, gA=None, flags=GS_GRAD_PARAMS):
    d = dev()
    t = lambda a: None if a is None else torch.as_tensor(np.ascontiguousarray(a, np.float32), device=d)
    g = Grads.zeros(r.n, d) if flags & GS_GRAD_PARAMS else None
    maps = dict(dL_dcolor=t(gC), dL_ddepth=t(gD), dL_dalpha=t(gA))
    r.backward(P, v, flags | GS_BWD_PIXELS_ONLY, g, **maps)
    torch.cuda.synchronize()
    out = dict(g2=to_np(r.grad2d)[:, G2_FROM_GPU].copy())
    r.backward(P, v, flags | GS_BWD_GAUSS_ONLY, g, **maps)
    torch.cuda.synchronize()
    assert not to_np(r.grad2d).any()  # scratch returned zeroed
    if g is not None:
        out["g3"] = np.concatenate([to_np(g.mean_opa), to_np(g.quat), to_np(g.logscale), to_np(g.rgb)], 1)
    return out


__all__ = ["GS_GRAD_PARAMS", "GS_GRAD_POSE", "oracle"]
