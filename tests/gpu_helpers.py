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


def small_submap(seed=5, n=40_000, V=4):
    """BJ.configs[3] reduced: n Gaussians, V views of 320x184 on the 1 m arc."""
    from paper_2312_10070_b200 import inputs
    s = inputs.config3(seed=seed, n=n, n_views=V)
    s.cam = inputs.Camera(320, 184, 160.0, 160.0, 159.5, 91.5)
    return s


def oracle_mapping_reference(s, ambig_residual=1e-5):
    """The fp64 oracle's mapping iteration over all views of scene s (Eq. 12
    L1 colour + depth, lambda = 1/V per view, R20): targets = the oracle's
    render of the perturbed copy rounded to fp32 (fed to both sides);
    per view the ambiguous pixels (R2 margin <= AMBIG, or a colour / valid
    depth residual within ambig_residual of 0, R21), whose upstream maps are
    zeroed on both sides; the summed gradient g3 [n,16] and its R23 scale m3,
    and the per-view losses (total, colour, depth) of the unmodified loss."""
    V = s.views.shape[0]
    p64 = oracle.params64(*s.params())
    tp = oracle.params64(*s.extra["target_params"])
    out = dict(tc={}, td={}, amb={}, loss=np.zeros((V, 3)), g3=np.zeros((s.n, 16)), m3=np.zeros((s.n, 16)))
    for v in range(V):
        view = s.views[v].astype(np.float64)
        tgt = oracle.forward(tp, view, s.cam)
        tc = tgt["color"].astype(np.float32)
        td = tgt["depth"].astype(np.float32)
        fr = oracle.forward(p64, view, s.cam)
        L, gc, gd = oracle.loss(s.cam, fr["color"], fr["depth"], tc, td, None, 1.0 / V, 1.0 / V)
        amb = (fr["margin"] <= AMBIG) | (np.abs(fr["color"] - tc) < ambig_residual).any(0) | (
            (td > 0) & (np.abs(fr["depth"] - td) < ambig_residual))
        gc[:, amb] = 0.0
        gd[amb] = 0.0
        b = oracle.backward(p64, view, s.cam, fr["sorted_idx"], fr["tile_range"], gc, gd)
        out["tc"][v], out["td"][v], out["amb"][v] = tc, td, amb
        out["loss"][v] = L
        out["g3"] += b["g3"]
        out["m3"] += b["m3"]
    return out


def zero_upstream_hook(ms, amb_dev):
    """A MapStep "bwd" stage hook: zero the view's loss-gradient maps at the
    oracle's ambiguous pixels (R2 treatment), then the ordinary per-pixel
    backward stage (on the lane's stream)."""
    def bwd(r, k, v):
        m = amb_dev[v]
        r.dL_dcolor.masked_fill_(m.unsqueeze(0).expand_as(r.dL_dcolor), 0.0)
        r.dL_ddepth.masked_fill_(m, 0.0)
        ms.stage_bwd(r, k, v)
    return bwd


def grads_as_g3(g):
    """A Grads buffer [4, n, 4] in the oracle's g3 layout [n, 16]."""
    return np.concatenate([to_np(g.mean_opa), to_np(g.quat), to_np(g.logscale), to_np(g.rgb)], 1)
