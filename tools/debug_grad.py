"""Debug: worst gradient components of the full-size sampled backward parity."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from gpu_helpers import AMBIG, GS_GRAD_PARAMS, gpu_backward, gpu_forward, oracle, oracle_view
from paper_2312_10070_b200 import inputs
from test_gpu_fullsize import _tile_mask, _pixel_mask
s = inputs.config3(); view = s.views[0]
r, P, v = gpu_forward(s, view=view)
p64 = oracle.params64(*s.params())
pr = oracle.project(p64, oracle_view(s, view), s.cam)
idx, trg = oracle.bin_sort(pr["rect"], pr["culled"], pr["depth_key"], s.cam)
tmask = _tile_mask(s.cam, 48, 7)
fr = oracle.render(pr, p64["rgb"], idx, trg, s.cam, tile_mask=tmask)
gc, gd, ga = inputs.upstream_maps(11, s.cam)
keep = _pixel_mask(s.cam, tmask) & (fr["margin"] > AMBIG)
gc, gd, ga = gc * keep, gd * keep, ga * keep
gb = gpu_backward(r, P, v, gc, gd, ga, GS_GRAD_PARAMS)
ob = oracle.backward(p64, oracle_view(s, view), s.cam, idx, trg, gc, gd, ga, tile_mask=tmask)
for name, g, gs, m in (("g2", gb["g2"], ob["g2"], ob["m2"]), ("g3", gb["g3"], ob["g3"], ob["m3"])):
    err = np.abs(g - gs)
    score = err / (1e-3 * np.abs(gs) + 1e-6 * m + 1e-300)
    order = np.argsort(score.ravel())[::-1][:8]
    print(name)
    for o in order:
        i, c = divmod(o, g.shape[1])
        print(f"  gauss {i} comp {c}: gpu {g[i, c]: .6e} orc {gs[i, c]: .6e} m* {m[i, c]:.3e} err/m {err[i, c] / max(m[i, c], 1e-300):.2e} score {score[i, c]:.2f}")
        if name == "g3":
            print("     g2 gpu", np.array2string(gb["g2"][i], precision=4), "\n     g2 orc", np.array2string(ob["g2"][i], precision=4))
            print("     params", s.mean_opa[i], s.quat[i], s.logscale[i], "pz", pr["pz"][i], "conic", pr["conic"][i])
