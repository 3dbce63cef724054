"""One mapping view of BJ.configs[3] (or [1]/[4]) for ncu captures.

    python tools/profile_view.py [--config 3] [--reps 2]

Runs `reps` untimed passes of project -> bin_sort -> render + loss (fused) -> bwd on
view 0 after setup, so `ncu -k regex:<kernel> -s <reps-1> -c 1` captures one
steady-state launch of each kernel.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2312_10070_b200 import GS_GRAD_PARAMS, GS_GRAD_POSE, Grads, Params, Rasterizer, inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--pose", action="store_true")
    a = ap.parse_args()
    s = {1: inputs.config1, 2: inputs.config2, 3: inputs.config3, 4: inputs.config4}[a.config]()
    d = torch.device("cuda")
    P = Params.from_numpy(*s.params(), device=d)
    v = torch.as_tensor(s.views[0], device=d)
    r = Rasterizer(s.n, s.cam, device=d)
    r.size_for(P, v)
    if "target_params" in s.extra:
        Pt = Params.from_numpy(*s.extra["target_params"], device=d)
        r.forward(Pt, v)
    else:
        r.forward(P, v)
    tc, td = r.frame.color.clone(), r.frame.depth.clone()
    g = Grads.zeros(s.n, d)
    sc = r.loss_scales(td)
    torch.cuda.synchronize()
    for _ in range(a.reps):
        # the step's path: S3 + S4 fused (gs_render_fwd_l1 + gs_loss_from_tiles);
        # gs_loss once more for its own capture (the SSIM step's loss kernels)
        r.project(P, v)
        r.bin_sort()
        r.render_l1(tc, td, 1.0, 1.0, sc)
        r.compute_loss(tc, td)
        r.backward(P, v, GS_GRAD_POSE if a.pose else GS_GRAD_PARAMS, None if a.pose else g)
        if a.pose:
            r.pose_grad(v)
    torch.cuda.synchronize()
    print("pairs", int(r.n_pairs.item()))


if __name__ == "__main__":
    main()
