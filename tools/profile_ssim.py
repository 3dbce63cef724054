"""gs_ssim at BJ.configs[3] size (1200x680), for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_10070_b200 import inputs  # noqa: E402
from paper_2312_10070_b200.raster import camera, gs_ssim, lib  # noqa: E402

dev = torch.device("cuda:0")
cam = camera(inputs.Camera(1200, 680, 600.0, 600.0, 599.5, 339.5))
x = torch.rand(3, 680, 1200, device=dev)
y = (x * 0.9).contiguous()
ws = torch.empty((lib().gs_ssim_workspace_bytes(cam) + 15) // 16 * 4, dtype=torch.float32, device=dev)
loss = torch.zeros(4, device=dev)
g = torch.zeros_like(x)
for _ in range(3):
    gs_ssim(cam, x, y, 0.2, ws, loss, g)
torch.cuda.synchronize()
