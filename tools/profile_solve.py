"""Run the C3 hot kernels a few times on one 4K frame (for ncu / sanitizer).

    python tools/profile_solve.py [--mode fast|exact|gnu] [--solver 0|1|2] [--iters N]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_09582_b200 as glu  # noqa: E402
from paper_2307_09582_b200 import workloads  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--mode", default="fast")
p.add_argument("--solver", type=int, default=0)
p.add_argument("--iters", type=int, default=3)
p.add_argument("--width", type=int, default=3840)
p.add_argument("--height", type=int, default=2160)
p.add_argument("--scale", type=int, default=8)
p.add_argument("--window", type=int, default=3)
p.add_argument("--frames", type=int, default=0,
               help="> 1: the batched video path (glu_cu_upsample_frames over N frames)")
a = p.parse_args()
if a.frames > 1:
    fr = torch.from_numpy(np.stack([workloads.scene(a.width, a.height, 3, k)
                                    for k in range(a.frames)])).cuda()
    for _ in range(a.iters):
        vid = glu.glu.upsample_frames(fr, a.scale, "matte", mode=glu.mode_from_name(a.mode))
    torch.cuda.synchronize()
    print("ok", tuple(vid.shape))
    sys.exit(0)

img = torch.from_numpy(workloads.scene(a.width, a.height, 3, 0)).cuda()
ctx = glu.glu.context()
ctx.set_solver(a.solver)
low, grid = glu.grid_downsample(img, a.scale)
matte = glu.op_matte(low)
cfg = glu.GluConfig(windowSide=a.window)
for _ in range(a.iters):
    out, _ = glu.solve_apply(img, low, grid, matte, cfg, glu.mode_from_name(a.mode))
    field = glu.optimize_field(img, low, grid, cfg, glu.mode_from_name(a.mode))
    rec = glu.apply_field(field, low)
torch.cuda.synchronize()
print("ok", out.shape, ctx.launches, "launches", ctx.fallbacks, "fp64-verified pixels")
