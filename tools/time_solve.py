"""Time optimize_field on one 4K C3 frame for each mode / window / solver.

    python tools/time_solve.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2307_09582_b200 as glu  # noqa: E402
from paper_2307_09582_b200 import workloads  # noqa: E402

img = torch.from_numpy(workloads.scene(3840, 2160, 3, 0)).cuda()
low, grid = glu.grid_downsample(img, 8)
ctx = glu.glu.context()
for mode in ("fast", "gnu", "exact"):
    for S in (3, 5):
        for solver in (0, 1):
            ctx.set_solver(solver)
            cfg = glu.GluConfig(windowSide=S)
            md = glu.mode_from_name(mode)
            for _ in range(2):
                glu.optimize_field(img, low, grid, cfg, md)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                glu.optimize_field(img, low, grid, cfg, md)
            e1.record()
            torch.cuda.synchronize()
            print(f"{mode:5s} S={S} solver={solver}: {e0.elapsed_time(e1) / 5:.3f} ms", flush=True)
ctx.set_solver(0)
