"""A/B helper: time the C3 solve (optimize_field and the fused solve + 1-ch
apply) on one 4K frame with the fp32-filter kernels and check the field bit
for bit against the fp64 reference-order kernel (solver 1).

    python tools/ab_time.py [--mode exact|fast|gnu] [--tag NAME]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2307_09582_b200 as glu  # noqa: E402
from paper_2307_09582_b200 import workloads  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--mode", default="exact")
p.add_argument("--tag", default="")
p.add_argument("--reps", type=int, default=20)
a = p.parse_args()

img = torch.from_numpy(workloads.scene(3840, 2160, 3, 0)).cuda()
low, grid = glu.grid_downsample(img, 8)
matte = glu.op_matte(low)
ctx = glu.glu.context()
md = glu.mode_from_name(a.mode)
cfg = glu.GluConfig()


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps


ctx.set_solver(1)
ref = glu.optimize_field(img, low, grid, cfg, md).params.clone()
ref_out, _ = glu.solve_apply(img, low, grid, matte, cfg, md)
ctx.set_solver(0)
f0 = ctx.fallbacks
got = glu.optimize_field(img, low, grid, cfg, md).params
out, _ = glu.solve_apply(img, low, grid, matte, cfg, md)
same = bool(torch.equal(ref.view(torch.int32), got.view(torch.int32))) and bool(
    torch.equal(ref_out.view(torch.int32), out.view(torch.int32)))
t_field = timed(lambda: glu.optimize_field(img, low, grid, cfg, md))
t_fused = timed(lambda: glu.solve_apply(img, low, grid, matte, cfg, md))
print(json.dumps({"tag": a.tag, "mode": a.mode, "field_ms": round(t_field, 4),
                  "fused_ms": round(t_fused, 4), "bitexact": same,
                  "fallbacks": ctx.fallbacks - f0}), flush=True)
