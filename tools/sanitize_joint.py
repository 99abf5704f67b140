"""Run the joint loop (every trial schedule) and the C3 solve kernels once, as
a checking workload: under the -DGLU_DEBUG_CHECKS build (tools/debug_checks.sh)
or, where a pool allows it, compute-sanitizer (one tool per call; the B200
pool used for this repo has it closed):

    compute-sanitizer --tool memcheck python tools/sanitize_joint.py --size 2048
    compute-sanitizer --tool racecheck python tools/sanitize_joint.py --size 384

Checks the results against the sequential schedule (bitwise) and exits 1 on a
mismatch."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2307_09582_b200 as glu  # noqa: E402
from paper_2307_09582_b200 import workloads  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--size", type=int, default=2048)
p.add_argument("--scale", type=int, default=8)
p.add_argument("--no-solve", action="store_true")
a = p.parse_args()

high = torch.from_numpy(workloads.scene(a.size, a.size, 2, 0)).cuda()
ctx = glu.glu.context()
res = {}
for trials in (1, 0, 2):  # sequential, speculative, dataflow
    ctx.set_trials(trials)
    res[trials] = glu.joint_optimize(high, a.scale)
ctx.set_trials(0)
ok = all(torch.equal(res[1].low, r.low) and torch.equal(res[1].field.params, r.field.params)
         and torch.equal(res[1].errors, r.errors) for r in res.values())
if not a.no_solve:
    low, grid = glu.grid_downsample(high, a.scale)
    matte = glu.op_matte(low)
    for m in ("fast", "gnu", "exact"):
        glu.solve_apply(high, low, grid, matte, None, glu.mode_from_name(m))
        glu.optimize_field(high, low, grid, None, glu.mode_from_name(m))
torch.cuda.synchronize()
print(f"joint {a.size}^2 s={a.scale}: {res[1].trialsAccepted}/{res[1].trialsRejected} trials, "
      f"schedules agree: {ok}")
sys.exit(0 if ok else 1)
