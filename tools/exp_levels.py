import sys, time, os
sys.path.insert(0, "/root/repo")
import torch
import paper_2307_09582_b200 as glu
from paper_2307_09582_b200 import workloads, distributed as D
for c in (2, 4):
    cfg = workloads.CONFIGS[c]
    high = torch.from_numpy(workloads.scene(cfg["W"], cfg["H"], c, 0)).cuda()
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        r, st = D.joint_optimize_local(high, cfg["scale"], 1)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    ref = glu.joint_optimize(high, cfg["scale"])
    same = torch.equal(r[0].errors, ref.errors)
    print(c, "level-sync world=1: %.1f ms" % (dt * 1e3), st["levels"], same, flush=True)
    # per-level timing of run_trials vs levels
