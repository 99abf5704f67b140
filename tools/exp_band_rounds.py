"""Experiment: rounds of a banded trial schedule.  Trials are owned by the
HR row band holding their component's first pixel; a trial's round is the
longest path to it counting only edges between trials of different owners
(trials of one owner in one round run under the local dataflow scheduler).
Also: trials whose affected rows leave the owner's band + R-row halo.

    python tools/exp_band_rounds.py [--config 4]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_09582_b200 as glu  # noqa: E402
from paper_2307_09582_b200 import sharding, workloads  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=4)
a = p.parse_args()
cfg = workloads.CONFIGS[a.config]
W, H, s = cfg["W"], cfg["H"], cfg["scale"]
high = torch.from_numpy(workloads.scene(W, H, a.config, 0)).cuda()
r = glu.joint_optimize(high, s, glu.GluConfig(maxIterations=0))
les = glu.find_large_error(r.errors, glu.GluConfig().errorThreshold)
comps = [np.asarray(c, dtype=np.int64) for c in les.components]
n = len(comps)
h, reach = 1, 2
box = np.array([[(c % W).min() // s, (c // W).min() // s, (c % W).max() // s, (c // W).max() // s]
                for c in comps])
preds = []
for i in range(n):
    dx = np.maximum(0, np.maximum(box[:i, 0] - box[i, 2], box[i, 0] - box[:i, 2]))
    dy = np.maximum(0, np.maximum(box[:i, 1] - box[i, 3], box[i, 1] - box[:i, 3]))
    preds.append(np.nonzero(np.maximum(dx, dy) <= reach)[0])
depth = np.zeros(n, np.int64)
for i in range(n):
    depth[i] = 1 + (depth[preds[i]].max() if len(preds[i]) else 0)
print(f"{cfg['name']}: {n} trials, depth {depth.max()}, edges {sum(len(q) for q in preds)}")
lh = (H + s - 1) // s
for world in (2, 4, 8):
    bands = sharding.row_bands(H, s, 3, world)
    starts = np.array([b.lr_rows[0] for b in bands])
    owner = np.searchsorted(starts, box[:, 1], side="right") - 1
    rnd = np.zeros(n, np.int64)
    cross = 0
    for i in range(n):
        best = 0
        for j in preds[i]:
            if owner[j] == owner[i]:
                best = max(best, rnd[j])
            else:
                best = max(best, rnd[j] + 1)
                cross += 1
        rnd[i] = best
    out = {}
    for R in (2, 3, 4, 6):
        lo = starts[owner] - R
        hi = np.array([bands[o].lr_rows[1] for o in owner]) + R
        out[R] = int(((box[:, 1] - h < lo) | (box[:, 3] + h >= hi)).sum())
    per = np.bincount(owner, minlength=world)
    print(f"  world {world}: rounds {rnd.max() + 1}, cross-band edges {cross}, trials per band "
          f"{per.min()}..{per.max()}, non-local trials by halo R: {out}")
