"""Experiment: how much of the first joint sweep's dependency depth comes from
bounding-box over-approximation?  Depth (trials on the longest conflict chain)
with the box rule used by the scheduler vs the exact rule (some pair of the
components' cells within Chebyshev 2h).

    python tools/exp_conflicts.py [--config 2]
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
p.add_argument("--config", type=int, default=2)
a = p.parse_args()
cfg = workloads.CONFIGS[a.config]
W, H, s = cfg["W"], cfg["H"], cfg["scale"]
high = torch.from_numpy(workloads.scene(W, H, a.config, 0)).cuda()
r = glu.joint_optimize(high, s, glu.GluConfig(maxIterations=0))
les = glu.find_large_error(r.errors, glu.GluConfig().errorThreshold)
comps = [np.asarray(c, dtype=np.int64) for c in les.components]
n = len(comps)
reach = 2
cells = [np.unique(((c // W) // s) * 100000 + (c % W) // s) for c in comps]
box = np.array([[ (cc % 100000).min(), (cc // 100000).min(), (cc % 100000).max(), (cc // 100000).max()]
                for cc in cells])
# dilated cell sets for the exact rule
dil = []
for cc in cells:
    ys, xs = cc // 100000, cc % 100000
    d = set()
    for dy in range(-reach, reach + 1):
        for dx in range(-reach, reach + 1):
            d.update(((ys + dy) * 100000 + xs + dx).tolist())
    dil.append(d)
depth_box = np.zeros(n, np.int64)
depth_ex = np.zeros(n, np.int64)
edges_box = edges_ex = 0
for i in range(n):
    dx = np.maximum(0, np.maximum(box[:i, 0] - box[i, 2], box[i, 0] - box[:i, 2]))
    dy = np.maximum(0, np.maximum(box[:i, 1] - box[i, 3], box[i, 1] - box[:i, 3]))
    cand = np.nonzero(np.maximum(dx, dy) <= reach)[0]
    edges_box += len(cand)
    depth_box[i] = 1 + (depth_box[cand].max() if len(cand) else 0)
    ex = [j for j in cand if not dil[i].isdisjoint(cells[j].tolist())]
    edges_ex += len(ex)
    depth_ex[i] = 1 + (depth_ex[ex].max() if ex else 0)
print(f"{cfg['name']}: {n} components; box rule: {edges_box} edges, depth {depth_box.max()}; "
      f"exact cell rule: {edges_ex} edges, depth {depth_ex.max()}")
