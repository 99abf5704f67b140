"""C1 (BASELINE.json configs[0]): the CPU-runnable GLU- case.

512x512 RGB guide, s = 4, the LR image a 4x4 box mean (harness-supplied, the
reference has no box filter), target = clamp(M I + b) of the LR image (seeded
affine operator, seed 1001).  Path: optimize_field (upsample.cpp:194-216) then
apply_field (235-252).  Prints one JSON line: GPU latency per call pair
(CUDA events, device-resident), the reference library's CPU time for the same
calls (its own threading, and on all cores), and byte parity of the output.

    python tools/bench_c1.py [--reps N]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_09582_b200 as glu  # noqa: E402
from paper_2307_09582_b200 import workloads  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--reps", type=int, default=50)
a = p.parse_args()

cfg = workloads.CONFIGS[1]
W, H, s = cfg["W"], cfg["H"], cfg["scale"]
img = workloads.scene(W, H, 1, 0)
low = workloads.box_downsample(img, s)
target = workloads.affine_op(1001).apply_numpy(low)

high_d, low_d, tgt_d = (torch.from_numpy(x).cuda() for x in (img, low, target))
grid = glu.GridSpec.create(W, H, s)


def gpu_once():
    f = glu.optimize_field(high_d, low_d, grid)
    return glu.apply_field(f, tgt_d)


for _ in range(5):
    out = gpu_once()
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
      for _ in range(a.reps)]
for e0, e1 in ev:
    e0.record()
    out = gpu_once()
    e1.record()
torch.cuda.synchronize()
ms = sorted(e0.elapsed_time(e1) for e0, e1 in ev)

import oracle  # noqa: E402  (test infrastructure: the CPU reference arm)
ref = oracle.Reference()
ref.set_num_threads(0)
t = time.perf_counter()
P = ref.optimize_field(img, low, s)
want = ref.apply_field(P, s, target)
cpu_ms = (time.perf_counter() - t) * 1e3
t = time.perf_counter()
P2 = ref.optimize_field_allcores(img, low, s)
ref.apply_field(P2, s, target)
cpu_all_ms = (time.perf_counter() - t) * 1e3

print(json.dumps({
    "config": cfg["name"], "path": "optimize_field + apply_field (device-resident)",
    "gpu_ms_median": ms[len(ms) // 2], "gpu_ms_min": ms[0],
    "hr_mpix_per_s": W * H / (ms[len(ms) // 2] * 1e-3) / 1e6,
    "cpu_reference_ms": cpu_ms, "cpu_reference_threads": "its own: min(nproc, ceil(H/1024))",
    "cpu_reference_allcores_ms": cpu_all_ms, "cpu_threads": os.cpu_count(),
    "parity": bool(out.cpu().numpy().tobytes() == want.tobytes()),
    "data": "synthetic: seeded scene, 4x4 box-mean LR, affine operator seed 1001",
}), flush=True)
