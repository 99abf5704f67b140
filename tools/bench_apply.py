"""C5 (BASELINE.json configs[4]): upsample-only interactive editing at 8K.

Params of a 7680x4320 / s=16 solve stay resident; 64 successive LR targets
(480x270 RGB, each a seeded colour-matrix edit of the LR image) are applied.
Reports HR Mpix/s and the apply kernel's HBM fraction (algorithmic bytes =
12 B params + 12 B RGB out per HR pixel + the LR target), parity of a sample
of targets against the CPU oracle, and the reference apply_field on the host.

    python tools/bench_apply.py [--targets 64] [--channels 3] [--cpu]
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
p.add_argument("--targets", type=int, default=64)
p.add_argument("--channels", type=int, default=3)
p.add_argument("--cpu", action="store_true")
p.add_argument("--tag", default="")
a = p.parse_args()

W, H, s = 7680, 4320, 16

# Under torchrun (WORLD_SIZE > 1): C5 over HR row bands (banded.py) -- each
# rank keeps its band of the field, rank 0 broadcasts every LR target over
# NCCL (double-buffered), rank 0 prints the max-over-ranks throughput.
WORLD = int(os.environ.get("WORLD_SIZE", "1"))
if WORLD > 1:
    import torch.distributed as dist
    from paper_2307_09582_b200 import banded
    LOCAL = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(LOCAL)
    dist.init_process_group("nccl", device_id=torch.device("cuda", LOCAL))
    rank = dist.get_rank()
    high = torch.from_numpy(workloads.scene(W, H, 4, 0)).cuda()
    low, grid = glu.grid_downsample(high, s)
    field = glu.optimize_field(high, low, grid)
    y0, y1 = banded.band_rows(grid, 3, WORLD, rank)
    band = field.params[y0:y1].clone()
    del field, high
    targets = None
    if rank == 0:
        targets = [glu.op_color(low, workloads.mix_op(1005 + k).M) for k in range(a.targets)]
        if a.channels == 1:
            targets = [glu.op_matte(t) for t in targets]
    shape = (y1 - y0, W, 3) if a.channels == 3 else (y1 - y0, W)
    outs = [torch.empty(shape, device="cuda") for _ in range(2)]
    state = {"k": 0}

    def app(p, g, t, c):
        o = outs[state["k"] % 2]
        state["k"] += 1
        return glu.glu.apply_field_band(p, g, t, c, out=o)

    for _ in range(2):  # warm-up (NCCL communicator, kernels)
        banded.run_banded_apply(band, grid, targets, min(3, a.targets), a.channels, apply=app)
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    banded.run_banded_apply(band, grid, targets, a.targets, a.channels, apply=app)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        ms = float(t.item())
        print(json.dumps({"config": f"C5 7680x4320 s16 upsample-only, {a.targets} targets, "
                                    f"{a.channels}-ch, {WORLD} row bands",
                          "n_gpus": WORLD, "scaling": "strong", "ms_total": ms,
                          "hr_mpix_per_s": a.targets * W * H / (ms * 1e-3) / 1e6,
                          "broadcast_bytes_per_target": grid.lowW * grid.lowH * 4 * a.channels}),
              flush=True)
    dist.destroy_process_group()
    sys.exit(0)

img = workloads.scene(W, H, 4, 0)
high = torch.from_numpy(img).cuda()
low, grid = glu.grid_downsample(high, s)
field = glu.optimize_field(high, low, grid)
targets = [glu.op_color(low, workloads.mix_op(1005 + k).M) for k in range(a.targets)]
if a.channels == 1:
    targets = [glu.op_matte(t) for t in targets]
shape = (H, W, 3) if a.channels == 3 else (H, W)
outs = [torch.empty(shape, device="cuda") for _ in range(2)]
for t in targets[:3]:
    glu.apply_field(field, t)
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
      for _ in targets]
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ctx = glu.glu.context()
import ctypes as C  # noqa: E402
lib, gc = glu._native.lib(), grid.c()
t0.record()
for k, t in enumerate(targets):
    ev[k][0].record()
    glu._native.check(lib.glu_cu_apply_field(ctx.handle, C.c_void_p(field.params.data_ptr()),
                                             C.byref(gc), C.c_void_p(t.data_ptr()), a.channels, 1,
                                             C.c_void_p(outs[k % 2].data_ptr())))
    ev[k][1].record()
t1.record()
torch.cuda.synchronize()
total_ms = t0.elapsed_time(t1)
kms = [e0.elapsed_time(e1) for e0, e1 in ev]
npx = W * H
nbytes = npx * (12 + 4 * a.channels) + grid.lowW * grid.lowH * 4 * a.channels
hbm = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                  "MEASURED_PEAKS.json")))["hbm_gbs"]
mean_ms = float(np.mean(kms))
line = {"config": f"C5 7680x4320 s16 upsample-only, {a.targets} targets, {a.channels}-ch",
        "hr_mpix_per_s": a.targets * npx / (total_ms * 1e-3) / 1e6,
        "apply_ms_mean": mean_ms, "apply_ms_min": min(kms),
        "algorithmic_bytes_per_launch": nbytes,
        "hbm_achieved_gbs": nbytes / (mean_ms * 1e-3) / 1e9,
        "hbm_frac_of_measured": nbytes / (mean_ms * 1e-3) / 1e9 / hbm,
        "hbm_peak_gbs_measured": hbm}
# parity on two targets against the oracle (bit-exact)
import oracle  # noqa: E402
ora = oracle.Oracle()
P = field.numpy()
for k in (0, a.targets - 1):
    want = ora.apply_field(P, targets[k].cpu().numpy())
    got = glu.apply_field(field, targets[k]).cpu().numpy()
    line[f"parity_target_{k}"] = bool(want.tobytes() == got.tobytes())
if a.cpu and a.channels == 3:
    ref = oracle.Reference()
    ref.set_num_threads(0)
    tt = time.perf_counter()
    n = 0
    while n < a.targets and time.perf_counter() - tt < 10:
        ref.apply_field(P, s, targets[n].cpu().numpy())
        n += 1
    line["cpu_reference_mpix_per_s"] = n * npx / (time.perf_counter() - tt) / 1e6
    line["cpu_threads"] = os.cpu_count()
print(json.dumps(line), flush=True)
