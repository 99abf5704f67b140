"""Time joint_optimize (C2 / C4 of BASELINE.json) on the GPU and the reference on CPU.

    python tools/bench_joint.py [--config 2|4] [--reps N] [--cpu]

Prints one JSON line per config: GPU wall/CUDA-event time of glu_cu_joint_optimize
(device-resident input), its sweep / trial counts, bitwise parity with the
reference library (oracle/_ref) and the reference's own CPU time.
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
p.add_argument("--config", type=int, nargs="+", default=[2, 4])
p.add_argument("--reps", type=int, default=3)
p.add_argument("--cpu", action="store_true")
p.add_argument("--trials", type=int, default=0, help="GLU_OPT_TRIALS (0 speculative, 2 dataflow)")
p.add_argument("--mode", default="fast", choices=["fast", "exact", "gnu"])
p.add_argument("--tag", default="")
a = p.parse_args()

# Under torchrun (WORLD_SIZE > 1) the level-synchronous multi-rank loop runs
# over NCCL, one rank per GPU, and rank 0 reports the max-over-ranks time.
WORLD = int(os.environ.get("WORLD_SIZE", "1"))
if WORLD > 1:
    import torch.distributed as dist
    from paper_2307_09582_b200 import distributed as D
    LOCAL = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(LOCAL)
    dist.init_process_group("nccl", device_id=torch.device("cuda", LOCAL))
    for c in a.config:
        cfg = workloads.CONFIGS[c]
        img = torch.from_numpy(workloads.scene(cfg["W"], cfg["H"], c, 0)).cuda()
        D.joint_optimize_distributed(img, cfg["scale"])
        times = []
        for _ in range(a.reps):
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = D.joint_optimize_distributed(img, cfg["scale"])
            e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            times.append(float(t.item()))
        if dist.get_rank() == 0:
            print(json.dumps({"config": cfg["name"], "ranks": WORLD, "gpu_ms": min(times),
                              "accepted": r.trialsAccepted, "rejected": r.trialsRejected}),
                  flush=True)
    dist.destroy_process_group()
    sys.exit(0)

glu.glu.context().set_trials(a.trials)
for c in a.config:
    cfg = workloads.CONFIGS[c]
    W, H, s = cfg["W"], cfg["H"], cfg["scale"]
    img = workloads.scene(W, H, c, 0)
    high = torch.from_numpy(img).cuda()
    md = glu.mode_from_name(a.mode)
    r = glu.joint_optimize(high, s, None, md)  # warm-up
    torch.cuda.synchronize()
    times = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = glu.joint_optimize(high, s, None, md)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    line = {"config": cfg["name"], "mode": a.mode, "tag": a.tag, "gpu_ms": min(times), "gpu_ms_all": times,
            "iterations": r.iterations, "accepted": r.trialsAccepted,
            "rejected": r.trialsRejected, "components": r.components,
            "hr_mpix_per_s": W * H / (min(times) * 1e-3) / 1e6}
    if a.cpu:
        import oracle
        ref = oracle.Reference()
        ref.set_num_threads(0)
        t0 = time.perf_counter()
        o = ref.joint_optimize(img, s, mode=a.mode)
        line["cpu_ms"] = 1e3 * (time.perf_counter() - t0)
        line["cpu_threads"] = os.cpu_count()
        line["parity"] = bool(
            o["low"].tobytes() == r.low.cpu().numpy().tobytes()
            and o["errors"].tobytes() == r.errors.cpu().numpy().tobytes()
            and o["field"].tobytes() == r.field.numpy().tobytes()
            and (o["accepted"], o["rejected"]) == (r.trialsAccepted, r.trialsRejected))
    print(json.dumps(line), flush=True)
