"""Critical-path analysis of the parallel trial scheduler (k_trial_sched).

    GPU box:  bash tools/ab_sched.sh -DGLU_SCHED_TRACE -- python tools/sched_trace.py run
    here:     python tools/sched_trace.py show gpurun_out/sched_trace.bin

`run` times one joint_optimize per config (after a warm-up) with the trace
build, which appends per-trial {claim, ready, end} %globaltimer stamps and
the trial boxes of every k_trial_sched launch to $GLU_SCHED_TRACE_FILE.
`show` reports, per launch: span, mean wait / run time, and the critical
path through the conflict graph (Chebyshev box distance <= 2h) weighted by
the measured run times -- the lower bound of any in-order schedule.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(out):
    import torch
    import paper_2307_09582_b200 as glu
    from paper_2307_09582_b200 import workloads
    for c in (2, 4):
        cfg = workloads.CONFIGS[c]
        high = torch.from_numpy(workloads.scene(cfg["W"], cfg["H"], c, 0)).cuda()
        glu.joint_optimize(high, cfg["scale"])
        torch.cuda.synchronize()
        os.environ["GLU_SCHED_TRACE_FILE"] = out + ".C%d" % c
        glu.joint_optimize(high, cfg["scale"])
        torch.cuda.synchronize()
        del os.environ["GLU_SCHED_TRACE_FILE"]


def launches(path):
    raw = open(path, "rb").read()
    o = 0
    while o < len(raw):
        magic, n = np.frombuffer(raw, np.uint64, 2, o)
        assert magic in (0x5452414345, 0x5452414346)
        words = 3 if magic == 0x5452414345 else 5
        n = int(n)
        o += 16
        allw = np.frombuffer(raw, np.uint64, words * n, o).astype(np.int64)
        st = allw[:3 * n].reshape(n, 3)
        sp = allw[3 * n:].reshape(n, 2) if words == 5 else np.zeros((n, 2), np.int64)
        o += 8 * words * n
        bx = np.frombuffer(raw, np.int32, 4 * n, o).reshape(n, 4).astype(np.int64)
        o += 16 * n
        yield st, bx, sp


def show(path, reach=2):
    for k, (st, bx, sp) in enumerate(launches(path)):
        n = len(st)
        t0 = st[:, 0].min()
        wait = (st[:, 1] - st[:, 0]) / 1e3
        runt = (st[:, 2] - st[:, 1]) / 1e3
        fin = np.zeros(n)
        depth = np.zeros(n, np.int64)
        for i in range(n):
            dx = np.maximum(0, np.maximum(bx[:i, 0] - bx[i, 2], bx[i, 0] - bx[:i, 2]))
            dy = np.maximum(0, np.maximum(bx[:i, 1] - bx[i, 3], bx[i, 1] - bx[:i, 3]))
            dep = np.maximum(dx, dy) <= reach
            fin[i] = runt[i] + (fin[:i][dep].max() if dep.any() else 0.0)
            depth[i] = 1 + (depth[:i][dep].max() if dep.any() else 0)
        # speculation bound: only accepted predecessors order a trial
        acc = (st[:, 2] & 1).astype(bool)
        fin2 = np.zeros(n)
        for i in range(n):
            dx = np.maximum(0, np.maximum(bx[:i, 0] - bx[i, 2], bx[i, 0] - bx[:i, 2]))
            dy = np.maximum(0, np.maximum(bx[:i, 1] - bx[i, 3], bx[i, 1] - bx[:i, 3]))
            dep = (np.maximum(dx, dy) <= reach) & acc[:i]
            fin2[i] = runt[i] + (fin2[:i][dep].max() if dep.any() else 0.0)
        span = (st[:, 2].max() - t0) / 1e3
        print(f"launch {k}: {n} trials, span {span:.0f} us, run mean {runt.mean():.1f} "
              f"p50 {np.median(runt):.1f} max {runt.max():.1f} us, wait mean {wait.mean():.1f} us, "
              f"sum run {runt.sum():.0f} us, critical path {fin.max():.0f} us "
              f"({depth.max()} trials deep); accepted {acc.sum()}, critical path through "
              f"accepted predecessors only {fin2.max():.0f} us")
        used = (st[:, 2] & 2).astype(bool)
        if True:
            print(f"   parked records used {used.sum()}: finalize mean {runt[used].mean():.1f} us, "
                  f"normal runs mean {runt[~used].mean():.1f} us; speculative runs "
                  f"{(sp[:, 0] > 0).sum()}, mean {((sp[:, 1] - sp[:, 0])[sp[:, 0] > 0]).mean() / 1e3:.1f} us")
        # the realised critical chain: walk back from the last trial to finish
        # through the predecessor that finished last before it became ready
        x = int(np.argmax(st[:, 2] >> 2))
        links = []
        endt = (st[:, 2] >> 2) << 2
        while True:
            dx = np.maximum(0, np.maximum(bx[:x, 0] - bx[x, 2], bx[x, 0] - bx[:x, 2]))
            dy = np.maximum(0, np.maximum(bx[:x, 1] - bx[x, 3], bx[x, 1] - bx[:x, 3]))
            dep = np.nonzero(np.maximum(dx, dy) <= reach)[0]
            links.append(x)
            if len(dep) == 0:
                break
            x = int(dep[np.argmax(endt[dep])])
        links = links[::-1]
        gaps = [(st[b, 1] - endt[a]) / 1e3 for a, b in zip(links, links[1:])]
        runs = [runt[b] for b in links]
        print(f"   realised chain: {len(links)} trials, run {np.sum(runs):.0f} us "
              f"(mean {np.mean(runs):.1f}), gaps {np.sum(gaps):.0f} us, parked used "
              f"{int(used[links].sum()) if used.any() else 0}, accepted {int(acc[links].sum())}; "
              f"starts at {(st[links[0], 1] - t0) / 1e3:.0f} us")
        # claim timeline: when did the last trial get claimed / become ready
        print(f"   last claim at {(st[:, 0].max() - t0) / 1e3:.0f} us, "
              f"last ready at {(st[:, 1].max() - t0) / 1e3:.0f} us")


PHASES = ["group", "replace", "affected", "backup+e0", "re-solve", "verdict", "log",
          "rollback+reset", "release"]


def show_phases(path):
    if not os.path.exists(path):
        return
    for k, line in enumerate(open(path)):
        v = [int(x) for x in line.split()]
        n = v[-1]
        print(f"launch {k} phases (SM cycles / trial): " +
              ", ".join(f"{nm} {c / n:.0f}" for nm, c in zip(PHASES, v[:9])))
        if len(v) > 10:
            print(f"   re-solved pixels / trial {v[10] / n:.0f}, fp64 fallbacks {v[9]} "
                  f"({100.0 * v[9] / max(1, v[10]):.3f}%)")
        if len(v) > 19:
            print(f"   speculative runs {v[18]}, parked records committed {v[17]}")
        if len(v) > 24:
            print(f"   spec pushes at start {v[19]}, at release {v[20]}, pops {v[21]}, "
                  f"finalizer saw in-flight {v[22]}, still queued {v[23]}")
        if len(v) > 25:
            print(f"   re-solved pixels kept unchanged (incremental test) {v[24]} "
                  f"({100.0 * v[24] / max(1, v[10] + v[24]):.1f} % of affected pixels)")
        if len(v) > 17:
            print("   fallback rule: nan %d, no-a/tiny %d, a-tie %d, zero-b %d, b-tie %d; "
                  "b close calls settled in double %d" % tuple(v[11:17]))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/sched_trace.bin")
    else:
        for f in sys.argv[2:]:
            print("==", f)
            show(f)
            show_phases(f + ".phases")
