"""Summarise ncu outputs into profiles/ (tracked).

  python tools/ncu_summary.py launches <launches.csv> <out.md>
  python tools/ncu_summary.py kernel <report.ncu-rep> <out.md> [--traffic-key KEY] [--id N]
                                    [--sources a.cu,b.cuh]

`launches`: per-kernel launch count, total / mean device time and share of the
captured launches (ncu's launch list is cold-cache and serialised: compare
shares, not absolutes).  `kernel`: the SOL / occupancy / instruction / DRAM
metrics of one `--set full` capture plus the executed-instruction mix from the
SASS source page; with --traffic-key the per-launch DRAM bytes are also stored
in profiles/traffic.json for bench.py's roofline.traffic.
"""
from __future__ import annotations

import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FRAMES = 1  # frames per captured launch (--frames: a batched launch's numbers / frame)


def short(name: str) -> str:
    name = re.sub(r"\(.*$", "", name)
    name = name.replace("glu_cu::<unnamed>::", "").replace("unnamed>::", "")
    return name.strip()


def launches(path: str, out: str) -> None:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        try:
            agg[short(r[ik])].append(float(r[iv]) / 1e3)
        except ValueError:
            pass
    total = sum(sum(v) for v in agg.values())
    lines = [f"# ncu launch list: `{os.path.basename(path)}`", "",
             "gpu__time_duration.sum per launch, --clock-control none (cold-cache, serialised).",
             "", "| kernel | launches | total us | mean us | share |", "|---|---:|---:|---:|---:|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v):.1f} | {sum(v) / len(v):.2f} | "
                     f"{100 * sum(v) / total:.1f}% |")
    lines.append(f"| **total** | {sum(len(v) for v in agg.values())} | {total:.1f} | | 100% |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


WANT = [
    "Duration", "SM Frequency", "Elapsed Cycles", "Compute (SM) Throughput", "Memory Throughput",
    "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy",
    "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy", "Executed Instructions",
    "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler", "No Eligible",
    "Avg. Active Threads Per Warp", "Grid Size", "Block Size",
]


def kernel(rep: str, out: str, traffic_key: str | None, kid: int = 0,
           sources: list[str] | None = None) -> None:
    """Summarise result `kid` (0-based, ncu's ID) of the report."""
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    hdr = rows[0]
    im, iu, iv, ik = (hdr.index("Metric Name"), hdr.index("Metric Unit"),
                      hdr.index("Metric Value"), hdr.index("Kernel Name"))
    iid = hdr.index("ID")
    rows = [hdr] + [r for r in rows[1:] if r[iid] == str(kid)]
    kname = short(rows[1][ik]) if len(rows) > 1 else "?"
    vals = {}
    for r in rows[1:]:
        if r[im] in WANT and r[im] not in vals:
            vals[r[im]] = (r[iv], r[iu])
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    rawd = dict(zip(rr[0], rr[2 + kid])) if len(rr) > 2 + kid else {}
    units = dict(zip(rr[0], rr[1])) if len(rr) > 1 else {}

    def rawval(name):
        v = rawd.get(name)
        if v is None:
            return None
        v = float(v.replace(",", ""))
        u = units.get(name, "")
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)

    dram_r, dram_w = rawval("dram__bytes_read.sum"), rawval("dram__bytes_write.sum")
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                          capture_output=True, text=True).stdout
    blocks, cur = [], None
    for r in csv.reader(io.StringIO(sass)):
        if r and r[0] == "Kernel Name":
            cur = []
            blocks.append(cur)
        elif cur is not None:
            cur.append(r)
    # (the page may list a result twice in a row -- one block per source
    # view -- so identical consecutive blocks are merged)
    dedup = []
    for blk in blocks:
        if not dedup or dedup[-1][:3] != blk[:3] or len(dedup[-1]) != len(blk):
            dedup.append(blk)
    srows = [["Kernel Name"]] + (dedup[kid] if kid < len(dedup) else [])
    mix = collections.Counter()
    packed_flop = [0]  # warp-level flop lanes of the packed fp32 instructions
    if len(srows) > 2:
        h2 = srows[1]
        ie, isrc = h2.index("Instructions Executed"), h2.index("Source")
        for r in srows[2:]:
            try:
                n = int(r[ie])
            except (ValueError, IndexError):
                continue
            toks = r[isrc].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            mix[op.split(".")[0]] += n
            # packed fp32 pairs (FADD2 / FMUL2 / FFMA2): ncu's per-opcode thread
            # counters below do not include them; lanes = 2 when an operand is a
            # register pair (.F32x2), 1 for the all-scalar form
            if op.split(".")[0] in ("FADD2", "FMUL2", "FFMA2"):
                lanes = 2 if "F32x2" in r[isrc] else 1
                packed_flop[0] += n * lanes * (2 if op.startswith("FFMA2") else 1)
    lines = [f"# ncu --set full: `{kname}` ({os.path.basename(rep)})", "",
             "| metric | value |", "|---|---|"]
    for k in WANT:
        if k in vals:
            lines.append(f"| {k} | {vals[k][0]} {vals[k][1]} |")
    if dram_r is not None:
        lines.append(f"| dram__bytes_read.sum | {dram_r:.4g} B |")
        lines.append(f"| dram__bytes_write.sum | {dram_w:.4g} B |")
    tot = sum(mix.values())
    if tot:
        lines += ["", f"Executed warp instructions by opcode (total {tot}):", "",
                  "| opcode | warp instr | share |", "|---|---:|---:|"]
        for op, n in mix.most_common(20):
            lines.append(f"| {op} | {n} | {100 * n / tot:.1f}% |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    # executed floating-point work per launch (thread-level, predicated on):
    # FFMA = 2 flops (the north-star's hardware FP32 FLOP/s)
    cyc = rawval("smsp__cycles_elapsed.avg") or rawval("smsp__cycles_elapsed.max")

    def thread_ops(op):
        v = rawval(f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed")
        return v * cyc if v is not None and cyc else None

    f32 = [thread_ops(o) for o in ("ffma", "fadd", "fmul")]
    f64 = [thread_ops(o) for o in ("dfma", "dadd", "dmul")]
    fp32_exec = 2 * f32[0] + f32[1] + f32[2] if None not in f32 else None
    if fp32_exec is not None and packed_flop[0]:
        try:  # warp-level counts x the kernel's average active threads per warp
            act = float(vals["Avg. Active Threads Per Warp"][0])
        except (KeyError, ValueError):
            act = 32.0
        fp32_exec += packed_flop[0] * act
    fp64_exec = 2 * f64[0] + f64[1] + f64[2] if None not in f64 else None
    if fp32_exec is not None:
        extra = [f"| executed FP32 flop (2 FFMA + FADD + FMUL, thread-level; packed FFMA2 / FADD2 "
                 f"/ FMUL2 lanes included) | {fp32_exec:.4g} |",
                 f"| executed FP64 flop (2 DFMA + DADD + DMUL) | {fp64_exec:.4g} |"]
        lines[4:4] = extra
        open(out, "w").write("\n".join(lines) + "\n")
    if traffic_key and dram_r is not None:
        import hashlib
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        d = json.load(open(tp)) if os.path.exists(tp) else {}
        fr = FRAMES
        d[traffic_key] = (dram_r + dram_w) / fr
        if tot:  # executed warp instructions per launch (bench.py's issue bound)
            d[traffic_key + "_warp_instr"] = tot / fr
        if fp32_exec is not None:
            d[traffic_key + "_fp32_flop_executed"] = fp32_exec / fr
            d[traffic_key + "_fp64_flop_executed"] = fp64_exec / fr
        if fr > 1:
            d[traffic_key + "_frames_per_launch"] = fr
        if sources:  # bench.py flags the numbers stale when these files change
            h = hashlib.sha256()
            for f in sources:
                h.update(open(os.path.join(ROOT, f), "rb").read())
            d[traffic_key + "_src"] = {"files": sources, "sha256": h.hexdigest()[:16]}
        json.dump(d, open(tp, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        if "--frames" in sys.argv:  # a batched launch: per-frame numbers for traffic.json
            FRAMES = int(sys.argv[sys.argv.index("--frames") + 1])
        key = sys.argv[sys.argv.index("--traffic-key") + 1] if "--traffic-key" in sys.argv else None
        kid = int(sys.argv[sys.argv.index("--id") + 1]) if "--id" in sys.argv else 0
        srcs = (sys.argv[sys.argv.index("--sources") + 1].split(",")
                if "--sources" in sys.argv else None)
        kernel(sys.argv[2], sys.argv[3], key, kid, srcs)
