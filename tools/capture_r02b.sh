#!/bin/bash
# On the GPU box: round-2 (second session) joint-loop evidence, each command
# run plain first and then under ncu / the trace build (one process per run).
#   bash tools/capture_r02b.sh
cd "$(dirname "$0")/.."
T=r02b
python tools/bench_joint.py --config 2 4 --reps 5 > gpurun_out/${T}_joint.jsonl 2>&1
# C4 joint launch list (the warm-up run is skipped by -s: its launches come first)
python tools/bench_joint.py --config 4 --reps 1 > gpurun_out/plain_joint.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_joint_c4_launches.csv python tools/bench_joint.py --config 4 --reps 1 \
    > gpurun_out/ncu_joint.log 2>&1
echo "joint launches rc=$?"
# scheduler trace (rebuilds glu_joint.cu with -DGLU_SCHED_TRACE; restore with a normal build)
bash tools/ab_sched.sh -DGLU_SCHED_TRACE -- python tools/sched_trace.py run gpurun_out/${T}_sched_trace.bin \
    > gpurun_out/${T}_trace_run.log 2>&1
echo "trace rc=$?"
