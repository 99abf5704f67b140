#!/bin/bash
# On the GPU box: the round-2 evidence set, each command run plain first and
# then under ncu (one process per ncu run; 1 GPU).
#   bash tools/capture_r02.sh
cd "$(dirname "$0")/.."
T=r02
bash tools/capture_c3.sh $T
# launch list of one default bench step set (C3 frames, warm-up excluded)
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-c4 --no-c5 > gpurun_out/plain_bench.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 200 --csv \
    --log-file gpurun_out/${T}_bench_launches.csv python bench.py --steps 2 --warmup 1 \
    --no-cpu-baseline --no-c4 --no-c5 > gpurun_out/ncu_bench.log 2>&1
echo "bench launches rc=$?"
# C4 joint launch list (warm-up run skipped)
python tools/bench_joint.py --config 4 --reps 1 > gpurun_out/plain_joint.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_joint_c4_launches.csv python tools/bench_joint.py --config 4 --reps 1 \
    > gpurun_out/ncu_joint.log 2>&1
echo "joint launches rc=$?"
# C5 RGB apply (k_apply3b) full capture
python tools/bench_apply.py --targets 4 > gpurun_out/plain_apply.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_apply3b -s 2 -c 1 \
    -o gpurun_out/${T}_apply3b python tools/bench_apply.py --targets 4 > gpurun_out/ncu_apply.log 2>&1
echo "apply rc=$?"
