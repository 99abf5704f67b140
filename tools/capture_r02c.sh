#!/bin/bash
# On the GPU box: the end-of-round evidence set (round 2), each command run
# plain first and then under ncu (one process per ncu run; 1 GPU).
#   bash tools/capture_r02c.sh [tag]
cd "$(dirname "$0")/.."
T=${1:-r02c}
bash tools/capture_c3.sh $T
python bench.py > gpurun_out/${T}_bench.log 2>&1; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_ref.log 2>&1; echo "ref rc=$?"
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-c4 --no-c5 > gpurun_out/plain_bench.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${T}_bench_launches.csv python bench.py --steps 2 --warmup 1 \
    --no-cpu-baseline --no-c4 --no-c5 > gpurun_out/ncu_bench.log 2>&1
echo "bench launches rc=$?"
