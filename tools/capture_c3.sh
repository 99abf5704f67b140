#!/bin/bash
# On the GPU box: one `ncu --set full` capture of each C3 solve kernel as the
# bench runs it (the batched launch over 16 frames),
# after a plain run of the same command.  Summarise here with
# tools/ncu_summary.py (--frames 16 for the batched captures; profiles/README.md).
#   bash tools/capture_c3.sh <tag>
cd "$(dirname "$0")/.."
TAG=${1:-r02}
for m in fast:k_solve32f:16 exact:k_solve32x:16 gnu:k_solve32f:16; do
  IFS=: read mode k nf <<< "$m"
  python tools/profile_solve.py --mode $mode --iters 1 --frames $nf > gpurun_out/plain_$mode.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
      -o gpurun_out/${TAG}_c3_$mode python tools/profile_solve.py --mode $mode --iters 1 --frames $nf \
      > gpurun_out/ncu_$mode.log 2>&1
  echo "$mode rc=$?"
done
