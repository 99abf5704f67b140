#!/bin/bash
# On the GPU box: one `ncu --set full` capture of the first k_solve32f launch
# (the fused 4K frame) per libglu_cuda.so variant (tools/ab_head.sh builds them).
#   bash tools/ab_ncu.sh <mode> v1 v2 ...
cd "$(dirname "$0")/.."
L=paper_2307_09582_b200/lib
MODE=$1; shift
cp $L/libglu_cuda.so /tmp/libglu_cuda.so.main
for v in "$@"; do
  cp $L/variants/$v/libglu_cuda.so $L/libglu_cuda.so
  ncu --set full --clock-control none --import-source on -k regex:k_solve32f -c 1 -f \
      -o gpurun_out/ab_${MODE}_$v python tools/profile_solve.py --mode $MODE --iters 1 \
      > gpurun_out/ab_ncu_${MODE}_$v.log 2>&1
  echo "$v rc=$?"
done
cp /tmp/libglu_cuda.so.main $L/libglu_cuda.so
