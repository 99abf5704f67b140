#!/bin/bash
# On the GPU box: for each variant directory built by tools/ab_variants.sh,
# swap its libglu_cuda.so in and run the command (default: tools/ab_time.py).
#   bash tools/ab_run.sh "python tools/ab_time.py --mode exact" v1 v2 ...
cd "$(dirname "$0")/.."
L=paper_2307_09582_b200/lib
CMD=$1; shift
cp $L/libglu_cuda.so /tmp/libglu_cuda.so.main
for v in "$@"; do
  cp $L/variants/$v/libglu_cuda.so $L/libglu_cuda.so
  $CMD --tag $v
done
cp /tmp/libglu_cuda.so.main $L/libglu_cuda.so
