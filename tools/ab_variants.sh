#!/bin/bash
# Build libglu_cuda.so variants of one source with different nvcc flags here
# (cross-compiled), into paper_2307_09582_b200/lib/variants/<name>/:
#   bash tools/ab_variants.sh glu_solve32x.cu NAME [flags...]
# On the GPU box, tools/ab_run.sh copies each variant in and times it.
set -e
cd "$(dirname "$0")/.."
SRC=$1; NAME=$2; shift 2
L=paper_2307_09582_b200/lib
V=$L/variants/$NAME
mkdir -p $V
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false \
  -std=c++17 -Xcompiler -fPIC -diag-suppress 177,550 -Iinclude -Xptxas -v "$@" \
  -c paper_2307_09582_b200/csrc/$SRC -o $V/$SRC.o 2>&1 | grep -E "registers|spill" | sed "s/^/[$NAME] /" >&2
OBJS=""
for f in glu_kernels glu_solve32 glu_solve32f glu_solve32x glu_ccl glu_joint glu_glup glu_metrics glu_baselines glu_capi; do
  if [ "$f.cu" = "$SRC" ]; then OBJS="$OBJS $V/$SRC.o"; else OBJS="$OBJS $L/$f.cu.o"; fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC \
  -o $V/libglu_cuda.so $OBJS
