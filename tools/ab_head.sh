#!/bin/bash
# Build a libglu_cuda.so variant whose glu_solve32f.cu (or another source) is
# taken from a git revision, into paper_2307_09582_b200/lib/variants/<name>/:
#   bash tools/ab_head.sh <rev> <source.cu> <name> [nvcc flags...]
set -e
cd "$(dirname "$0")/.."
REV=$1; SRC=$2; NAME=$3; shift 3
L=paper_2307_09582_b200/lib
V=$L/variants/$NAME
mkdir -p $V
TMP=paper_2307_09582_b200/csrc/_ab_$SRC
git show $REV:paper_2307_09582_b200/csrc/$SRC > $TMP
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false \
  -std=c++17 -Xcompiler -fPIC -diag-suppress 177,550 -Iinclude "$@" -c $TMP -o $V/$SRC.o
rm -f $TMP
OBJS=""
for f in glu_kernels glu_solve32 glu_solve32f glu_solve32x glu_ccl glu_joint glu_glup glu_metrics glu_baselines glu_capi; do
  if [ "$f.cu" = "$SRC" ]; then OBJS="$OBJS $V/$SRC.o"; else OBJS="$OBJS $L/$f.cu.o"; fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o $V/libglu_cuda.so $OBJS
