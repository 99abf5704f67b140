#!/bin/bash
# Rebuild one CUDA source with extra nvcc flags on the GPU box, relink
# libglu_cuda.so, then run a command:
#   bash tools/ab_build.sh glu_solve32x.cu -DGLU_X_MIN_BLOCKS=3 -- python bench.py --mode exact
set -e
cd "$(dirname "$0")/.."
SRC=$1; shift
FLAGS=()
while [ "$1" != "--" ]; do FLAGS+=("$1"); shift; done
shift
L=paper_2307_09582_b200/lib
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false \
  -std=c++17 -Xcompiler -fPIC -diag-suppress 177,550 -Iinclude "${FLAGS[@]}" \
  -c paper_2307_09582_b200/csrc/$SRC -o $L/$SRC.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC \
  -o $L/libglu_cuda.so $L/glu_kernels.cu.o $L/glu_solve32.cu.o $L/glu_solve32f.cu.o $L/glu_solve32x.cu.o \
  $L/glu_ccl.cu.o $L/glu_joint.cu.o $L/glu_glup.cu.o $L/glu_metrics.cu.o $L/glu_baselines.cu.o $L/glu_capi.cu.o
echo "== $SRC ${FLAGS[*]}" >&2
"$@"
