#!/bin/bash
# Rebuild glu_joint.cu with extra nvcc flags on the GPU box and run a command:
#   bash tools/ab_sched.sh -DGLU_SCHED_THREADS=512 -- python tools/bench_joint.py
# (the in-tree library is restored by the next `python -m paper_2307_09582_b200.build --force`).
set -e
cd "$(dirname "$0")/.."
FLAGS=()
while [ "$1" != "--" ]; do FLAGS+=("$1"); shift; done
shift
L=paper_2307_09582_b200/lib
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false \
  -std=c++17 -Xcompiler -fPIC -diag-suppress 177,550 -Iinclude "${FLAGS[@]}" \
  -c paper_2307_09582_b200/csrc/glu_joint.cu -o $L/glu_joint.cu.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC \
  -o $L/libglu_cuda.so $L/glu_kernels.cu.o $L/glu_solve32.cu.o $L/glu_solve32f.cu.o $L/glu_solve32x.cu.o \
  $L/glu_ccl.cu.o $L/glu_joint.cu.o $L/glu_glup.cu.o $L/glu_metrics.cu.o $L/glu_baselines.cu.o $L/glu_capi.cu.o
echo "== flags: ${FLAGS[*]}"
"$@"
