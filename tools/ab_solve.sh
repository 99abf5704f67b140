#!/bin/bash
# Rebuild glu_solve32.cu with extra nvcc flags on the GPU box, then time the
# C3 solve kernel through bench.py (kernel_ms of the roofline object):
#   bash tools/ab_solve.sh -DGLU_SOLVE_MIN_BLOCKS=7
set -e
cd "$(dirname "$0")/.."
L=paper_2307_09582_b200/lib
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false \
  -std=c++17 -Xcompiler -fPIC -diag-suppress 177,550 -Iinclude "$@" \
  -c paper_2307_09582_b200/csrc/glu_solve32.cu -o $L/glu_solve32.cu.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC \
  -o $L/libglu_cuda.so $L/glu_kernels.cu.o $L/glu_solve32.cu.o $L/glu_solve32f.cu.o $L/glu_solve32x.cu.o \
  $L/glu_ccl.cu.o $L/glu_joint.cu.o $L/glu_glup.cu.o $L/glu_metrics.cu.o $L/glu_baselines.cu.o $L/glu_capi.cu.o
python bench.py --steps 5 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('flags: $*', 'kernel_ms %.4f' % r['kernel_ms'], 'value %.0f' % d['value'], 'frac %.3f' % r['frac'])"
