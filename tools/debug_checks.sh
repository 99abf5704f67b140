#!/bin/bash
# On the GPU box: rebuild every CUDA source with -DGLU_DEBUG_CHECKS (device
# bounds / invariant checks that trap) and run the GPU suite plus the C2 / C4
# joint runs against it; restore the release build afterwards.
#   bash tools/debug_checks.sh
cd "$(dirname "$0")/.."
L=paper_2307_09582_b200/lib
mkdir -p /tmp/glu_release && cp $L/*.o $L/libglu_cuda.so /tmp/glu_release/
for f in glu_kernels glu_solve32 glu_solve32f glu_solve32x glu_ccl glu_joint glu_glup glu_metrics glu_baselines glu_capi; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false \
    -std=c++17 -Xcompiler -fPIC -diag-suppress 177,550 -Iinclude -DGLU_DEBUG_CHECKS \
    -c paper_2307_09582_b200/csrc/$f.cu -o $L/$f.cu.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC \
  -o $L/libglu_cuda.so $L/glu_kernels.cu.o $L/glu_solve32.cu.o $L/glu_solve32f.cu.o $L/glu_solve32x.cu.o \
  $L/glu_ccl.cu.o $L/glu_joint.cu.o $L/glu_glup.cu.o $L/glu_metrics.cu.o $L/glu_baselines.cu.o $L/glu_capi.cu.o
echo "== debug-checks build: $(date)"
python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3
for m in fast gnu exact; do python tools/bench_joint.py --config 2 4 --reps 1 --mode $m 2>&1 | grep -c '"config"'; done
python tools/bench_joint.py --config 2 4 --reps 1 --trials 2 2>&1 | grep -c '"config"'
python tools/sanitize_joint.py --size 2048 2>&1 | tail -1
cp /tmp/glu_release/* $L/
