#!/bin/bash
# On the GPU box: the bench's headline (C3 batched frames) per libglu_cuda.so variant.
#   bash tools/ab_bench.sh v1 v2 ...
cd "$(dirname "$0")/.."
L=paper_2307_09582_b200/lib
cp $L/libglu_cuda.so /tmp/libglu_cuda.so.main
for v in "$@"; do
  cp $L/variants/$v/libglu_cuda.so $L/libglu_cuda.so
  python bench.py --steps 20 --warmup 5 --no-c4 --no-c5 $BENCH_FLAGS 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
ps = d['roofline'].get('pair_search', {})
print('$v', round(d['value'], 1), round(d['roofline']['kernel_ms'], 5), (d.get('cpu_baseline') or {}).get('parity_vs_gpu'),
      'exact', round(ps.get('kernel_ms', 0), 5), ps.get('parity'))"
done
cp /tmp/libglu_cuda.so.main $L/libglu_cuda.so
