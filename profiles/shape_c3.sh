#!/bin/bash
# C3 (N=1): 3x16 vs 4x16, alternating, 2 repeats.
mkdir -p gpurun_out/shape_c3
for i in 1 2; do for s in "3 16" "4 16"; do set -- $s; o=gpurun_out/shape_c3/C3_$1x$2_$i.json
  timeout 300 python bench.py --config C3 --depth $1 --bundle $2 --no-cpu-baseline --out $o > /dev/null 2>&1
  python -c "import json; d=json.load(open('$o')); print('C3', '$1x$2', $i, round(d['minibatches_per_s']), round(d['roofline']['frac'],3))" 2>/dev/null || echo "C3 $1x$2 failed"
done; done | tee gpurun_out/shape_c3/summary.txt
