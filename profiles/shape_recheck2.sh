#!/bin/bash
# C2 / C4: 3x16 vs 4x16, alternating, 3 repeats each (N=1).
mkdir -p gpurun_out/shape2
for i in 1 2 3; do for C in C2 C4; do for s in "3 16" "4 16"; do set -- $s
  o=gpurun_out/shape2/${C}_$1x$2_$i.json
  timeout 300 python bench.py --config $C --depth $1 --bundle $2 --no-cpu-baseline --out $o > /dev/null 2>&1
  python -c "import json; d=json.load(open('$o')); print('$C', '$1x$2', $i, round(d['minibatches_per_s']), round(d['roofline']['frac'],3))" 2>/dev/null || echo "$C $1x$2 failed"
done; done; done | tee gpurun_out/shape2/summary.txt
