#!/bin/bash
# Re-check the pipeline shape (lanes x bundle) after the count/scan block-floor change (C2, C4, N=1).
mkdir -p gpurun_out/shape
for C in C2 C4; do for s in "3 16" "2 32" "3 32" "4 16" "3 24" "4 12"; do set -- $s
  timeout 300 python bench.py --config $C --depth $1 --bundle $2 --no-cpu-baseline --out gpurun_out/shape/${C}_$1x$2.json > /dev/null 2>&1
  python -c "import json; d=json.load(open('gpurun_out/shape/${C}_$1x$2.json')); print('$C', '$1x$2', round(d['minibatches_per_s']), round(d['roofline']['frac'],3))" || echo "$C $1x$2 failed"
done; done | tee gpurun_out/shape/summary.txt
