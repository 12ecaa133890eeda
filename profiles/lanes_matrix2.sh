#!/bin/bash
# pipeline shape with the TMA gather (C2, C4)
for cfg in C2 C4; do for db in "4 8" "6 8" "8 8" "4 12" "3 16"; do
  set -- $db
  timeout 600 python bench.py --config $cfg --depth $1 --bundle $2 --no-cpu-baseline --no-e2e --out gpurun_out/lm2_${cfg}_$1x$2.json > /dev/null 2>> gpurun_out/lm2.err
  python -c "import json; d=json.load(open('gpurun_out/lm2_${cfg}_$1x$2.json')); r=d['roofline']; print('$cfg', '$1x$2', round(d['minibatches_per_s']), round(r['frac'],3))"
done; done
