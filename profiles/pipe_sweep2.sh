#!/bin/bash
# depth x bundle sweep on the current kernels (C2, C3, C4)
for cfg in C2 C3 C4; do for db in "4 8" "4 12" "6 8" "3 16" "2 16"; do
  set -- $db
  python bench.py --config $cfg --depth $1 --bundle $2 --no-cpu-baseline --no-e2e --out gpurun_out/ps_${cfg}_$1x$2.json > /dev/null 2>> gpurun_out/ps.err
  python -c "import json; d=json.load(open('gpurun_out/ps_${cfg}_$1x$2.json')); print('$cfg', '$1x$2', round(d['minibatches_per_s']), round(d['roofline']['frac'],3))"
done; done
