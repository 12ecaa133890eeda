#!/bin/bash
# pipeline depth x bundle on C2 / C3 / C4 with every lane's graph captured during warm-up
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_lanes.log 2>&1; echo pytest=$?
for cfg in C2 C3 C4; do for db in "4 8" "6 8" "8 8" "8 4" "12 4"; do
  set -- $db
  python bench.py --config $cfg --depth $1 --bundle $2 --no-cpu-baseline --no-e2e --out gpurun_out/lm_${cfg}_$1x$2.json > /dev/null 2>> gpurun_out/lm.err
  python -c "import json; d=json.load(open('gpurun_out/lm_${cfg}_$1x$2.json')); r=d['roofline']; print('$cfg', '$1x$2', round(d['minibatches_per_s']), round(r['frac'],3))"
done; done
