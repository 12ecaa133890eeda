#!/bin/bash
# node priority with the TMA gather: gather-first vs sampling-first, repeated
for cfg in C2 C3; do for pr in gather sample gather sample; do
  EG_PRIO=$pr python bench.py --config $cfg --no-cpu-baseline --no-e2e --out gpurun_out/p2_${cfg}_$pr.json > /dev/null 2>> gpurun_out/p2.err
  python -c "import json; d=json.load(open('gpurun_out/p2_${cfg}_$pr.json')); r=d['roofline']; print('$cfg', '$pr', round(d['minibatches_per_s']), round(r['frac'],3))"
done; done
