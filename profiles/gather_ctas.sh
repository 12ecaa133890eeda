#!/bin/bash
# A/B: gather CTAs per SM (1 vs the default max resident) in the pipelined bench
for cfg in C2 C3 C4; do for n in 1 0; do
  EG_GATHER_CTAS=$n python bench.py --config $cfg --no-cpu-baseline --no-e2e --out gpurun_out/gc_${cfg}_$n.json > /dev/null 2>> gpurun_out/gc.err
  python -c "import json; d=json.load(open('gpurun_out/gc_${cfg}_$n.json')); r=d['roofline']; print('$cfg', 'ctas=$n', round(d['minibatches_per_s']), round(r['frac'],3), round(r['gather_ms_per_launch'],4), round(r['sample_chain_ms_per_launch'],4))"
done; done
