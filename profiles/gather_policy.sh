#!/bin/bash
# A/B: L2 eviction hints on the gather's row loads / output stores (EG_GATHER_POLICY)
for cfg in C2 C3 C4; do for pol in 0 1 3; do
  EG_GATHER_POLICY=$pol python bench.py --config $cfg --no-cpu-baseline --no-e2e --out gpurun_out/gp_${cfg}_$pol.json > /dev/null 2>> gpurun_out/gp.err
  python -c "import json; d=json.load(open('gpurun_out/gp_${cfg}_$pol.json')); r=d['roofline']; print('$cfg', 'pol=$pol', round(d['minibatches_per_s']), round(r['frac'],3), round(r['gather_ms_per_launch'],4), round(r['sample_chain_ms_per_launch'],4))"
done; done
