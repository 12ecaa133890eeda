#!/bin/bash
# TMA gather with L2 evict-first hints on gather4 loads and bulk stores vs none (interleaved)
for cfg in C2 C4; do for v in base l2h base l2h; do
  lib=""; [ $v != base ] && lib="EG_LIB=$PWD/scratch/libegonet_$v.so"
  env $lib timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-e2e --out gpurun_out/tl2_${cfg}_$v.json > /dev/null 2>> gpurun_out/tl2.err
  python -c "import json; d=json.load(open('gpurun_out/tl2_${cfg}_$v.json')); r=d['roofline']; print('$cfg', '$v', round(d['minibatches_per_s']), round(r['frac'],3), round(r['sample_chain_ms_per_launch'],4))"
done; done
