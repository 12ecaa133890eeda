#!/bin/bash
# k_select register budget: launch_bounds(256,4) (64 regs, 76 B spill; default) vs (256,3) (80 regs)
for cfg in C2 C3 C4; do for v in base sel3 base sel3; do
  lib=""; [ $v != base ] && lib="EG_LIB=$PWD/scratch/libegonet_$v.so"
  env $lib timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-e2e --out gpurun_out/sr_${cfg}_$v.json > /dev/null 2>> gpurun_out/sr.err
  python -c "import json; d=json.load(open('gpurun_out/sr_${cfg}_$v.json')); r=d['roofline']; print('$cfg', '$v', round(d['minibatches_per_s']), round(r['sample_chain_ms_per_launch'],4))"
done; done
