#!/bin/bash
# A/B: gather register budget (102 regs, 2 CTAs/SM) vs launch_bounds(256,3) (80 regs) at 2 and 3 CTAs/SM
for cfg in C2 C3 C4; do
  for v in "base 0" "mb3 2" "mb3 0"; do set -- $v
    lib=""; [ $1 = mb3 ] && lib="EG_LIB=$PWD/scratch/libegonet_mb3.so"
    env $lib EG_GATHER_CTAS=$2 python bench.py --config $cfg --no-cpu-baseline --no-e2e --out gpurun_out/gr_${cfg}_$1_$2.json > /dev/null 2>> gpurun_out/gr.err
    python -c "import json; d=json.load(open('gpurun_out/gr_${cfg}_$1_$2.json')); r=d['roofline']; print('$cfg', '$1 ctas=$2', round(d['minibatches_per_s']), round(r['frac'],3), round(r['gather_ms_per_launch'],4), round(r['sample_chain_ms_per_launch'],4))"
  done
done
