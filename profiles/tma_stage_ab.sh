#!/bin/bash
# TMA gather ring shape: 4 x 16 KB (default) vs 3 x 32 KB vs 6 x 8 KB stages per CTA (2 CTAs/SM)
for cfg in C2 C4; do for v in base s32k3 s8k6; do
  lib=""; [ $v != base ] && lib="EG_LIB=$PWD/scratch/libegonet_$v.so"
  env $lib timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-e2e --out gpurun_out/tsa_${cfg}_$v.json > /dev/null 2>> gpurun_out/tsa.err
  python -c "import json; d=json.load(open('gpurun_out/tsa_${cfg}_$v.json')); r=d['roofline']; print('$cfg', '$v', round(d['minibatches_per_s']), r['kernel'], round(r['frac'],3), round(r['gather_ms_per_launch'],4), round(r['sample_chain_ms_per_launch'],4))"
done; done
