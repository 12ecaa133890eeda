#!/bin/bash
# virtual blocks per relation in count / scan, finer sweep
for cfg in C2 C3 C4; do for v in sb16 sb8 sb4 sb16i16k sb8i16k; do
  lib="EG_LIB=$PWD/scratch/libegonet_$v.so"
  env $lib timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-e2e --out gpurun_out/sb2_${cfg}_$v.json > /dev/null 2>> gpurun_out/sb2.err
  python -c "import json; d=json.load(open('gpurun_out/sb2_${cfg}_$v.json')); r=d['roofline']; print('$cfg', '$v', round(d['minibatches_per_s']), round(r['sample_chain_ms_per_launch'],4))"
done; done
