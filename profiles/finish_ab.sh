#!/bin/bash
# fused relabel+reset (k_finish) vs the previous build, interleaved
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_finish.log 2>&1; echo pytest=$?
for cfg in C2 C3 C4; do for v in prev new prev new; do
  lib=""; [ $v = prev ] && lib="EG_LIB=$PWD/scratch/libegonet_prev.so"
  env $lib timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-e2e --out gpurun_out/fa_${cfg}_$v.json > /dev/null 2>> gpurun_out/fa.err
  python -c "import json; d=json.load(open('gpurun_out/fa_${cfg}_$v.json')); r=d['roofline']; print('$cfg', '$v', round(d['minibatches_per_s']), d['gpu_launches'], round(r['sample_chain_ms_per_launch'],4))"
done; done
