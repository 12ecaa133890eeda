#!/bin/bash
# depth (lanes in flight) x bundle (mini-batches per launch) sweep, one B200, N=1.
# usage: bash profiles/pipeline_sweep.sh [config]   (under gpurun)
C=${1:-C2}
for cfg in "1 1" "4 1" "1 8" "2 8" "4 4" "4 8" "8 8" "2 16" "4 16"; do
  set -- $cfg
  timeout 300 python bench.py --config $C --steps 512 --warmup 32 --depth $1 --bundle $2 --no-e2e --no-cpu-baseline \
      --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1 || { echo "depth $1 bundle $2 failed"; continue; }
  python -c "import json; d=json.load(open('gpurun_out/sweep.json')); r=d['roofline']; print('$C depth $1 bundle $2', round(d['ms_per_step']*1e3,1), 'us/batch', round(d['minibatches_per_s']), 'b/s', round(d['value']/1e9,3), 'Gedge/s gather', round(r['achieved']), 'GB/s', round(r['frac'],3), round(r['gather_ms_per_launch']*1e3,1), 'us/launch')"
done
