#!/bin/bash
# Full bench lines per config.  usage: bash profiles/results_run.sh N "C1 C2 ..."
N=${1:-1}; CFGS=${2:-"C1 C2 C3 C4"}
mkdir -p gpurun_out/results
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node $N"
for C in $CFGS; do
  o=gpurun_out/results/${C}_n$N.json
  if [ $N = 1 ]; then timeout 900 python bench.py --config $C --out $o > gpurun_out/results/${C}_n$N.log 2>&1
  else timeout 900 $R --master-port $((29700 + N * 100 + RANDOM % 90)) bench.py --gpus $N --config $C --no-cpu-baseline --out $o \
      > gpurun_out/results/${C}_n$N.log 2>&1; fi
  echo "$C n$N rc=$?"
  python -c "
import json; d=json.load(open('$o')); r=d['roofline']; e=d.get('e2e') or {}; c=d.get('cpu_baseline') or {}
print('$C', 'N=$N', round(d['minibatches_per_s']), 'b/s', round(d['value']/1e9,3), 'Gedge/s', 'gather', round(d.get('gather_GBps',0)), 'GB/s', r['bound'], round(r['frac'],3), 'e2e', round(e.get('value',0)/1e9,3), 'cpu', c.get('value'), c.get('unit'))" 2>/dev/null
done
