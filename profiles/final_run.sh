#!/bin/bash
# Results sweep for BASELINE.md §4 (gpurun --gpus 4): node classification C1-C5 at
# N = 1, 2, 4; link prediction C2 / C4 at N = 1, 2, 4.
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p gpurun_out/final
run() {   # run N config task extra...
  local N=$1 C=$2 T=$3; shift 3
  local o=gpurun_out/final/${C}_${T}_n$N.json
  if [ $N = 1 ]; then CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --config $C --task $T "$@" --out $o > ${o%.json}.log 2>&1
  else timeout 900 $R --nproc-per-node $N --master-port $((29900 + N * 10 + RANDOM % 9)) bench.py --gpus $N --config $C \
      --task $T --no-cpu-baseline "$@" --out $o > ${o%.json}.log 2>&1; fi
  python -c "
import json; d=json.load(open('$o')); r=d['roofline']; e=d.get('e2e') or {}; c=d.get('cpu_baseline') or {}
print('$C $T N=$N', round(d['minibatches_per_s']), 'b/s', round(d['value']/1e9,3), 'Gedge/s', r['bound'], round(r['achieved']), round(r['frac'],3), 'e2e', round(e.get('value',0)/1e9,3), 'cpu', c.get('value'))" 2>/dev/null || echo "$C $T N=$N failed"
}
for C in C1 C2 C3 C4; do run 1 $C nc; done
for C in C2 C4; do run 1 $C lp; done
for N in 2 4; do for C in C1 C2 C3 C4 C5; do run $N $C nc; done; for C in C2 C4; do run $N $C lp; done; done
