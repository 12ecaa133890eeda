#!/bin/bash
# C2 / C4 at the 4 x 16 default, N = 1, 2, 4 (weak scaling).
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p gpurun_out/scale
for N in 1 2 4; do for C in C2 C4; do o=gpurun_out/scale/${C}_n$N.json
  if [ $N = 1 ]; then CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --config $C --no-cpu-baseline --out $o > /dev/null 2>&1
  else timeout 300 $R --nproc-per-node $N --master-port $((29800 + N * 10)) bench.py --gpus $N --config $C --no-cpu-baseline --out $o > /dev/null 2>&1; fi
  python -c "import json; d=json.load(open('$o')); print('$C N=$N', round(d['minibatches_per_s']), round(d['value']/1e9,2), 'Gedge/s', d['roofline']['bound'], round(d['roofline']['frac'],3))" 2>/dev/null || echo "$C N=$N failed"
done; done | tee gpurun_out/scale/summary.txt
