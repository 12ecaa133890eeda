#!/bin/bash
# N=2: C2 / C4 at 3x16 vs 4x16, alternating, 2 repeats.
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
mkdir -p gpurun_out/shape_n2
for i in 1 2; do for C in C2 C4; do for s in "3 16" "4 16"; do set -- $s
  o=gpurun_out/shape_n2/${C}_$1x$2_$i.json
  timeout 300 $R --master-port $((29700 + RANDOM % 200)) bench.py --gpus 2 --config $C --depth $1 --bundle $2 --no-cpu-baseline --out $o > /dev/null 2>&1
  python -c "import json; d=json.load(open('$o')); print('$C N=2', '$1x$2', $i, round(d['minibatches_per_s']), round(d['roofline']['frac'],3))" 2>/dev/null || echo "$C $1x$2 failed"
done; done; done | tee gpurun_out/shape_n2/summary.txt
