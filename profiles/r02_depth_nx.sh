#!/bin/bash
# Pipeline depth at N = 2 / 4 (C4, C2 sharded): more launches in flight to hide NVLink latency?
D=gpurun_out/r02depth; mkdir -p $D
run() {  # n cfg depth rep
  local n=$1 cfg=$2 dp=$3 rep=$4 out=$D/${2}_n${1}_d${3}_$4.json
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --config $cfg --depth $dp --steps 32 --warmup 8 --no-e2e \
      --out $out > $out.log 2>&1
  python -c "import json;d=json.load(open('$out'));print('$cfg N=$n depth $dp rep $rep', round(d['minibatches_per_s']), d['clocks'])" || echo "$cfg N=$n d$dp failed"
}
for rep in 1 2; do
  for dp in 4 6 8; do run 2 C4 $dp $rep; done
done
for dp in 4 6; do run 4 C4 $dp 1; done
for dp in 4 6; do run 2 C2 $dp 1; done
