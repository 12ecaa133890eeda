#!/bin/bash
# Replicated feature partition policy for every type whose table fits the HBM
# budget: C2 (0.99 GB), C3 (0.98 GB), C4 (28.4 GB) at N = 2 and 4, against the sharded (auto) lines.
D=gpurun_out/r02rep; mkdir -p $D
run() {  # n cfg tag rep
  local n=$1 cfg=$2 tag=$3 rep=$4
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --config $cfg --steps 20 --warmup 5 --no-e2e \
      --replicate $rep --out $D/${cfg}_n${n}_${tag}.json > $D/${cfg}_n${n}_${tag}.log 2>&1
  python -c "import json;d=json.load(open('$D/${cfg}_n${n}_${tag}.json'));r=d['roofline'];print('$cfg N=$n $tag', round(d['minibatches_per_s']), round(d['value']/1e9,2), r['bound'], round(r['achieved']), round(r['frac'],3))" || echo "$cfg N=$n $tag failed"
}
run 2 C3 all 0
run 4 C3 all 0
run 4 C3 auto auto
run 2 C2 all 0,1,2,3
run 4 C2 all 0,1,2,3
run 2 C4 all 0
run 4 C4 all 0
