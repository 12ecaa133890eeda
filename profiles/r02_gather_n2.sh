#!/bin/bash
# N=2 gather variants (the NVLink gather bounds the path at N > 1): CTAs per SM, LDG gather.
D=gpurun_out/r02gn2; mkdir -p $D
run() {  # cfg tag env...
  local cfg=$1 tag=$2; shift 2
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port $((29600 + RANDOM % 300)) bench.py --gpus 2 --config $cfg --steps 32 --warmup 8 --no-e2e \
      --out $D/${cfg}_${tag}.json > $D/${cfg}_${tag}.log 2>&1
  python -c "import json;d=json.load(open('$D/${cfg}_${tag}.json'));r=d['roofline'];print('$cfg N=2 $tag', round(d['minibatches_per_s']), round(r['achieved']), round(r['gather_ms_per_launch'],4))" || echo "$cfg $tag failed"
}
for cfg in C4 C3; do
  run $cfg ctas2 EG_TMA_CTAS=2
  run $cfg ctas3 EG_TMA_CTAS=3
  run $cfg ldg EG_GATHER=ldg
  run $cfg ctas2b EG_TMA_CTAS=2
done
