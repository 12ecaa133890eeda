#!/bin/bash
# Multi-GPU weak scaling on the current kernels (C4, C3, C2) at N = 2 and 4, per-owner gather4
# maps on (default) and off (EG_PEER_MAPS=0) for C3 / C4 at N = 2; dist parity at N = 4.
D=gpurun_out/r02scale; mkdir -p $D
run() {  # n cfg tag [env]
  local n=$1 cfg=$2 tag=$3; shift 3
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --config $cfg --steps 20 --warmup 5 --no-e2e \
      --out $D/${cfg}_n${n}_${tag}.json > $D/${cfg}_n${n}_${tag}.log 2>&1
  python -c "import json;d=json.load(open('$D/${cfg}_n${n}_${tag}.json'));r=d['roofline'];print('$cfg N=$n $tag', round(d['minibatches_per_s']), round(d['value']/1e9,2), r['bound'], round(r['achieved']), round(r['frac'],3))" || echo "$cfg N=$n $tag failed"
}
run 2 C3 maps
run 2 C3 nomaps EG_PEER_MAPS=0
run 2 C4 maps
run 2 C4 nomaps EG_PEER_MAPS=0
run 4 C3 maps
run 4 C4 maps
run 4 C2 maps
run 4 C3 nomaps EG_PEER_MAPS=0
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29597 \
    tests/dist_gpu_parity.py --config C3 --batches 2 --depth 2 --bundle 4 > $D/dist_parity_c3_n4.log 2>&1; echo distc3n4=$?
