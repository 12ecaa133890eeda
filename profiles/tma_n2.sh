#!/bin/bash
# TMA gather (per-row bulk copies from peer shards over NVLink) vs LDG at N = 2
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
EG_GATHER=tma timeout 900 $R --master-port 29611 tests/dist_gpu_parity.py --config C2 --batches 2 > gpurun_out/tn2_dist.log 2>&1; echo dist_tma=$?; tail -1 gpurun_out/tn2_dist.log
for cfg in C2 C4; do for m in ldg tma; do
  EG_GATHER=$m timeout 600 $R --master-port $((29620 + RANDOM % 50)) bench.py --gpus 2 --config $cfg --no-cpu-baseline --no-e2e --out gpurun_out/tn2_${cfg}_$m.json > gpurun_out/tn2_${cfg}_$m.log 2>&1
  python -c "import json; d=json.load(open('gpurun_out/tn2_${cfg}_$m.json')); r=d['roofline']; print('$cfg N=2', '$m', round(d['minibatches_per_s']), r['kernel'], round(r['frac'],3), round(r['gather_ms_per_launch'],4), round(r['sample_chain_ms_per_launch'],4))"
done; done
