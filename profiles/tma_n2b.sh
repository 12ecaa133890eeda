#!/bin/bash
# TMA (per-row bulk) vs LDG gather: C3 at N = 1 and 2, C5 at N = 2
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for m in ldg tma; do
  CUDA_VISIBLE_DEVICES=0 EG_GATHER=$m timeout 600 python bench.py --config C3 --no-cpu-baseline --no-e2e --out gpurun_out/tn2b_C3_n1_$m.json > /dev/null 2>&1
  python -c "import json; d=json.load(open('gpurun_out/tn2b_C3_n1_$m.json')); r=d['roofline']; print('C3 N=1', '$m', round(d['minibatches_per_s']), r['kernel'], round(r['frac'],3), round(r['gather_ms_per_launch'],4), round(r['sample_chain_ms_per_launch'],4))"
done
for cfg in C3 C5; do for m in ldg tma; do
  EG_GATHER=$m timeout 900 $R --master-port $((29620 + RANDOM % 50)) bench.py --gpus 2 --config $cfg --no-cpu-baseline --no-e2e --out gpurun_out/tn2b_${cfg}_$m.json > gpurun_out/tn2b_${cfg}_$m.log 2>&1
  python -c "import json; d=json.load(open('gpurun_out/tn2b_${cfg}_$m.json')); r=d['roofline']; print('$cfg N=2', '$m', round(d['minibatches_per_s']), r['kernel'], round(r['frac'],3), round(r['gather_ms_per_launch'],4), round(r['sample_chain_ms_per_launch'],4))"
done; done
