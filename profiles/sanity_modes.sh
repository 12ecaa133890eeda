#!/bin/bash
# sanity: host-memory features (N=1) and planted-community confined seeds (N=2) at the default shape
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --features host --no-cpu-baseline --no-e2e --out gpurun_out/sm_host.json > gpurun_out/sm_host.log 2>&1; echo host=$?
python -c "import json; d=json.load(open('gpurun_out/sm_host.json')); r=d['roofline']; print('C2 host features', round(d['minibatches_per_s']), r['kernel'], r['bound'], round(r['frac'],3))"
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $R --master-port 29655 bench.py --gpus 2 --config C2L --confine --no-cpu-baseline --no-e2e --out gpurun_out/sm_c2l.json > gpurun_out/sm_c2l.log 2>&1; echo c2l=$?
python -c "import json; d=json.load(open('gpurun_out/sm_c2l.json')); r=d['roofline']; print('C2L confined N=2', round(d['minibatches_per_s']), r['kernel'], r['bound'], round(r['frac'],3))"
