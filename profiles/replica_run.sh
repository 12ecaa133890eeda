#!/bin/bash
# Replicated small feature types (institution, field) at N = 2: parity (multi-process,
# both policies) and the bench with / without replicas; the new GPU tests on one GPU.
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "replica" > gpurun_out/pytest_replica.log 2>&1; echo pytest=$?
timeout 900 $R --nproc-per-node 2 --master-port 29601 tests/dist_gpu_parity.py --config C2 --batches 2 \
    > gpurun_out/dist_c2_n2_rep.log 2>&1; echo dist_c2_n2=$?; tail -1 gpurun_out/dist_c2_n2_rep.log
for rep in none auto; do
  timeout 600 $R --nproc-per-node 2 --master-port 2961${#rep} bench.py --gpus 2 --replicate $rep --out gpurun_out/bench_n2_$rep.json \
      > gpurun_out/bench_n2_$rep.log 2>&1; echo bench_$rep=$?
  python -c "import json; d=json.load(open('gpurun_out/bench_n2_$rep.json')); r=d['roofline']; print('$rep', round(d['minibatches_per_s']), 'b/s', round(d['value']/1e9,3), 'Gedge/s', r['bound'], round(r['achieved']), round(r['frac'],3), r.get('remote_row_fraction'), d['config'].get('feature_replicas'))"
done
