#!/bin/bash
# Multi-GPU checks on one box (gpurun --gpus 4): parity at world 4 (C2) and world 2 (C5,
# 187 GB of features -> 93.5 GB per GPU), then the bench at N = 1, 2, 4.
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $R --nproc-per-node 4 --master-port 29601 tests/dist_gpu_parity.py --config C2 --batches 2 \
    > gpurun_out/dist_c2_n4.log 2>&1; echo dist_c2_n4=$?; tail -1 gpurun_out/dist_c2_n4.log
for n in 1 2 4; do
  if [ $n = 1 ]; then timeout 600 python bench.py --out gpurun_out/bench_n$n.json > gpurun_out/bench_n$n.log 2>&1;
  else timeout 600 $R --nproc-per-node $n --master-port 2961$n bench.py --gpus $n --out gpurun_out/bench_n$n.json \
      > gpurun_out/bench_n$n.log 2>&1; fi
  echo bench_n$n=$?
  python -c "import json; d=json.load(open('gpurun_out/bench_n$n.json')); r=d['roofline']; print($n, round(d['ms_per_step']*1e3,1), 'us/step', round(d['minibatches_per_s']), 'b/s', round(d['value']/1e9,3), 'Gedge/s', r['bound'], round(r['achieved']), round(r['frac'],3), 'e2e', round(d['e2e']['value']/1e9,3) if d.get('e2e') else None)"
done
CUDA_VISIBLE_DEVICES=0,1 timeout 1500 $R --nproc-per-node 2 --master-port 29621 tests/dist_gpu_parity.py --config C5 \
    --batches 1 > gpurun_out/dist_c5_n2.log 2>&1; echo dist_c5_n2=$?; tail -2 gpurun_out/dist_c5_n2.log
timeout 600 $R --nproc-per-node 4 --master-port 29631 profiles/nvlink_sweep.py > gpurun_out/nvlink_sweep_n4.log 2>&1; echo nvlink_n4=$?
grep '^{' gpurun_out/nvlink_sweep_n4.log | tail -1
