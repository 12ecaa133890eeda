#!/bin/bash
# Multi-process parity (N=2) in the bench's 4 x 16 pipelined launch shape: C2 and C4.
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
mkdir -p gpurun_out/dp
for C in C2 C4; do
  timeout 600 $R --master-port $((29650 + RANDOM % 100)) tests/dist_gpu_parity.py --config $C --batches 2 --depth 4 --bundle 16 \
    > gpurun_out/dp/${C}_n2_4x16.log 2>&1; echo $C=$?; tail -1 gpurun_out/dp/${C}_n2_4x16.log
done
