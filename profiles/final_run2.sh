#!/bin/bash
# Round-end sweep (gpurun --gpus 4): multi-process parity C2 at world 4 (replicated small
# types, the default) and C5 at world 2, then profiles/final_run.sh.
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p gpurun_out/final
timeout 900 $R --nproc-per-node 4 --master-port 29601 tests/dist_gpu_parity.py --config C2 --batches 2 \
    > gpurun_out/final/dist_c2_n4.log 2>&1; echo dist_c2_n4=$?; tail -1 gpurun_out/final/dist_c2_n4.log
CUDA_VISIBLE_DEVICES=0,1 timeout 1500 $R --nproc-per-node 2 --master-port 29621 tests/dist_gpu_parity.py --config C5 \
    --batches 1 > gpurun_out/final/dist_c5_n2.log 2>&1; echo dist_c5_n2=$?; tail -1 gpurun_out/final/dist_c5_n2.log
bash profiles/final_run.sh
