#!/bin/bash
# "fit" replica policy: GPU parity (one process, world 2) and multi-process parity at N = 4 (C3, C4).
D=gpurun_out/r02repc; mkdir -p $D
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "replicated" --timeout 300 > $D/pytest_rep.log 2>&1; echo pytest=$?
for c in C3 C4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 300)) \
    tests/dist_gpu_parity.py --config $c --batches 2 --depth 2 --bundle 4 --replicate fit > $D/dist_parity_${c}_n4_fit.log 2>&1; echo dist$c=$?
done
