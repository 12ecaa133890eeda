#!/bin/bash
# NVLink counters (ncu, single process driving 2 GPUs) of the gather and the sampling kernels
# of rank 0 of a 2-GPU C4 partition; plus the plain 2-rank bench for context.
D=gpurun_out/r02nv; mkdir -p $D
nvidia-smi topo -m > $D/topo.txt 2>&1
timeout 600 python profiles/nvlink_probe.py --config C4 --check > $D/probe_plain.log 2>&1; echo probe=$?
M=gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none --devices 0 --csv --log-file $D/nvlink_c4.csv \
    python profiles/nvlink_probe.py --config C4 --launches 4 > $D/ncu_probe.log 2>&1; echo ncu=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e --out $D/bench_c4_n2.json > $D/bench_n2.log 2>&1; echo bench2=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
    bench.py --gpus 2 --config C3 --steps 20 --warmup 5 --no-e2e --out $D/bench_c3_n2.json > $D/bench_c3_n2.log 2>&1; echo bench3=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 \
    bench.py --gpus 2 --config C2 --steps 20 --warmup 5 --no-e2e --out $D/bench_c2_n2.json > $D/bench_c2_n2.log 2>&1; echo bench2c2=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29536 \
    tests/dist_gpu_parity.py --config C4 --batches 2 --depth 2 --bundle 4 > $D/dist_parity_c4.log 2>&1; echo distc4=$?
