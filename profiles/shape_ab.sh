#!/bin/bash
# default pipeline shape 3 x 16 vs 4 x 8 (TMA gather), N = 1 and 2, + parity of both shapes
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bench_launch" > gpurun_out/pytest_shape.log 2>&1; echo pytest=$?
for cfg in C2 C3 C4; do for sh in "4 8" "3 16"; do set -- $sh
  CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --config $cfg --depth $1 --bundle $2 --no-cpu-baseline --no-e2e --out gpurun_out/sh_${cfg}_$1x$2.json > /dev/null 2>> gpurun_out/sh.err
  python -c "import json; d=json.load(open('gpurun_out/sh_${cfg}_$1x$2.json')); r=d['roofline']; print('$cfg N=1', '$1x$2', round(d['minibatches_per_s']), round(r['frac'],3))"
done; done
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --config C2 --task lp --depth 3 --bundle 16 --no-cpu-baseline --no-e2e --out gpurun_out/sh_lp.json > /dev/null 2>> gpurun_out/sh.err
python -c "import json; d=json.load(open('gpurun_out/sh_lp.json')); r=d['roofline']; print('C2 lp N=1 3x16', round(d['minibatches_per_s']), round(r['frac'],3))"
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for cfg in C2 C4; do for sh in "4 8" "3 16"; do set -- $sh
  timeout 900 $R --master-port $((29620 + RANDOM % 50)) bench.py --gpus 2 --config $cfg --depth $1 --bundle $2 --no-cpu-baseline --no-e2e --out gpurun_out/sh2_${cfg}_$1x$2.json > gpurun_out/sh2.log 2>&1
  python -c "import json; d=json.load(open('gpurun_out/sh2_${cfg}_$1x$2.json')); r=d['roofline']; print('$cfg N=2', '$1x$2', round(d['minibatches_per_s']), round(r['frac'],3))"
done; done
