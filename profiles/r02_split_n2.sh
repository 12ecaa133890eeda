#!/bin/bash
# N=2: full path vs sampling + compaction alone (--diag-no-gather), C4 / C3.
D=gpurun_out/r02split2; mkdir -p $D
for cfg in C4 C3; do
  for mode in full nogather; do
    X=""; [ $mode = nogather ] && X="--diag-no-gather"
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port $((29600 + RANDOM % 300)) bench.py --gpus 2 --config $cfg --steps 32 --warmup 8 --no-e2e $X \
      --out $D/${cfg}_$mode.json > $D/${cfg}_$mode.log 2>&1
    python -c "import json;d=json.load(open('$D/${cfg}_$mode.json'));r=d['roofline'];print('$cfg N=2 $mode', round(d['minibatches_per_s']), round(d['ms_per_step'],4), round(r['sample_chain_ms_per_launch'],4), round(r['gather_ms_per_launch'],4))" || echo "$cfg $mode failed"
  done
done
