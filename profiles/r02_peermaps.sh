#!/bin/bash
# per-owner gather4 maps over peer shards: correctness (1 GPU, emulated worlds) + C3 / C4 N=1 lines
bash profiles/r02_compact_check.sh
D=gpurun_out/r02pm; mkdir -p $D
timeout 300 python bench.py --config C3 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --out $D/c3_n1.json > /dev/null 2> $D/c3_n1.err
python -c "import json;d=json.load(open('$D/c3_n1.json'));print('C3 N=1', round(d['minibatches_per_s']), round(d['value']/1e9,2))"
