#!/bin/bash
# Pipeline shape sweep on the current kernels (C4 and C2, N=1): lanes x bundle.
D=gpurun_out/r02shape; mkdir -p $D
for cfg in C4 C2; do
  for shape in "4 16" "6 16" "8 16" "8 8" "12 8"; do
    set -- $shape
    timeout 300 python bench.py --config $cfg --depth $1 --bundle $2 --steps 32 --warmup 8 --no-e2e --no-cpu-baseline \
        --out $D/${cfg}_d$1_b$2.json > /dev/null 2> $D/${cfg}_d$1_b$2.err
    python -c "import json;d=json.load(open('$D/${cfg}_d$1_b$2.json'));print('$cfg d$1 b$2', round(d['minibatches_per_s']), round(d['roofline']['frac'],3))" 2>/dev/null || echo "$cfg d$1 b$2 failed"
  done
done
