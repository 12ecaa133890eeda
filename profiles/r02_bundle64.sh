#!/bin/bash
# Larger bundles (build variant EG_MAX_BUNDLE=64), N = 1.
D=gpurun_out/r02b64; mkdir -p $D
L=paper_2112_15345_b200/libegonet_b64.so
for cfg in C4 C2 C3; do
  for shape in "4 32" "6 32" "8 32" "2 64" "3 64" "4 64"; do
    set -- $shape
    EG_LIB=$L timeout 300 python bench.py --config $cfg --depth $1 --bundle $2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
        --out $D/${cfg}_d$1_b$2.json > /dev/null 2> $D/${cfg}_d$1_b$2.err
    python -c "import json;d=json.load(open('$D/${cfg}_d$1_b$2.json'));print('$cfg d$1 b$2', round(d['minibatches_per_s']), round(d['roofline']['frac'],3))" 2>/dev/null || echo "$cfg d$1 b$2 failed"
  done
done
