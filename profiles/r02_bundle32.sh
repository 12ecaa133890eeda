#!/bin/bash
# Bundles of 32 (build variant EG_MAX_BUNDLE=32) against the 4 x 16 default, N = 1.
D=gpurun_out/r02b32; mkdir -p $D
for cfg in C4 C2 C3; do
  for shape in "4 16 def" "2 32 b32" "3 32 b32" "4 32 b32" "4 16 b32"; do
    set -- $shape
    if [ $3 = b32 ]; then L=paper_2112_15345_b200/libegonet_b32.so; else L=; fi
    EG_LIB=$L timeout 300 python bench.py --config $cfg --depth $1 --bundle $2 --steps 24 --warmup 6 --no-e2e --no-cpu-baseline \
        --out $D/${cfg}_d$1_b$2_$3.json > /dev/null 2> $D/${cfg}_d$1_b$2_$3.err
    python -c "import json;d=json.load(open('$D/${cfg}_d$1_b$2_$3.json'));print('$cfg d$1 b$2 $3', round(d['minibatches_per_s']), round(d['roofline']['frac'],3), d.get('parity_checked'))" 2>/dev/null || echo "$cfg d$1 b$2 $3 failed"
  done
done
