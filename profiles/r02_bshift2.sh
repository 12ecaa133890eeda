#!/bin/bash
# Bucket width x big-bucket threshold (task elements T, sort-path limit B; T + B <= 256) on C4.
D=gpurun_out/r02bshift2; mkdir -p $D
L=$PWD/paper_2112_15345_b200
for rep in 1 2; do
  for cfgv in "13 base" "13 t192b64" "13 t128b128" "13 t96b160" "12 t128b128" "11 base"; do
    set -- $cfgv
    EG_BSHIFT=$1 EG_LIB=$L/libegonet_$2.so timeout 300 python bench.py --steps 32 --warmup 8 --no-e2e --no-cpu-baseline \
        --out $D/c4_b$1_$2_$rep.json > /dev/null 2> $D/c4_b$1_$2_$rep.err
    python -c "import json;d=json.load(open('$D/c4_b$1_$2_$rep.json'));print('C4 bshift $1 $2 rep $rep', round(d['minibatches_per_s']))" || echo "b$1 $2 failed"
  done
done
