#!/bin/bash
# A/B of library variants (EG_LIB) on the default C4 bench, alternating runs.
D=gpurun_out/r02ab; mkdir -p $D
for rep in 1 2; do
  for v in default "$@"; do
    if [ "$v" = default ]; then L=""; else L="EG_LIB=$PWD/paper_2112_15345_b200/libegonet_$v.so"; fi
    env $L timeout 300 python bench.py --steps 32 --warmup 8 --no-e2e --no-cpu-baseline --out $D/${v}_$rep.json > /dev/null 2> $D/${v}_$rep.err
    python -c "import json;d=json.load(open('$D/${v}_$rep.json'));print('$v rep $rep', round(d['minibatches_per_s']), round(d['roofline']['frac'],3))" || echo "$v failed"
  done
done
