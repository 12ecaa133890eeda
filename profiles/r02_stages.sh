#!/bin/bash
# TMA gather ring shape at the final kernels (stages x stage bytes): 4 x 16 KB (base), 3 x 16, 6 x 16, 8 x 8 KB.
D=gpurun_out/r02stages; mkdir -p $D
for cfg in C4; do for rep in 1 2; do for v in base st3 st6 sb8; do
  EG_LIB=$PWD/paper_2112_15345_b200/libegonet_$v.so timeout 300 python bench.py --config $cfg --no-e2e --no-cpu-baseline \
      --out $D/${cfg}_${v}_$rep.json > /dev/null 2> $D/${cfg}_${v}_$rep.err
  python -c "import json;d=json.load(open('$D/${cfg}_${v}_$rep.json'));print('$cfg $v rep $rep', round(d['minibatches_per_s']), round(d['roofline']['frac'],3), d['parity_checked'])" || echo "$cfg $v failed"
done; done; done
