#!/bin/bash
# L2 evict-first hints on the TMA gather's row loads and output stores (EG_TMA_L2_HINT=1) at the
# final kernels: alternating C4 / C2 benches.
D=gpurun_out/r02l2h; mkdir -p $D
for cfg in C4 C2; do for rep in 1 2 3; do for v in base l2h; do
  EG_LIB=$PWD/paper_2112_15345_b200/libegonet_$v.so timeout 300 python bench.py --config $cfg --no-e2e --no-cpu-baseline \
      --out $D/${cfg}_${v}_$rep.json > /dev/null 2> $D/${cfg}_${v}_$rep.err
  python -c "import json;d=json.load(open('$D/${cfg}_${v}_$rep.json'));print('$cfg $v rep $rep', round(d['minibatches_per_s']), round(d['roofline']['frac'],3), d['parity_checked'])" || echo "$cfg $v failed"
done; done; done
