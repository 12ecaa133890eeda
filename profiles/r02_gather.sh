#!/bin/bash
# Gather in the pipelined C4 run: CTAs per SM A/B (EG_TMA_CTAS), then one ncu --set full
# capture of the gather at the default shape (DRAM traffic + duration alone, for bench.py's
# roofline.traffic via profiles/gather_traffic.json).
D=gpurun_out/r02g; mkdir -p $D
for ctas in 2 3 1 2; do
  EG_TMA_CTAS=$ctas timeout 300 python bench.py --steps 32 --warmup 8 --no-e2e --no-cpu-baseline --out $D/ab_ctas$ctas.json > /dev/null 2> $D/ab_ctas$ctas.err
  python -c "import json;d=json.load(open('$D/ab_ctas$ctas.json'));print('ctas $ctas', round(d['minibatches_per_s']), round(d['roofline']['frac'],3), round(d['roofline']['gather_ms_per_launch'],4))"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather_tma_kernel --launch-skip 6 --launch-count 1 \
    -o $D/ncu_gather_c4 python bench.py --steps 4 --warmup 4 --no-e2e --no-cpu-baseline > $D/ncu_gather.log 2>&1; echo ncu=$?
