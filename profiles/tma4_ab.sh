#!/bin/bash
# TMA gather: CTAs per SM A/B + one ncu --set full of the TMA gather (C2)
for cfg in C2 C4; do for n in 2 3; do
  EG_TMA_CTAS=$n timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-e2e --out gpurun_out/t4ab_${cfg}_$n.json > /dev/null 2>> gpurun_out/t4ab.err
  python -c "import json; d=json.load(open('gpurun_out/t4ab_${cfg}_$n.json')); r=d['roofline']; print('$cfg', 'ctas=$n', round(d['minibatches_per_s']), round(r['frac'],3), round(r['gather_ms_per_launch'],4), round(r['sample_chain_ms_per_launch'],4))"
done; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gather_tma" -s 2 -c 1 -o gpurun_out/prof_tma4 \
  python bench.py --steps 16 --warmup 16 --no-e2e --no-cpu-baseline > gpurun_out/ncu_tma4.log 2>&1; echo ncu=$?
