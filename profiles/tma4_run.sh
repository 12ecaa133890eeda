#!/bin/bash
# gather4 TMA gather: parity under every gather mode, then the bench A/B vs the LDG gather
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_tma4_auto.log 2>&1; echo pytest_auto=$?
for m in ldg tma; do
  EG_GATHER=$m timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lp.py -m gpu -x -q \
     -k "c2_full or c4_full or c3_full or world or minibatch or replica or bundle or bench" > gpurun_out/pytest_tma4_$m.log 2>&1; echo pytest_$m=$?
done
for cfg in C2 C4 C1; do for m in auto ldg; do
  EG_GATHER=$m timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-e2e --out gpurun_out/t4_${cfg}_$m.json > /dev/null 2>> gpurun_out/t4.err
  python -c "import json; d=json.load(open('gpurun_out/t4_${cfg}_$m.json')); r=d['roofline']; print('$cfg', '$m', round(d['minibatches_per_s']), round(r['frac'],3), round(r['gather_ms_per_launch'],4), round(r['sample_chain_ms_per_launch'],4))"
done; done
