#!/bin/bash
# gather4 with padded groups (C3: 400-B rows) -- parity + bench vs LDG
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c3 or c1 or c2_full or c4_full or bench or minibatch" > gpurun_out/pytest_tc3.log 2>&1; echo pytest=$?
EG_GATHER=tma timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "world or replica" > gpurun_out/pytest_tc3w.log 2>&1; echo pytest_world_tma=$?
for m in auto ldg; do
  EG_GATHER=$m timeout 600 python bench.py --config C3 --no-cpu-baseline --no-e2e --out gpurun_out/tc3_$m.json > /dev/null 2>> gpurun_out/tc3.err
  python -c "import json; d=json.load(open('gpurun_out/tc3_$m.json')); r=d['roofline']; print('C3', '$m', round(d['minibatches_per_s']), r['kernel'], round(r['frac'],3), round(r['gather_ms_per_launch'],4), round(r['sample_chain_ms_per_launch'],4))"
done
