#!/bin/bash
# bucket rule bshift >= 12: GPU suite (incl. EG_BSHIFT overrides) + C1..C4 benches.
D=gpurun_out/r02bshift4; mkdir -p $D
timeout 1800 python -m pytest tests -m gpu -q --timeout 300 > $D/pytest_gpu.log 2>&1; echo gpu=$?; tail -1 $D/pytest_gpu.log
for cfg in C4 C1 C2 C3; do
  timeout 600 python bench.py --config $cfg --out $D/${cfg}.json > /dev/null 2> $D/${cfg}.err; echo $cfg=$?
  python profiles/r02_row.py $D/${cfg}.json
done
EG_BSHIFT=10 timeout 300 python bench.py --config C1 --steps 32 --warmup 8 --no-e2e --no-cpu-baseline --out $D/C1_b10.json > /dev/null 2>&1
python -c "import json;d=json.load(open('$D/C1_b10.json'));print('C1 bshift 10', round(d['minibatches_per_s']))"
