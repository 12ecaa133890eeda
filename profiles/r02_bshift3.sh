#!/bin/bash
# bucket rule <= 2^14: GPU suite + default bench, then C2 / C3 at coarser buckets (EG_BSHIFT).
D=gpurun_out/r02bshift3; mkdir -p $D
timeout 1800 python -m pytest tests -m gpu -q --timeout 300 > $D/pytest_gpu.log 2>&1; echo gpu=$?; tail -1 $D/pytest_gpu.log
timeout 600 python bench.py --out $D/bench.json > /dev/null 2> $D/bench.err; echo bench=$?
python profiles/r02_row.py $D/bench.json
for cfg in C2 C3; do for b in 10 11 12; do
  EG_BSHIFT=$b timeout 300 python bench.py --config $cfg --steps 32 --warmup 8 --no-e2e --no-cpu-baseline --out $D/${cfg}_b$b.json > /dev/null 2> $D/${cfg}_b$b.err
  python -c "import json;d=json.load(open('$D/${cfg}_b$b.json'));print('$cfg bshift $b', round(d['minibatches_per_s']))" || echo "$cfg b$b failed"
done; done
