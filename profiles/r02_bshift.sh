#!/bin/bash
# Compaction bucket width A/B (EG_BSHIFT, C4 default 11 = 54k buckets): parity at 13, then
# alternating C4 benches at 11 / 12 / 13.
D=gpurun_out/r02bshift; mkdir -p $D
EG_BSHIFT=13 timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -k "C4 or c4 or bench" > $D/pytest_b13.log 2>&1; echo "pytest b13 rc=$?"; tail -1 $D/pytest_b13.log
for rep in 1 2; do
  for b in 11 12 13; do
    EG_BSHIFT=$b timeout 300 python bench.py --steps 32 --warmup 8 --no-e2e --no-cpu-baseline --out $D/c4_b${b}_$rep.json > /dev/null 2> $D/c4_b${b}_$rep.err
    python -c "import json;d=json.load(open('$D/c4_b${b}_$rep.json'));print('C4 bshift $b rep $rep', round(d['minibatches_per_s']), round(d['roofline']['frac'],3))" || echo "b$b failed"
  done
done
EG_BSHIFT=13 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $D/launches_c4_b13.csv python bench.py --steps 4 --warmup 4 --no-e2e --no-cpu-baseline > $D/ncu.log 2>&1; echo ncu=$?
