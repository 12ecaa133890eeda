bash profiles/ab_run.sh tiny64 C2 C3 C4 > gpurun_out/ab_tiny64.txt 2>&1
for pr in none gather; do for i in 1 2; do
EG_PRIO=$pr python bench.py --config C1 --no-cpu-baseline --no-e2e --out gpurun_out/c1_$pr$i.json > /dev/null 2>&1
python -c "import json; d=json.load(open('gpurun_out/c1_$pr$i.json')); print('C1', '$pr', round(d['minibatches_per_s']), d['host_us_per_batch'])" >> gpurun_out/ab_tiny64.txt
done; done
