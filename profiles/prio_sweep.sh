set -x
for cfg in C2 C4; do for pr in none gather sample; do
  EG_PRIO=$pr python bench.py --config $cfg --no-cpu-baseline --no-e2e --out gpurun_out/prio_${cfg}_${pr}.json > /dev/null 2>> gpurun_out/prio.err
done; done
python - <<'P'
import json
for cfg in ["C2","C4"]:
  for pr in ["none","gather","sample"]:
    try: d=json.load(open(f"gpurun_out/prio_{cfg}_{pr}.json"))
    except Exception as e: print(cfg,pr,e); continue
    print(cfg,pr,round(d["minibatches_per_s"]),round(d["roofline"]["frac"],3), round(d["roofline"]["gather_ms_per_launch"],4), round(d["roofline"]["sample_chain_ms_per_launch"],4))
P
