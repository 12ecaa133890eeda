#!/bin/bash
# A/B helper: gpu tests + bench lines for the configs given (no e2e / cpu baseline)
# usage: bash profiles/ab_run.sh TAG CFG...
tag=$1; shift
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${tag}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${tag}.log
for cfg in "$@"; do
  python bench.py --config $cfg --no-cpu-baseline --no-e2e --out gpurun_out/ab_${tag}_${cfg}.json > /dev/null 2>> gpurun_out/ab_${tag}.err
done
python - "$tag" "$@" <<'P'
import json, sys
tag = sys.argv[1]
for cfg in sys.argv[2:]:
    try:
        d = json.load(open(f"gpurun_out/ab_{tag}_{cfg}.json"))
        print(tag, cfg, round(d["minibatches_per_s"]), round(d["roofline"]["frac"], 3),
              round(d["roofline"]["gather_ms_per_launch"], 4), round(d["roofline"]["sample_chain_ms_per_launch"], 4))
    except Exception as e:
        print(tag, cfg, "ERR", e)
P
