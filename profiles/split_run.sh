#!/bin/bash
# Diagnostic: throughput of sampling + compaction alone (no gather) vs the full path
for cfg in C2 C3 C4; do
  python bench.py --config $cfg --no-cpu-baseline --no-e2e --diag-no-gather --out gpurun_out/split_${cfg}_nog.json > /dev/null 2>> gpurun_out/split.err
  python -c "import json; d=json.load(open('gpurun_out/split_${cfg}_nog.json')); print('$cfg', 'no-gather', round(d['minibatches_per_s']), d['roofline']['sample_chain_ms_per_launch'])"
done
