#!/bin/bash
# Is the pipelined path the sum of its parts?  sampling + compaction alone (--diag-no-gather)
# vs the full path, C4 and C2, N=1.
D=gpurun_out/r02split; mkdir -p $D
for cfg in C4 C2; do
  for mode in full nogather; do
    X=""; [ $mode = nogather ] && X="--diag-no-gather"
    timeout 300 python bench.py --config $cfg --steps 32 --warmup 8 --no-e2e --no-cpu-baseline $X --out $D/${cfg}_$mode.json > /dev/null 2> $D/${cfg}_$mode.err
    python -c "import json;d=json.load(open('$D/${cfg}_$mode.json'));print('$cfg $mode', round(d['minibatches_per_s']), round(d['ms_per_step'],4), round(d['roofline']['sample_chain_ms_per_launch'],4), round(d['roofline']['gather_ms_per_launch'],4))" || echo "$cfg $mode failed"
  done
done
