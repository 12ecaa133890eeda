#!/bin/bash
# Per-stage breakdown of a config: EG_TRACE stage stamps (serialised phases) + ncu launch list
# usage: bash profiles/breakdown.sh CFG...
for c in "$@"; do
B="python bench.py --config $c --steps 16 --warmup 16 --no-e2e --no-cpu-baseline"
EG_TRACE=1 $B --out gpurun_out/trace_$c.json > /dev/null 2> gpurun_out/trace_$c.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$c.csv $B > gpurun_out/ncu_list_$c.log 2>&1
done
