#!/bin/bash
# C4 per-stage breakdown: EG_TRACE stage stamps (serialised phases) + an ncu launch list
B="python bench.py --config C4 --steps 16 --warmup 16 --no-e2e --no-cpu-baseline"
EG_TRACE=1 $B --out gpurun_out/c4_trace.json > /dev/null 2> gpurun_out/c4_trace.err
$B > gpurun_out/c4_plain.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c4.csv $B > gpurun_out/ncu_list_c4.log 2>&1
