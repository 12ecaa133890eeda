#!/bin/bash
# C4 launch list (per-kernel time + DRAM bytes) and EG_TRACE stage stamps of the current kernels.
D=gpurun_out/${1:-r02d}; mkdir -p $D
B="python bench.py --config C4 --steps 16 --warmup 8 --no-e2e --no-cpu-baseline"
EG_TRACE=1 timeout 300 $B --out $D/c4_trace.json > /dev/null 2> $D/c4_trace.err
timeout 300 $B --out $D/c4_plain.json > /dev/null 2> $D/c4_plain.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size --clock-control none --csv \
    --log-file $D/launches_c4.csv python bench.py --config C4 --steps 4 --warmup 4 --no-e2e --no-cpu-baseline > $D/ncu_list.log 2>&1
