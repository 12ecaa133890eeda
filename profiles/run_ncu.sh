#!/bin/bash
# ncu captures used for profiles/ (run under gpurun on one B200; see B200_PROFILING.md).
# 1) launch list (per-kernel device time, serialised / cold-cache: compare shares)
# 2) --set full of the gather kernel and of the hop-1 sampling / count / emit kernels
set -e
B="python bench.py --steps 8 --warmup 8 --depth 1 --bundle 8 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_select" -s 1 -c 1 \
    -o gpurun_out/prof_full $B > gpurun_out/ncu_full.log 2>&1
