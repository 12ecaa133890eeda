#!/bin/bash
# ncu captures used for profiles/ (run under gpurun on one B200; see B200_PROFILING.md).
# 1) launch list (per-kernel device time, serialised / cold-cache: compare shares)
# 2) --set full of the gather kernel and the sampling kernel of hop 1
set -e
B="python bench.py --steps 6 --warmup 2 --depth 1 --bundle 8 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gather_ldg -s 2 -c 1 -o gpurun_out/prof_gather $B \
    > gpurun_out/ncu_gather.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sample -s 5 -c 1 -o gpurun_out/prof_ksample $B \
    > gpurun_out/ncu_ksample.log 2>&1
