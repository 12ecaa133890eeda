#!/bin/bash
# ncu captures used for profiles/ (one B200; see B200_PROFILING.md).  ONE ncu per gpurun
# call: bash profiles/run_ncu.sh list | gather | hop
# The bench command is the default one (depth 4 x bundle 8) with few steps; ncu
# serialises the lanes anyway.
#   list    per-kernel device time + DRAM bytes of every launch (cold-cache, serialised:
#           compare shares, not absolutes), after a plain run of the same command
#   gather  --set full of one gather launch
#   hop     --set full of the hop-1 sampling / compaction kernels of one bundle
set -e
B="python bench.py --steps 32 --warmup 32 --no-e2e --no-cpu-baseline"
case "$1" in
  list)
    $B > gpurun_out/plain.log 2>&1
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1 ;;
  gather)
    ncu --set full --clock-control none --import-source on -k regex:"gather_(tma|ldg)" -s 2 -c 1 \
        -o gpurun_out/prof_gather $B > gpurun_out/ncu_gather.log 2>&1 ;;
  hop)
    ncu --set full --clock-control none --import-source on -k regex:"k_select|k_tiny|k_copy|k_emit|k_count" \
        -s 8 -c 5 -o gpurun_out/prof_hop1 $B > gpurun_out/ncu_hop1.log 2>&1 ;;
esac
