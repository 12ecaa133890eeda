#!/bin/bash
# SAGE layer (NEXT-4 i): parity vs the fp64 oracle, then the C2 / C3 / C4 input-layer timings.
D=gpurun_out/r02sage; mkdir -p $D
timeout 600 python -m pytest tests/test_gpu_sage.py -x -q --timeout 300 > $D/pytest_sage.log 2>&1; echo sage_tests=$?
for cfg in C4 C3 C2; do
  timeout 600 python profiles/sage_bench.py --config $cfg > $D/sage_$cfg.json 2> $D/sage_$cfg.err; echo $cfg=$?
  tail -c 600 $D/sage_$cfg.json
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $D/sage_launches_c4.csv python profiles/sage_bench.py --config C4 --reps 3 --batches 2 > $D/ncu_sage.log 2>&1; echo ncu=$?
