#!/bin/bash
D=gpurun_out/r02sage; mkdir -p $D
for k in sage_gemm sage_aggregate; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 2 --launch-count 1 \
      -o $D/ncu_$k python profiles/sage_bench.py --config C4 --reps 3 --batches 2 > $D/ncu_$k.log 2>&1; echo $k=$?
done
