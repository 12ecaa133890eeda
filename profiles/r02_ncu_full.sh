#!/bin/bash
# ncu --set full captures of single kernels of the default C4 launch (level / hop chosen by
# the launch skip: occurrence o of a kernel that runs k times per launch -> skip 8k + o).
D=gpurun_out/${1:-r02h}; mkdir -p $D
B="python bench.py --config C4 --steps 4 --warmup 8 --no-e2e --no-cpu-baseline"
shift
for spec in "$@"; do
  name=${spec%%:*}; skip=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$name" --launch-skip $skip --launch-count 1 \
      -o $D/ncu_${name}_${skip} $B > $D/ncu_${name}_${skip}.log 2>&1
  echo "$name $skip rc=$?"
done
