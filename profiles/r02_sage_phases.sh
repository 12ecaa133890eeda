#!/bin/bash
# SAGE layer on C4: phase costs of the round-1 kernel (builds with phases compiled out,
# EG_SAGE_SKIP bits: 1 neighbour rows, 2 self rows, 4 MMA + its wait, 8 epilogue, 16 W
# staging; timing only, outputs wrong), then the flattened A build (sflat): parity + timing.
D=gpurun_out/r02sagep; mkdir -p $D
EG_LIB=$PWD/paper_2112_15345_b200/libegonet_sflat.so timeout 600 python -m pytest tests/test_gpu_sage.py -q --timeout 300 \
    > $D/pytest_sflat.log 2>&1; echo "sflat tests rc=$?"; tail -1 $D/pytest_sflat.log
for v in base sflat sk1 sk3 sk4 sk12 sk16 sk31; do
  EG_LIB=$PWD/paper_2112_15345_b200/libegonet_$v.so timeout 300 python profiles/sage_bench.py --config C4 --reps 20 --batches 4 \
      > $D/sage_$v.json 2> $D/sage_$v.err
  python -c "import json;d=json.load(open('$D/sage_$v.json'));print('$v', d['median_us'])" || echo "$v failed"
done
for cfg in C3 C2; do for v in base sflat; do
  EG_LIB=$PWD/paper_2112_15345_b200/libegonet_$v.so timeout 300 python profiles/sage_bench.py --config $cfg --reps 20 --batches 4 \
      > $D/sage_${cfg}_$v.json 2> $D/sage_${cfg}_$v.err
  python -c "import json;d=json.load(open('$D/sage_${cfg}_$v.json'));print('$cfg $v', d['median_us'])" || echo "$cfg $v failed"
done; done
