#!/bin/bash
# SAGE layer variants (EG_LIB=libegonet_<v>.so): parity (tests/test_gpu_sage.py), then
# kernel-only durations under ncu (warm: --cache-control none; cold: all) and event timings,
# C4 / C3 / C2 input layers.   usage: r02_sage_ab.sh TAG v1 [v2 ...]
T=$1; shift
D=gpurun_out/r02sage_$T; mkdir -p $D
for v in "$@"; do
  EG_LIB=$PWD/paper_2112_15345_b200/libegonet_$v.so timeout 600 python -m pytest tests/test_gpu_sage.py -q --timeout 300 \
      > $D/pytest_$v.log 2>&1; echo "tests $v rc=$?"; tail -1 $D/pytest_$v.log
done
for cfg in C4 C3 C2; do
for v in base "$@"; do
  for cc in none all; do
    EG_LIB=$PWD/paper_2112_15345_b200/libegonet_$v.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --cache-control $cc -k regex:sage --csv --log-file $D/${cfg}_${v}_$cc.csv \
        python profiles/sage_bench.py --config $cfg --reps 5 --batches 2 > $D/${cfg}_${v}_$cc.log 2>&1
    python - <<PY
import csv
rows=[r for r in csv.reader(open("$D/${cfg}_${v}_$cc.csv")) if len(r)>10]
h=rows[0]; iv=h.index("Metric Value"); im=h.index("Metric Name"); iu=h.index("Metric Unit")
t=sorted(float(r[iv].replace(',',''))*(1e-3 if r[iu]=="nsecond" else 1) for r in rows[1:] if r[im]=="gpu__time_duration.sum")
print("$cfg $v $cc", "n=%d"%len(t), "median %.1f us"%t[len(t)//2], "min %.1f max %.1f"%(t[0],t[-1]))
PY
  done
  EG_LIB=$PWD/paper_2112_15345_b200/libegonet_$v.so timeout 300 python profiles/sage_bench.py --config $cfg --reps 20 --batches 4 \
      > $D/${cfg}_${v}_ev.json 2> $D/${cfg}_${v}_ev.err
  python -c "import json;d=json.load(open('$D/${cfg}_${v}_ev.json'));print('$cfg $v events', d['median_us'])" || echo "$cfg $v failed"
done
done
