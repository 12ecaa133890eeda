#!/bin/bash
# SAGE kernel-only durations (ncu gpu__time_duration, warm = --cache-control none, cold = all)
# for the round-1 kernel, the flattened A build and the phase-skipping builds (C4).
D=gpurun_out/r02sagen; mkdir -p $D
for v in base sflat sk12 sk31; do
  for cc in none all; do
    EG_LIB=$PWD/paper_2112_15345_b200/libegonet_$v.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --cache-control $cc -k regex:sage --csv --log-file $D/sage_${v}_$cc.csv \
        python profiles/sage_bench.py --config C4 --reps 5 --batches 2 > $D/sage_${v}_$cc.log 2>&1
    python - <<PY
import csv
rows=[r for r in csv.reader(open("$D/sage_${v}_$cc.csv")) if len(r)>10]
h=rows[0]; iv=h.index("Metric Value"); im=h.index("Metric Name")
t=[float(r[iv].replace(',','')) for r in rows[1:] if r[im]=="gpu__time_duration.sum"]
t=sorted(t); print("$v $cc", "n=%d"%len(t), "median %.1f us"%(t[len(t)//2]/1e3 if t[0]>1000 else t[len(t)//2]), "min %.1f"%(t[0]/1e3 if t[0]>1000 else t[0]))
PY
  done
done
