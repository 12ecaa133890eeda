#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over profiles/sanitize/run_small.py
# (C1; default compaction and EG_COMPACT=bitmap).  Logs -> gpurun_out/sanitize/.
mkdir -p gpurun_out/sanitize
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for mode in default bitmap; do
    EG_COMPACT=$mode timeout 1200 $S --tool $tool --error-exitcode 9 --print-limit 50 \
        python profiles/sanitize/run_small.py C1 > gpurun_out/sanitize/${tool}_${mode}.log 2>&1
    echo "$tool $mode rc=$?"
  done
done
