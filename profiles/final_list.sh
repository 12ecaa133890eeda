#!/bin/bash
timeout 600 python bench.py > gpurun_out/bench_default2.json 2> gpurun_out/bench_default2.err; echo bench=$?
bash profiles/run_ncu.sh list; echo list=$?
