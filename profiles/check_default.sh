#!/bin/bash
# full GPU suite + smoke + the default bench line (as the driver runs them)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_final.log 2>&1; echo pytest=$?
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_final.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench=$?
for c in C3 C4; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_final_$c.json 2>> gpurun_out/bench_final.err; echo bench_$c=$?; done
