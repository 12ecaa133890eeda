#!/bin/bash
# Round 2 check: the new GPU tests first, then the whole GPU suite, then the default bench line.
mkdir -p gpurun_out/r02b
timeout 1500 python -m pytest tests/test_gpu_coverage.py -x -q > gpurun_out/r02b/pytest_cov.log 2>&1; echo cov=$?
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02b/pytest_gpu.log 2>&1; echo gpu=$?
timeout 900 python bench.py --out gpurun_out/r02b/bench.json > gpurun_out/r02b/bench.out 2> gpurun_out/r02b/bench.err; echo bench=$?
timeout 900 python bench.py --steps 20 --warmup 5 --out gpurun_out/r02b/bench_20_5.json > /dev/null 2> gpurun_out/r02b/bench_20_5.err; echo bench20=$?
