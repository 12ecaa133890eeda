#!/bin/bash
# Correctness gate of a kernel change: smoke, the parity tests (per-test timeout), a C4 bench line.
mkdir -p gpurun_out/r02c
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 180 > gpurun_out/r02c/pytest_parity.log 2>&1; echo parity=$?
timeout 600 python -m pytest tests/test_gpu_lp.py tests/test_gpu_coverage.py -x -q --timeout 180 > gpurun_out/r02c/pytest_lp_cov.log 2>&1; echo lpcov=$?
timeout 300 python bench.py --steps 20 --warmup 5 --out gpurun_out/r02c/bench.json > /dev/null 2> gpurun_out/r02c/bench.err; echo bench=$?
