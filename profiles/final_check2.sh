#!/bin/bash
# Round-end check at the 4 x 16 default: pytest -m gpu, smoke, bench (N=1), launch list.
mkdir -p gpurun_out/fc2
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/fc2/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc2/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/fc2/smoke.log
timeout 600 python bench.py > gpurun_out/fc2/bench.json 2> gpurun_out/fc2/bench.err; echo bench=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fc2/launches.csv \
  python bench.py --steps 64 --warmup 16 --no-cpu-baseline > gpurun_out/fc2/ncu.log 2>&1; echo ncu=$?
