mkdir -p gpurun_out/fc
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/fc/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/fc/smoke.log
timeout 600 python bench.py > gpurun_out/fc/bench.json 2> gpurun_out/fc/bench.err; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/fc/bench_ref.json 2> gpurun_out/fc/bench_ref.err; echo ref=$?
