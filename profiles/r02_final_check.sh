#!/bin/bash
# Round-2 end check on the final tree: GPU suite, smoke, default bench line (and 20/5), ncu launch list
# of the default bench command.
D=gpurun_out/${1:-r02end}; mkdir -p $D
timeout 1800 python -m pytest tests -m gpu -q --timeout 300 > $D/pytest_gpu.log 2>&1; echo gpu=$?
timeout 300 python -c "import __graft_entry__ as e; e.smoke(); print('smoke ok')" > $D/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py --out $D/bench.json > $D/bench.out 2> $D/bench.err; echo bench=$?
timeout 900 python bench.py --steps 20 --warmup 5 --out $D/bench_20_5.json > /dev/null 2> $D/bench_20_5.err; echo bench20=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $D/launches_default.csv python bench.py --no-cpu-baseline > $D/ncu_list.log 2>&1; echo ncu=$?
