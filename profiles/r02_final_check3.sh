#!/bin/bash
# Round-2 end check on the final tree: smoke, default bench line, ncu launch list of the default
# command (+ per-kernel table), the reference arm (oracle) at small steps.
D=gpurun_out/${1:-r02end3}; mkdir -p $D
timeout 1800 python -m pytest tests -m gpu -q --timeout 300 > $D/pytest_gpu.log 2>&1; echo gpu=$?; tail -1 $D/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke(); print('smoke ok')" > $D/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py --out $D/bench.json > $D/bench.out 2> $D/bench.err; echo bench=$?
timeout 900 python bench.py --steps 20 --warmup 5 --out $D/bench_20_5.json > /dev/null 2> $D/bench_20_5.err; echo bench20=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $D/launches_default.csv python bench.py --no-cpu-baseline > $D/ncu_list.log 2>&1; echo ncu=$?
python profiles/launch_table.py $D/launches_default.csv > $D/launches_default_table.txt 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 --out $D/reference.json > $D/reference.out 2> $D/reference.err; echo ref=$?
EG_LIB=$PWD/paper_2112_15345_b200/libegonet_check.so timeout 1800 python -m pytest tests -m gpu -q --timeout 300 \
    > $D/pytest_gpu_checked.log 2>&1; echo checked=$?; tail -1 $D/pytest_gpu_checked.log
