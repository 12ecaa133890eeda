#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_sage.py -m gpu -x -q > gpurun_out/pytest_sage.log 2>&1; echo pytest=$? 
for c in C2 C3 C4; do timeout 300 python profiles/sage_bench.py --config $c > gpurun_out/sage_$c.json 2> gpurun_out/sage_$c.err; echo $c=$?
python -c "import json; d=json.load(open('gpurun_out/sage_$c.json')); print('$c', d['median_us'], d['frac_hbm'], d['median_TFLOPs'])"; done
