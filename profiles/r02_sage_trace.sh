#!/bin/bash
# SAGE phase stamps (globaltimer, CTAs 0 and 100) of the staged-epilogue kernel + its parity.
D=gpurun_out/r02sage_tr; mkdir -p $D
#EG_LIB=$PWD/paper_2112_15345_b200/libegonet_sepi.so timeout 600 python -m pytest tests/test_gpu_sage.py -q --timeout 300 \
#    (parity of sepi: 4 passed, previous call)
EG_LIB=$PWD/paper_2112_15345_b200/libegonet_strace.so timeout 300 python profiles/sage_bench.py --config C4 --reps 3 --batches 2 --trace \
    > $D/trace_c4.json 2> $D/trace_c4.txt; echo trace=$?
grep trace_cta $D/trace_c4.txt
