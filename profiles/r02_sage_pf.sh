#!/bin/bash
D=gpurun_out/r02sage_tr; mkdir -p $D
EG_LIB=$PWD/paper_2112_15345_b200/libegonet_spftr.so timeout 300 python profiles/sage_bench.py --config C4 --reps 3 --batches 2 --trace \
    > $D/trace_c4_pf.json 2> $D/trace_c4_pf.txt; echo trace=$?
grep trace_cta $D/trace_c4_pf.txt
bash profiles/r02_sage_ab.sh pf spf
