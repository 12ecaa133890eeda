#!/bin/bash
# The GPU suite against the bounds-checked build (libegonet_check.so, EG_CHECK device asserts;
# compute-sanitizer is closed on this pool).
mkdir -p gpurun_out/r02chk
python paper_2112_15345_b200/build.py --check > /dev/null
EG_LIB=$PWD/paper_2112_15345_b200/libegonet_check.so timeout 1500 python -m pytest tests -m gpu -q --timeout 300 \
    > gpurun_out/r02chk/pytest_gpu_checked.log 2>&1; echo checked=$?
