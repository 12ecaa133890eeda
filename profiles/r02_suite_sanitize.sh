#!/bin/bash
# The whole GPU suite on the current kernels, then compute-sanitizer over the small workload.
mkdir -p gpurun_out/r02s
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r02s/pytest_gpu.log 2>&1; echo gpu=$?
bash profiles/sanitize/run.sh
