#!/bin/bash
# A/B of library variants (EG_LIB=libegonet_<v>.so) on C4 and C2 (default shape), alternating
# runs, after the variant's GPU parity tests.  usage: r02_ab2.sh TAG v1 [v2 ...]
T=$1; shift
D=gpurun_out/r02ab_$T; mkdir -p $D
for v in "$@"; do
  EG_LIB=$PWD/paper_2112_15345_b200/libegonet_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lp.py \
      -q --timeout 300 > $D/pytest_$v.log 2>&1; echo "pytest $v rc=$?"; tail -1 $D/pytest_$v.log
done
for cfg in C4 C2; do
for rep in 1 2 3; do
  for v in base "$@"; do
    EG_LIB=$PWD/paper_2112_15345_b200/libegonet_$v.so timeout 300 python bench.py --config $cfg --steps 32 --warmup 8 --no-e2e \
        --no-cpu-baseline --out $D/${cfg}_${v}_$rep.json > /dev/null 2> $D/${cfg}_${v}_$rep.err
    python -c "import json;d=json.load(open('$D/${cfg}_${v}_$rep.json'));print('$cfg $v rep $rep', round(d['minibatches_per_s']), round(d['roofline']['frac'],3))" || echo "$cfg $v failed"
  done
done
done
