#!/bin/bash
# Pipeline knobs at the final kernels (C4, N=1): lanes, gather CTAs per SM, node priority.
D=gpurun_out/r02knobs; mkdir -p $D
run() { # tag env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 32 --warmup 8 --no-e2e --no-cpu-baseline $EXTRA --out $D/$tag.json > /dev/null 2> $D/$tag.err
  python -c "import json;d=json.load(open('$D/$tag.json'));print('$tag', round(d['minibatches_per_s']), round(d['roofline']['frac'],3))" || echo "$tag failed"
}
for rep in 1 2; do
  EXTRA="" run def_$rep X=1
  EXTRA="--depth 5" run d5_$rep X=1
  EXTRA="--depth 6" run d6_$rep X=1
  EXTRA="" run cta3_$rep EG_TMA_CTAS=3
  EXTRA="" run prio_none_$rep EG_PRIO=none
  EXTRA="" run prio_sample_$rep EG_PRIO=sample
done
