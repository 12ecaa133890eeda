#!/bin/bash
# NEXT-2: locality-aware partition + seed confinement on planted-community graphs.
# usage (gpurun --gpus 4): bash profiles/locality_run.sh "C2L C4L" "1 2 4"
CFGS=${1:-"C2L C4L"}; NS=${2:-"1 2 4"}
mkdir -p gpurun_out/locality
for C in $CFGS; do for N in $NS; do for CF in "" "--confine"; do
  tag=${C}_n${N}${CF:+_confined}
  o=gpurun_out/locality/$tag.json
  if [ $N = 1 ]; then timeout 900 python bench.py --config $C $CF --no-e2e --no-cpu-baseline --out $o > gpurun_out/locality/$tag.log 2>&1
  else timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node $N \
      --master-port $((29800 + N * 10 + ${#CF})) bench.py --gpus $N --config $C $CF --no-e2e --no-cpu-baseline --out $o \
      > gpurun_out/locality/$tag.log 2>&1; fi
  python -c "
import json; d=json.load(open('$o')); r=d['roofline']
print('$tag', round(d['minibatches_per_s']), 'b/s', round(d['value']/1e9,3), 'Gedge/s', 'inputs/batch', round(d['input_vertices_per_batch_rank0']), 'edges/batch', round(d['sampled_edges_per_batch']), r['bound'], round(r['frac'],3), 'remote', r.get('remote_row_fraction'))" 2>/dev/null || echo "$tag failed"
done; done; done
