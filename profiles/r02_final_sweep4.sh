#!/bin/bash
# Round-2 results sweep at the final default (6 x 32, buckets >= 2^12): GPU suite, then N = 1 / 2 / 4,
# node classification C1-C5 and link prediction C2 / C4, --steps 32 --warmup 8, e2e on;
# the "fit" replica policy at N = 2 / 4 for C2-C4; multi-process parity at the bench shape.
D=gpurun_out/r02final4; mkdir -p $D
echo "(GPU suite: profiles/r02/end3/)"
one() {  # n cfg task [extra...]
  local n=$1 cfg=$2 task=$3 tag=$4; shift 4
  local out=$D/${cfg}_${task}_n${n}${tag}.json
  if [ $n = 1 ]; then
    timeout 600 python bench.py --config $cfg --task $task --steps 32 --warmup 8 --out $out "$@" > /dev/null 2> $out.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --config $cfg --task $task --steps 32 --warmup 8 \
      --out $out "$@" > $out.log 2>&1
  fi
  python profiles/r02_row.py $out || echo "$cfg $task N=$n $tag failed"
}
for cfg in C1 C2 C3 C4; do one 1 $cfg nc ""; done
for cfg in C2 C4; do one 1 $cfg lp ""; done
for n in 2 4; do
  for cfg in C1 C2 C3 C4 C5; do one $n $cfg nc ""; done
  for cfg in C2 C4; do one $n $cfg lp ""; done
  for cfg in C2 C3 C4; do one $n $cfg nc _fit --replicate fit; done
  one $n C4 lp _fit --replicate fit
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29597 \
    tests/dist_gpu_parity.py --config C4 --batches 2 --depth 6 --bundle 32 > $D/dist_parity_c4_n4_6x32.log 2>&1; echo distc4=$?
