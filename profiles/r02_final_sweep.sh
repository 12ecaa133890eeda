#!/bin/bash
# Round-2 results sweep: N = 1 / 2 / 4, node classification C1-C5 and
# link prediction C2 / C4, default pipeline (4 x 16), --steps 32 --warmup 8, e2e on.
D=gpurun_out/r02final; mkdir -p $D
one() {  # n cfg task
  local n=$1 cfg=$2 task=$3 out=$D/${2}_${3}_n${1}.json
  if [ $n = 1 ]; then
    timeout 600 python bench.py --config $cfg --task $task --steps 32 --warmup 8 --out $out > /dev/null 2> $out.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --config $cfg --task $task --steps 32 --warmup 8 \
      --out $out > $out.log 2>&1
  fi
  python profiles/r02_row.py $out || echo "$cfg $task N=$n failed"
}
for cfg in C1 C2 C3 C4; do one 1 $cfg nc; done
for cfg in C2 C4; do one 1 $cfg lp; done
for n in 2 4; do
  for cfg in C1 C2 C3 C4 C5; do one $n $cfg nc; done
  for cfg in C2 C4; do one $n $cfg lp; done
done
