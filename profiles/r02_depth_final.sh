#!/bin/bash
# Depth 6 default: N = 1 lines (32/8 and 20/5) against depth 4, C4 N = 2 / 4 lines at the new
# default (e2e on), C3 N = 1 / 2 check, bundle duplicate probe.
D=gpurun_out/r02dfin; mkdir -p $D
for rep in 1 2; do
  for dp in 6 4; do
    timeout 600 python bench.py --depth $dp --no-cpu-baseline --out $D/c4_n1_d${dp}_$rep.json > /dev/null 2> $D/c4_n1_d${dp}_$rep.err
    python -c "import json;d=json.load(open('$D/c4_n1_d${dp}_$rep.json'));print('C4 N=1 32/8 depth $dp', round(d['minibatches_per_s']), d['parity_checked'])"
    timeout 600 python bench.py --depth $dp --steps 20 --warmup 5 --no-cpu-baseline --parity 0 --out $D/c4_n1_20_d${dp}_$rep.json > /dev/null 2> $D/c4_n1_20_d${dp}_$rep.err
    python -c "import json;d=json.load(open('$D/c4_n1_20_d${dp}_$rep.json'));print('C4 N=1 20/5 depth $dp', round(d['minibatches_per_s']))"
  done
done
timeout 600 python bench.py --out $D/C4_nc_n1.json > /dev/null 2> $D/C4_nc_n1.err; python profiles/r02_row.py $D/C4_nc_n1.json
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --steps 32 --warmup 8 --out $D/C4_nc_n$n.json > $D/C4_nc_n$n.log 2>&1
  python profiles/r02_row.py $D/C4_nc_n$n.json
done
timeout 600 python bench.py --config C3 --depth 6 --no-cpu-baseline --out $D/c3_n1_d6.json > /dev/null 2>&1
python -c "import json;d=json.load(open('$D/c3_n1_d6.json'));print('C3 N=1 depth 6', round(d['minibatches_per_s']))"
for c in C4 C3 C2; do timeout 600 python profiles/dup_probe.py --config $c > $D/dup_$c.json 2> $D/dup_$c.err; cat $D/dup_$c.json; done
