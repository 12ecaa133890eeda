#!/bin/bash
# Last sanity check of bench.py defaults: C2 link prediction (4 lanes), default C4 20/5 line.
D=gpurun_out/r02last; mkdir -p $D
timeout 600 python bench.py --config C2 --task lp --steps 8 --warmup 3 --no-cpu-baseline --out $D/c2_lp.json > /dev/null 2> $D/c2_lp.err; echo c2lp=$?
python profiles/r02_row.py $D/c2_lp.json
timeout 600 python bench.py --steps 20 --warmup 5 --out $D/c4_20_5.json > /dev/null 2> $D/c4_20_5.err; echo c4=$?
python profiles/r02_row.py $D/c4_20_5.json
