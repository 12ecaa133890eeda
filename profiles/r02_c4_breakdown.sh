#!/bin/bash
# Round 2, first call: where does a C4 launch's time go (current kernels)?
#   EG_TRACE stage stamps (serialised phases), an ncu launch list with DRAM bytes,
#   and the NVLink metric names this ncu exposes (for the multi-GPU capture later).
mkdir -p gpurun_out/r02a
B="python bench.py --config C4 --steps 64 --warmup 16 --no-e2e --no-cpu-baseline"
( time python -c "import synth; c=synth.config('C4'); synth.build_host_graph(c, materialize_indices=True)" ) > gpurun_out/r02a/hostgraph_time.txt 2>&1
EG_TRACE=1 timeout 600 $B --out gpurun_out/r02a/c4_trace.json > /dev/null 2> gpurun_out/r02a/c4_trace.err
timeout 600 $B --out gpurun_out/r02a/c4_plain.json > /dev/null 2> gpurun_out/r02a/c4_plain.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
    --log-file gpurun_out/r02a/launches_c4.csv python bench.py --config C4 --steps 32 --warmup 16 --no-e2e --no-cpu-baseline > gpurun_out/r02a/ncu_list_c4.log 2>&1
ncu --query-metrics 2>/dev/null | grep -i -E "nvl|nvlrx|nvltx|lts__t_sectors_srcunit_ltcfabric|fabric" > gpurun_out/r02a/ncu_nvlink_metrics.txt
ncu --query-metrics-mode all --query-metrics 2>/dev/null | grep -i -E "nvl" | head -100 > gpurun_out/r02a/ncu_nvlink_metrics_all.txt
nvidia-smi topo -m > gpurun_out/r02a/topo.txt 2>&1
free -g > gpurun_out/r02a/free.txt; nproc >> gpurun_out/r02a/free.txt
