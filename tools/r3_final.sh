#!/bin/bash
# Final round-3 evidence for the default bench command: the plain run, then the ncu launch list
# of the same command (per-launch times, cold-cache and serialised; compare shares).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/f
python bench.py > gpurun_out/f/bench.json 2> gpurun_out/f/bench.err && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    -k regex:"stage|sample|threshold|scan_tc|kth|attend|clus_topk|head_topk|sort|append" \
    --log-file gpurun_out/f/r3_bench_cfg3_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/f/ncu.log 2>&1
ls gpurun_out/f
