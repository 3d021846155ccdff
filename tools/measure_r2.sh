#!/bin/bash
# Round-2 measurement pass (one B200): bench lines for every single-GPU config, the reference
# arm, cfg4 (one GPU and one tp8 / tp2 rank), the sharded per-rank stages, the k sweep, ncu
# launch lists (each after the same command ran plainly) and one full capture of the key scan.
mkdir -p gpurun_out/m
cd "$(dirname "$0")/.."
python bench.py > gpurun_out/m/bench_cfg3.json 2> gpurun_out/m/bench_cfg3.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/m/bench_cfg3_reference.json 2>&1
for c in cfg1 cfg2; do python bench.py --config $c --steps 100 --no-cpu-baseline > gpurun_out/m/bench_$c.json 2>&1; done
python bench.py --config cfg5 --steps 20 --no-cpu-baseline > gpurun_out/m/bench_cfg5.json 2>&1
python tools/bench_cfg4.py --steps 10 > gpurun_out/m/cfg4_t1.json 2>&1
python tools/bench_cfg4.py --steps 20 --tp-shard 8 > gpurun_out/m/cfg4_tp8.json 2>&1
python tools/bench_cfg4.py --steps 20 --tp-shard 2 > gpurun_out/m/cfg4_tp2.json 2>&1
python tools/shard_stage.py > gpurun_out/m/shard_stage.jsonl 2>&1
python tools/k_sweep.py --out gpurun_out/m/ksweep.json > gpurun_out/m/ksweep.log 2>&1
bash tools/ncu_r2.sh > gpurun_out/m/ncu_lists.log 2>&1
cp gpurun_out/r2_cfg*_launches.csv gpurun_out/m/ 2>/dev/null
python tools/scan_ab.py --config cfg3 --steps 3 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:scan_tc -s 3 -c 1 -o gpurun_out/m/scan_cfg3 \
      python tools/scan_ab.py --config cfg3 --steps 3 > gpurun_out/m/ncu_scan.log 2>&1
ls gpurun_out/m
