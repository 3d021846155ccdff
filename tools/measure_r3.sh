#!/bin/bash
# Round-3 measurement pass (one B200): bench lines for every single-GPU config, the reference
# arm, the sharded per-rank stages, ncu launch lists (each after the same command ran plainly)
# and full captures of the key scan (cfg3) and the cluster k-th + gather kernel (cfg2).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/m3
O=gpurun_out/m3
python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err
python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_cfg3_reference.json 2>&1
for c in cfg1 cfg2; do python bench.py --config $c --steps 100 --no-cpu-baseline > $O/bench_$c.json 2>&1; done
python bench.py --config cfg5 --steps 20 --no-cpu-baseline > $O/bench_cfg5.json 2>&1
python tools/shard_stage.py > $O/shard_stage.jsonl 2>&1
for c in cfg1 cfg2 cfg3; do
  python tools/scan_ab.py --config $c --steps 3 > $O/plain_$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
      -k regex:"stage|sample|threshold|scan_tc|kth|attend|head_topk|clus_topk|sort" \
      --log-file $O/r3_${c}_launches.csv python tools/scan_ab.py --config $c --steps 3 > $O/ncu_$c.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:scan_tc -s 3 -c 1 -o $O/scan_cfg3 \
    python tools/scan_ab.py --config cfg3 --steps 3 > $O/ncu_scan.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:clus_topk -s 3 -c 1 -o $O/clus_cfg2 \
    python tools/scan_ab.py --config cfg2 --steps 3 > $O/ncu_clus.log 2>&1
python tools/k_sweep.py --out $O/ksweep.json > $O/ksweep.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/tests.txt 2>&1
ls $O
