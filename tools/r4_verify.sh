#!/bin/bash
# Round-4 verification on one B200: GPU tests, smoke, bench lines (cfg3 default, cfg1, cfg2, cfg5),
# the G = 8 shard stage, an A/B of the sample-size rule against the previous build, and the ncu
# launch list of the cfg2 bench command.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r4; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/tests.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err
for c in cfg1 cfg2; do python bench.py --config $c --steps 100 --no-cpu-baseline > $O/bench_$c.json 2>&1; done
python bench.py --config cfg5 --steps 20 --no-cpu-baseline > $O/bench_cfg5.json 2>&1
timeout 300 python tools/shard_stage.py --shards 2 4 8 > $O/shard.jsonl 2>&1
[ -f exp/libtkv_base.so ] && timeout 600 bash tools/ab_libs.sh "cfg1 cfg2" exp/libtkv_base.so exp/libtkv_small3.so > $O/ab.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
  --log-file $O/cfg2_launches.csv python bench.py --config cfg2 --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu.log 2>&1
