#!/bin/bash
# Final round-4 verification on the committed build: GPU tests, smoke, bench lines
cd $GRAFT_REPO_ROOT
O=gpurun_out/r4z; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/tests.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err
for c in cfg1 cfg2; do python bench.py --config $c --steps 100 --no-cpu-baseline > $O/bench_$c.json 2>&1; done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
  --log-file $O/cfg1_launches.csv python bench.py --config cfg1 --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu.log 2>&1
