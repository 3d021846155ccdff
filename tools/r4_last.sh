#!/bin/bash
# Last call of round 4 on the committed build: smoke, default bench line, its ncu launch list
cd $GRAFT_REPO_ROOT
O=gpurun_out/r4l; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -x -q > $O/tests.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
  --log-file $O/cfg3_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu.log 2>&1
