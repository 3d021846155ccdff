#!/bin/bash
# N-dependent sample size A/B (base = 4096 samples everywhere, small2 = 2048 up to 2^17 rows with a
# grid sized to the sample), then the GPU test suite on the new build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/x5
timeout 700 bash tools/ab_libs.sh "cfg1 cfg2 cfg3 cfg5" exp/libtkv_base.so exp/libtkv_small2.so > gpurun_out/x5/ab.txt 2>&1
for l in base small2; do echo "== $l"; TKV_LIB_PATH=exp/libtkv_$l.so timeout 300 python tools/shard_stage.py --shards 8; done > gpurun_out/x5/shard.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/x5/tests.txt 2>&1
