#!/bin/bash
# quarter-size sample (1024 rows) for contexts of at most 2^15 rows (t15) vs the current build
cd $GRAFT_REPO_ROOT
O=gpurun_out/r4t; mkdir -p $O
timeout 600 bash tools/ab_libs.sh "cfg1" exp/libtkv_r17.so exp/libtkv_t15.so > $O/ab.txt 2>&1
