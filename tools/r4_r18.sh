#!/bin/bash
# half-size sample up to 2^17 rows (r17, current) vs up to 2^18 rows (r18: takes in cfg5)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r4r; mkdir -p $O
timeout 900 bash tools/ab_libs.sh "cfg5" exp/libtkv_r17.so exp/libtkv_r18.so > $O/ab.txt 2>&1
