#!/bin/bash
# Fused cluster sample + threshold (small contexts) vs the previous build, then the GPU tests
cd $GRAFT_REPO_ROOT
O=gpurun_out/r4f; mkdir -p $O
timeout 600 bash tools/ab_libs.sh "cfg1 cfg2 cfg3" exp/libtkv_small3.so exp/libtkv_fused.so > $O/ab.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/tests.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
