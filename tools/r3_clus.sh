cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/c
L=paper_2502_06766_b200/_lib
timeout 600 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_cluster.py -x -q > gpurun_out/c/tests_fuzz.txt 2>&1
for c in cfg1 cfg2 cfg3; do python tools/scan_ab.py --config $c --steps 100 --label auto; done > gpurun_out/c/ab.txt 2>&1
for c in cfg2; do echo "== $c auto"; TKV_LIB_PATH=$L/libtkv_diag.so python tools/timeline.py --config $c --graph; done > gpurun_out/c/timeline.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/c/tests.txt 2>&1
