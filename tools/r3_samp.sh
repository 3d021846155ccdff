cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sa
L=paper_2502_06766_b200/_lib
for rep in 1 2; do for lib in libtkv.so lib_s8k.so; do for c in cfg3 cfg2 cfg5; do
  TKV_LIB_PATH=$L/$lib python tools/scan_ab.py --config $c --steps 50 --label $lib; done; done; done > gpurun_out/sa/ab.txt 2>&1
TKV_LIB_PATH=$L/lib_s8k.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cluster.py -x -q > gpurun_out/sa/tests.txt 2>&1
