cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/st
L=paper_2502_06766_b200/_lib
TKV_LIB_PATH=$L/lib_st2.so timeout 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py tests/test_gpu_cluster.py -x -q > gpurun_out/st/tests.txt 2>&1
for rep in 1 2; do for lib in libtkv.so lib_st2.so; do for c in cfg2 cfg3 cfg1; do
  TKV_LIB_PATH=$L/$lib python tools/scan_ab.py --config $c --steps 100 --label $lib; done;
  TKV_LIB_PATH=$L/$lib python tools/scan_ab.py --config cfg2 --k 16384 --steps 100 --label $lib; done; done > gpurun_out/st/ab.txt 2>&1
for lib in libtkv_diag.so lib_st2_diag.so; do echo "== cfg2 $lib"; TKV_LIB_PATH=$L/$lib python tools/timeline.py --config cfg2 --graph; done > gpurun_out/st/timeline.txt 2>&1
