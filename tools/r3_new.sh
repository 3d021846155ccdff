cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/n2
L=paper_2502_06766_b200/_lib
TKV_LIB_PATH=$L/lib_new.so timeout 600 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_sharded_device.py -x -q > gpurun_out/n2/tests.txt 2>&1
for rep in 1 2; do for lib in libtkv.so lib_new.so; do for c in cfg1 cfg2; do
  TKV_LIB_PATH=$L/$lib python tools/scan_ab.py --config $c --steps 100 --label $lib; done; done; done > gpurun_out/n2/ab.txt 2>&1
for c in cfg1 cfg2; do echo "== $c"; TKV_LIB_PATH=$L/lib_new_diag.so python tools/timeline.py --config $c --graph; done > gpurun_out/n2/timeline.txt 2>&1
