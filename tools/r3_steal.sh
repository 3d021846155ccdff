cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s
L=paper_2502_06766_b200/_lib
for rep in 1 2; do for lib in libtkv.so lib_sc4.so lib_nosteal.so; do for c in cfg1 cfg2 cfg3; do
  TKV_LIB_PATH=$L/$lib python tools/scan_ab.py --config $c --steps 100 --label $lib; done; done; done > gpurun_out/s/ab.txt 2>&1
for lib in libtkv.so lib_sc4.so lib_nosteal.so; do TKV_LIB_PATH=$L/$lib python tools/scan_ab.py --config cfg5 --steps 20 --label $lib; done >> gpurun_out/s/ab.txt 2>&1
for c in cfg3; do echo "== $c"; TKV_LIB_PATH=$L/lib_diag_steal.so python tools/timeline.py --config $c --graph; done > gpurun_out/s/timeline.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s/tests.txt 2>&1
