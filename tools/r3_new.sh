cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/n3
L=paper_2502_06766_b200/_lib
for rep in 1 2; do for lib in libtkv.so lib_cores.so; do for c in cfg1 cfg2; do
  TKV_LIB_PATH=$L/$lib python tools/scan_ab.py --config $c --steps 100 --label $lib; done; done; done > gpurun_out/n3/ab.txt 2>&1
for lib in libtkv_diag.so lib_cores_diag.so; do for c in cfg1 cfg2; do echo "== $c $lib"; TKV_LIB_PATH=$L/$lib python tools/timeline.py --config $c --graph; done; done > gpurun_out/n3/timeline.txt 2>&1
