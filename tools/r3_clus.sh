cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/c
L=paper_2502_06766_b200/_lib
for lib in libtkv.so lib_pad.so lib_pad_r128.so lib_cl8.so; do for c in cfg1 cfg2 cfg3; do
  TKV_LIB_PATH=$L/$lib python tools/scan_ab.py --config $c --steps 100 --head cluster --label $lib; done; done > gpurun_out/c/ab.txt 2>&1
for lib in libtkv_diag.so lib_diag_pad.so; do for c in cfg2; do echo "== $c $lib"; TKV_LIB_PATH=$L/$lib TKV_CLUS=1 python tools/timeline.py --config $c --graph; done; done > gpurun_out/c/timeline.txt 2>&1
