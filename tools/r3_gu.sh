cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/gu
L=paper_2502_06766_b200/_lib
for rep in 1 2; do for lib in libtkv.so lib_gu16.so lib_gu12.so; do for c in cfg2 cfg1; do
  TKV_LIB_PATH=$L/$lib python tools/scan_ab.py --config $c --steps 100 --label $lib; done; done; done > gpurun_out/gu/ab.txt 2>&1
