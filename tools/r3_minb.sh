cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/a
L=paper_2502_06766_b200/_lib
for rep in 1 2; do for lib in libtkv.so lib_minb3.so lib_minb2.so; do for c in cfg3 cfg5; do
  TKV_LIB_PATH=$L/$lib python tools/scan_ab.py --config $c --steps 30 --label $lib; done; done; done > gpurun_out/a/ab.txt 2>&1
