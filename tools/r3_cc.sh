cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/cc
L=paper_2502_06766_b200/_lib
for rep in 1 2; do for lib in libtkv.so lib_cc2048.so lib_cc512.so; do for c in cfg3 cfg2 cfg5; do
  TKV_LIB_PATH=$L/$lib python tools/scan_ab.py --config $c --steps 30 --label $lib; done; done; done > gpurun_out/cc/ab.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/cc/shard_launches.csv python tools/shard_stage.py --shards 8 --steps 2 > gpurun_out/cc/ncu_shard.log 2>&1
