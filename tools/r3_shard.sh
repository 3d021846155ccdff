cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/h
L=paper_2502_06766_b200/_lib
export TKV_LIB_PATH=$L/libtkv_diag.so
TKV_SHARD_CLUS=1 timeout 900 python -m pytest tests/test_gpu_sharded_device.py tests/test_gpu_parity.py -x -q -k "shard or Shard" > gpurun_out/h/tests.txt 2>&1
for v in 0 1; do echo "== TKV_SHARD_CLUS=$v"; TKV_SHARD_CLUS=$v python tools/shard_stage.py; done > gpurun_out/h/stage.txt 2>&1
unset TKV_LIB_PATH
for rep in 1 2; do python tools/scan_ab.py --config cfg5 --steps 20; done > gpurun_out/h/cfg5.txt 2>&1
