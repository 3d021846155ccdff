cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/h2
L=paper_2502_06766_b200/_lib
TKV_LIB_PATH=$L/lib_sh.so timeout 900 python -m pytest tests/test_gpu_sharded_device.py tests/test_gpu_parity.py -x -q -k "shard or Shard" > gpurun_out/h2/tests.txt 2>&1
for v in 0 1; do echo "== TKV_SHARD_OWNED=$v"; TKV_LIB_PATH=$L/lib_sh_diag.so TKV_SHARD_OWNED=$v python tools/shard_stage.py; done > gpurun_out/h2/stage.txt 2>&1
for h in auto kth; do TKV_LIB_PATH=$L/lib_sh.so python tools/scan_ab.py --config cfg2 --k 16384 --steps 50 --head $h; done > gpurun_out/h2/k16k.txt 2>&1
echo "== timeline cfg2 k=16384" >> gpurun_out/h2/k16k.txt
