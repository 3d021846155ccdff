cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ac
L=paper_2502_06766_b200/_lib
for lib in libtkv.so lib_ac1k.so lib_ac2k.so; do echo "== $lib"; TKV_LIB_PATH=$L/$lib python tools/shard_stage.py; done > gpurun_out/ac/stage.txt 2>&1
TKV_LIB_PATH=$L/lib_ac2k.so timeout 600 python -m pytest tests/test_gpu_sharded_device.py -x -q > gpurun_out/ac/tests.txt 2>&1
