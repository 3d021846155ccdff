cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/mp2
L=paper_2502_06766_b200/_lib
timeout 900 python -m pytest tests/test_gpu_sharded_device.py tests/test_gpu_parity.py -x -q > gpurun_out/mp2/tests.txt 2>&1
python tools/shard_stage.py > gpurun_out/mp2/stage.jsonl 2>&1
TKV_LIB_PATH=$L/libtkv_diag.so python tools/shard_stage.py --shards 8 --phases > gpurun_out/mp2/phases.txt 2>&1
