cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/nr
timeout 900 python -m pytest tests/test_gpu_sharded_device.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q > gpurun_out/nr/tests.txt 2>&1
python tools/shard_stage.py > gpurun_out/nr/stage.jsonl 2>&1
