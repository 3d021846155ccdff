cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/c4
python tools/bench_cfg4.py --steps 10 > gpurun_out/c4/cfg4_t1.json 2>&1
python tools/bench_cfg4.py --steps 20 --tp-shard 8 > gpurun_out/c4/cfg4_tp8.json 2>&1
python tools/bench_cfg4.py --steps 20 --tp-shard 2 > gpurun_out/c4/cfg4_tp2.json 2>&1
