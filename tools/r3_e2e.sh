cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/e
for c in cfg3 cfg2 cfg1; do python bench.py --config $c --steps 50 --no-cpu-baseline > gpurun_out/e/bench_$c.json 2>&1; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/e/tests.txt 2>&1
