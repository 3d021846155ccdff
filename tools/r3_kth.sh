cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/kt2
for c in cfg5 cfg3; do python bench.py --config $c --steps 20 --no-cpu-baseline > gpurun_out/kt2/bench_$c.json 2>&1; done
python tools/k_sweep.py --out gpurun_out/kt2/ksweep.json > gpurun_out/kt2/ksweep.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/kt2/tests.txt 2>&1
