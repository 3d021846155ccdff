cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/v
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v/tests.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v/smoke.txt 2>&1
for c in cfg1 cfg2; do python bench.py --config $c --steps 100 --no-cpu-baseline > gpurun_out/v/bench_$c.json 2>&1; done
