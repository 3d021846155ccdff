cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/v2
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v2/tests.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v2/smoke.txt 2>&1
python bench.py > gpurun_out/v2/bench_cfg3.json 2> gpurun_out/v2/bench_cfg3.err
for c in cfg1 cfg2; do python bench.py --config $c --steps 100 --no-cpu-baseline > gpurun_out/v2/bench_$c.json 2>&1; done
