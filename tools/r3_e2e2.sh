cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/e2
timeout 600 python -m pytest tests -m gpu -x -q -k "decoder or Decoder or host or pinned" > gpurun_out/e2/tests.txt 2>&1
for c in cfg3 cfg2 cfg1; do python bench.py --config $c --steps 100 --no-cpu-baseline > gpurun_out/e2/bench_$c.json 2>&1; done
