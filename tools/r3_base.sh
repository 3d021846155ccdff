cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/b
for c in cfg1 cfg2; do python bench.py --config $c --steps 100 --no-cpu-baseline > gpurun_out/b/bench_$c.json 2>&1; done
export TKV_LIB_PATH=paper_2502_06766_b200/_lib/libtkv_diag.so
for c in cfg1 cfg2; do echo "== $c"; python tools/timeline.py --config $c --graph; done > gpurun_out/b/timeline.txt 2>&1
