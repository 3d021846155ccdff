cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/l
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/l/smoke.txt 2>&1
python bench.py > gpurun_out/l/bench.json 2> gpurun_out/l/bench.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/l/bench_reference.json 2>&1
bash tools/r3_cfg4.sh
cp gpurun_out/c4/* gpurun_out/l/ 2>/dev/null
