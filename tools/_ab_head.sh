timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 120 -k "decoder or host" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
timeout 300 python tools/e2e_probe.py 2>&1 | head -3
python bench.py 2>/dev/null | tail -1 > gpurun_out/bench.json; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['step_roofline']['frac'])"
