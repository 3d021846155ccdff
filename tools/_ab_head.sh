timeout 1300 python -m pytest tests -x -q -m gpu --timeout 120 > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
python bench.py 2>/dev/null | tail -1 > gpurun_out/bench.json; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['step_roofline']['frac'], d['clocks'])"
