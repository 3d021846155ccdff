timeout 1300 python -m pytest tests -x -q -m gpu --timeout 120 > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for c in cfg2 cfg3; do timeout 120 python tools/scan_ab.py --config $c --steps 200 2>&1 | tail -1; done
timeout 120 python tools/timeline.py --config cfg3 2>&1 | head -8
