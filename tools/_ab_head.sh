timeout 1300 python -m pytest tests -x -q -m gpu --timeout 120 > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for c in cfg1 cfg2; do for h in 0 1; do TKV_HEAD_TOPK=$h timeout 120 python tools/scan_ab.py --config $c --steps 200 --label head$h 2>&1 | tail -1; done; done
timeout 120 python tools/timeline.py --config cfg1 2>&1 | tail -11
