timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
TKV_HEAD_TOPK=1 timeout 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_scan_tc.py -x -q -m gpu 2>&1 | tail -2
for c in cfg1 cfg2 cfg3; do
  for h in 0 1; do TKV_HEAD_TOPK=$h timeout 120 python tools/scan_ab.py --config $c --steps 100 --label head$h 2>&1 | tail -1; done
done
