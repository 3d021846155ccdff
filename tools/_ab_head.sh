timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for c in cfg1 cfg2; do
  for h in 0 1; do TKV_HEAD_TOPK=$h timeout 120 python tools/scan_ab.py --config $c --steps 100 --label head$h 2>&1 | tail -1; done
done
timeout 600 python tools/k_sweep.py --steps 10 2>&1 | tail -8
