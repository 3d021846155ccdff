timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for c in cfg1 cfg2 cfg3; do TKV_PDL=1 timeout 120 python tools/scan_ab.py --config $c --steps 100 2>&1 | tail -1; done
timeout 120 python tools/timeline.py --config cfg3 2>&1 | head -8
timeout 300 python tools/e2e_probe.py 2>&1 | head -2
