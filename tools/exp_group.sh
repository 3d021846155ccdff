for c in cfg1 cfg2; do for g in off on; do python tools/scan_ab.py --config $c --group $g --steps 200; done; done
python tools/scan_ab.py --config cfg3 --steps 100
