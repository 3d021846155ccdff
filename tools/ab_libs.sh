#!/bin/bash
# Same-box A/B of alternative builds: bash tools/ab_libs.sh "cfg3 cfg2" lib1.so lib2.so ...
cfgs=$1; shift
for rep in 1 2; do
  for lib in "$@"; do
    for c in $cfgs; do
      echo -n "$(basename $lib) rep$rep: "; TKV_LIB_PATH=$lib python tools/scan_ab.py --config $c --steps 100
    done
  done
done
