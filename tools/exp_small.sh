#!/bin/bash
# Latency anatomy of the small-context configs (diagnostic build: TKV_DIAG knobs + timeline),
# and the release build's step time (eager and CUDA-graph replay).
for c in ${CONFIGS:-cfg1 cfg2 cfg3}; do
  python tools/scan_ab.py --config $c --steps 100
done
export TKV_LIB_PATH=paper_2502_06766_b200/_lib/libtkv_diag.so
for c in ${CONFIGS:-cfg1 cfg2 cfg3}; do
  echo "== $c timeline (graph replay)"; python tools/timeline.py --config $c --graph
done
