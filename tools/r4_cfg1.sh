#!/bin/bash
# cfg1 bench line, current build vs the previous (half-size-sample-only) build, twice each
cd $GRAFT_REPO_ROOT
O=gpurun_out/r4c; mkdir -p $O
for rep in 1 2; do for l in final r17; do
  echo -n "$l rep$rep "; TKV_LIB_PATH=exp/libtkv_$l.so python bench.py --config cfg1 --steps 100 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'])"
done; done > $O/cfg1.txt 2>&1
