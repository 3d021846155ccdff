#!/bin/bash
# Round-2 ncu evidence: per-launch device times (cold-cache, serialised) for cfg1/cfg2/cfg3 and a
# full capture of the key-scan kernel at cfg3. Each ncu command follows the same command run
# plainly (exit 0) first.
set -e
mkdir -p gpurun_out
for c in cfg1 cfg2 cfg3; do
  python tools/scan_ab.py --config $c --steps 3 > gpurun_out/plain_$c.log 2>&1
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
      -k regex:"stage|sample|threshold|scan_tc|kth|attend|head_topk|sort" \
      --log-file gpurun_out/r2_${c}_launches.csv python tools/scan_ab.py --config $c --steps 3 > gpurun_out/ncu_$c.log 2>&1
done
