L=paper_2502_06766_b200/_lib/libtkv.so
cp $L /tmp/new.so
for r in 1 2 3; do
  cp /tmp/new.so $L; echo "new"; timeout 120 python tools/timeline.py --config cfg3 2>&1 | grep "k-th  \|gather  "; timeout 120 python tools/scan_ab.py --config cfg3 --steps 200 2>&1 | tail -1
  cp tools/_alt/libtkv_oldkth.so $L; echo "old"; timeout 120 python tools/timeline.py --config cfg3 2>&1 | grep "k-th  \|gather  "; timeout 120 python tools/scan_ab.py --config cfg3 --steps 200 2>&1 | tail -1
done
cp /tmp/new.so $L
