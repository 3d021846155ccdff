"""Print the small-context plan (cluster size, rows per CTA, resident clusters) per config."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2502_06766_b200 import _lib, ops  # noqa: E402

for name, c in bench.CONFIGS.items():
    for g in (None, True):
        p = ops.make_problem(c["B"], 32, 8, c["N"] + 8, c["N"], c["k"], group=g)
        try:
            print(name, "forced" if g else "auto", _lib.group_plan(p))
        except Exception as e:  # noqa: BLE001
            print(name, "forced" if g else "auto", "error", e)
