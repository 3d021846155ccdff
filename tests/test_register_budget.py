"""Register budgets the layer pipeline's co-residency depends on (CPU-only: ptxas -v).

The kernels of one layer step overlap through programmatic dependent launch: the k-th kernel's
CTAs become resident beside the running tcgen05 scan CTA, and so do the threshold CTAs. An SM's
register file is four 16K-register sub-partitions; the 10-warp scan CTA puts 3 warps on two of
them, so (3 x scan regs + 4 x kth regs) x 32 lanes must fit 16384. Measured: a scan kernel at
130 registers (diagnostic timers compiled into the release build) pushed the k-th kernel behind
the scan and cost 18 us per cfg3 step. These checks keep the budgets from drifting silently.
"""

from __future__ import annotations

import re
import shutil
import subprocess
from pathlib import Path

import pytest

CSRC = Path(__file__).resolve().parents[1] / "paper_2502_06766_b200" / "csrc"
INC = Path(__file__).resolve().parents[1] / "include"
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"

pytestmark = pytest.mark.skipif(not Path(NVCC).exists(), reason="nvcc not available")


def _registers(src: str, rdc: bool = False) -> dict[str, int]:
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "--expt-relaxed-constexpr",
           "-I", str(INC), "-Xptxas", "-v", "-c", str(CSRC / src), "-o", "/dev/null"] + (["-rdc=true"] if rdc else [])
    r = subprocess.run(cmd, capture_output=True, text=True, check=True)
    regs, fn = {}, None
    for line in r.stderr.splitlines():
        m = re.search(r"Compiling entry function '([^']+)'", line)
        if m:
            fn = m.group(1)
        m = re.search(r"Used (\d+) registers", line)
        if m and fn:
            regs[fn] = int(m.group(1))
            fn = None
    return regs


def _find(regs: dict[str, int], name: str) -> int:
    hits = [v for k, v in regs.items() if name in k]
    assert hits, f"{name} not found in {sorted(regs)}"
    return max(hits)


def test_scan_and_kth_share_an_sm():
    scan = _find(_registers("scan_tc.cu"), "scan_tc_kernel")
    kth = _find(_registers("select.cu", rdc=True), "kth_kernel")
    assert scan <= 120, f"scan_tc_kernel uses {scan} registers (budget 120)"
    assert kth <= 32, f"kth_kernel uses {kth} registers (budget 32)"
    per_warp = lambda r: ((r + 7) // 8) * 8 * 32  # noqa: E731  (allocation granule: 8 per thread)
    assert 3 * per_warp(scan) + 4 * per_warp(kth) <= 16384


def test_threshold_fits_beside_the_scan():
    regs = _registers("scan.cu")
    thr = _find(regs, "threshold_kernel")
    assert thr <= 32, f"threshold_kernel uses {thr} registers (budget 32)"
