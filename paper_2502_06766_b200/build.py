"""Build libtkv.so (the sm_100a kernels + C ABI) in-tree with nvcc.

`python -m paper_2502_06766_b200.build` (or __graft_entry__.build()) compiles every
csrc/*.cu for sm_100a only and links them into paper_2502_06766_b200/_lib/libtkv.so, which
the package loads with ctypes. No torch headers are involved: the library is a plain C ABI
(include/tkv.h).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "libtkv.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
RDC_SOURCES = {"select.cu"}


def nvcc() -> str:
    cand = os.environ.get("NVCC") or shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError(f"nvcc not found (looked for {cand})")
    return cand


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*")) + [ROOT / "include" / "tkv.h", Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps if p.exists())


def build(force: bool = False, verbose: bool = False, out: Path | None = None, rdc: bool = True) -> Path:
    lib = Path(out) if out else LIB
    if not force and not _stale() and out is None:
        return LIB
    OUT_DIR.mkdir(parents=True, exist_ok=True)
    objs = []
    flags = ARCH + [
        "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
        "-I", str(ROOT / "include"), "-Xptxas", "-v" if verbose else "-O3",
    ] + ([] if rdc else ["-DTKV_NO_CDP"]) + os.environ.get("TKV_NVCC_FLAGS", "").split()
    rdc_objs = []
    for src in sources():
        obj = OUT_DIR / (src.stem + ".o")
        # only select.cu (k-th kernel + tail-launched fallback) needs relocatable device code;
        # the hot kernels stay whole-program compiled
        extra = ["-rdc=true"] if (rdc and src.name in RDC_SOURCES) else []
        if extra:
            rdc_objs.append(str(obj))
        cmd = [nvcc(), "-c", str(src), "-o", str(obj)] + flags + extra
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        objs.append(str(obj))
    if rdc:
        # device link: the k-th kernel tail-launches the exactness fallback (dynamic parallelism)
        dlink = OUT_DIR / "dlink.o"
        cmd = [nvcc(), "-dlink", "-o", str(dlink)] + rdc_objs + ARCH + ["-Xcompiler", "-fPIC", "-lcudadevrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc device link failed:\n{r.stdout}\n{r.stderr}")
        objs.append(str(dlink))
    tmp = OUT_DIR / "libtkv.so.tmp"
    cmd = [nvcc(), "-shared", "-o", str(tmp)] + objs + ARCH + ["-lcudadevrt", "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    for o in objs:
        os.unlink(o)
    return lib


if __name__ == "__main__":
    p = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(p)
