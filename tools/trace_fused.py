"""Timeline of the fused layer-step kernel (tkv_debug_trace): per item type, when it ran and
for how long. Diagnostic only.

    python tools/trace_fused.py --config cfg3
"""
import argparse
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

NAMES = ["SAMPLE", "THRESH", "SCAN", "KTH", "ATT", "FB_SCAN", "FB_KTH", "FB_ATT"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    args = ap.parse_args()
    import numpy as np
    import torch

    import bench
    import paper_2502_06766_b200 as tkv
    from paper_2502_06766_b200 import _lib

    cfg = bench.CONFIGS[args.config]
    dev = torch.device("cuda", 0)
    q, K, V, n = bench.make_inputs(cfg, cfg["N"] + 8, 0, dev)
    for _ in range(3):
        tkv.topk_decode_attention(q, K, V, n, cfg["k"], max_ctx=n, fused=True)
    cap = 1 << 16
    buf = torch.zeros(cap * 4, dtype=torch.int64, device=dev)
    lib = _lib.load()
    lib.tkv_debug_trace(ctypes.c_void_p(buf.data_ptr()), cap)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tkv.topk_decode_attention(q, K, V, n, cfg["k"], max_ctx=n, fused=True)
    e1.record()
    torch.cuda.synchronize()
    lib.tkv_debug_trace(None, 0)
    r = buf.cpu().numpy().view(np.uint64).reshape(cap, 4)
    r = r[r[:, 1] > 0]
    t0 = r[:, 0].min()
    start = (r[:, 0] - t0) / 1e3
    end = (r[:, 1] - t0) / 1e3
    typ = ((r[:, 2] >> 32) & 0xFF).astype(int)
    ready = start + ((r[:, 2] >> 40).astype(float) * 64) / 1e3  # dependency wait end (KTH / ATT)
    cta = (r[:, 2] & 0xffffffff).astype(int)
    print(f"event time {e0.elapsed_time(e1) * 1e3:.1f} us; traced span {end.max():.1f} us; items {len(r)}; "
          f"CTAs {len(set(cta.tolist()))}")
    for t in sorted(set(typ.tolist())):
        m = typ == t
        d = end[m] - start[m]
        print(f"  {NAMES[t]:8s} n={m.sum():6d} first_start={start[m].min():8.1f} last_end={end[m].max():8.1f} "
              f"dur mean={d.mean():7.2f} max={d.max():7.2f} us  busy={d.sum():9.1f} CTA-us")
    span = end.max()
    busy = (end - start).sum()
    ncta = len(set(cta.tolist()))
    print(f"  CTA occupancy {busy / (span * ncta):.3f}  (idle = waiting / claiming / tail)")
    # tc kernel: per-group scan windows of the epilogue warps (type SCAN, a = group, b = thr wait ns)
    m = typ == 2
    if m.any():
        grp = (r[:, 3] >> 32).astype(int)
        wait = (r[:, 3] & 0xffffffff).astype(float) / 1e3
        for g in sorted(set(grp[m].tolist())):
            mg = m & (grp == g)
            print(f"    group {g:3d}: start {start[mg].min():7.1f}..{start[mg].max():7.1f}  end "
                  f"{end[mg].min():7.1f}..{end[mg].max():7.1f}  thr wait max {wait[mg].max():6.1f} us")
        for t in (3, 4):
            mt = typ == t
            if mt.any():
                ga = (r[:, 3] >> 32).astype(int) // 4  # head → group (G = 4)
                for g in sorted(set(ga[mt].tolist()))[:16]:
                    mg = mt & (ga == g)
                    work = end[mg] - ready[mg]
                    print(f"    {NAMES[t]} group {g:3d}: claimed {start[mg].min():7.1f}  ready {ready[mg].min():7.1f}"
                          f"..{ready[mg].max():7.1f}  end {end[mg].max():7.1f}  work mean {work.mean():6.1f} "
                          f"max {work.max():6.1f} us")
    # scan throughput over time windows
    m = typ == 2
    w = 20.0
    for lo in np.arange(0, span, w):
        sel = m & (start >= lo) & (start < lo + w)
        print(f"    [{lo:6.0f},{lo + w:6.0f}) scan items started {sel.sum():5d}", end="")
        other = (~m) & (start >= lo) & (start < lo + w)
        kinds = {NAMES[t]: int(((typ == t) & other).sum()) for t in set(typ[other].tolist())}
        print("  ", kinds)


if __name__ == "__main__":
    main()
