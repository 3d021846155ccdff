"""Cross-kernel timeline of one multi-kernel layer step (tkv_debug_timeline): when each kernel
first started / last ended, relative to the sample kernel's start. Diagnostic only.

    python tools/timeline.py --config cfg3 [--steps 20]
"""
import argparse
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
NAMES = ["sample", "threshold", "threshold past wait", "scan", "scan epilogue past wait", "k-th", "gather",
         "head: threshold found", "head: rows compacted", "head: V gathered"]
PHASES = ["head CTA: start→params", "→hist+bucket", "→pass 1 (max, bucket members)", "→T",
          "→pads/meta + barriers", "→compaction loop", "→out_cnt reservation", "→V gather loop", "→ids written",
          "→partial slot written", "→finished (last CTA)",
          "kth CTA: past wait→hist+bucket", "→slice scan + max", "→cluster sync + pulls (rank 0)", "→T written (rank 0)",
          "threshold CTA: past wait→samples in smem", "→sample max", "→radix select (t_h)", "→hist zeroed, state written",
          "scan epilogue: one warp flush"]


EXTRA_EVENTS = {40: "scan CTA start", 41: "scan CTA end", 45: "threshold CTA past wait",
                53: "k-th CTA resident", 54: "k-th CTA past wait"}
EXTRA_PHASES = {42: "scan epilogue: wait for a unit's scores", 43: "scan epilogue: ld+emit of a unit",
                44: "scan MMA warp: wait for a unit's TMA", 46: "scan CTA lifetime",
                47: "merge: start→bounds + narrow count + rule", 48: "→histogram + cluster sums + bucket",
                49: "→bucket count", 50: "→members + barrier", 51: "→rank select + barrier",
                52: "→emit (2 passes) + barrier",
                55: "kth CTA: past wait→state loads", 56: "kth CTA: →hist in smem (then bucket)",
                60: "gather CTA: start→item prefix", 61: "gather: →batch candidates loaded",
                62: "gather: →compaction (2 barriers)", 63: "gather: →V rows accumulated",
                64: "gather: →ids written (per item)", 65: "gather: →partial written",
                66: "gather: →ticket / head finish",
                67: "cluster CTA: past wait→params", 68: "→hist + bucket", 69: "→slice scan + max",
                70: "→cluster barrier 1", 71: "→peer members + T", 72: "→compaction + V gather",
                73: "→partial hand-off (remote mbarrier arrivals)", 74: "→finish (rank 0)",
                75: "  (per batch: →compaction)", 76: "  (per batch: →V gather)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--graph", action="store_true", help="replay the step as a CUDA graph (no host launch gaps)")
    args = ap.parse_args()
    import numpy as np
    import torch

    import bench
    import paper_2502_06766_b200 as tkv
    from paper_2502_06766_b200 import _lib

    cfg = bench.CONFIGS[args.config]
    dev = torch.device("cuda", 0)
    q, K, V, n = bench.make_inputs(cfg, cfg["N"] + 8, 0, dev)
    B, k = cfg["B"], cfg["k"]
    nc = torch.full((B,), n, dtype=torch.int32, device=dev)
    kw = dict(max_ctx=n)
    lib = _lib.load()
    acc = np.zeros((len(NAMES), 2))
    ph = np.zeros(len(PHASES))
    xe = {e: [0.0, 0.0] for e in EXTRA_EVENTS}
    xp = {e: 0.0 for e in EXTRA_PHASES}
    buf = torch.zeros(256, dtype=torch.int64, device=dev)  # TKV_TIMELINE_WORDS
    init = torch.zeros_like(buf)
    init[0:2 * len(NAMES):2] = -1  # UINT64_MAX (first-start slots); phase sums stay 0
    for e in EXTRA_EVENTS:
        init[2 * e] = -1
    graphs = None
    if args.graph:
        tkv.topk_decode_attention(q, K, V, nc, k, **kw)
        torch.cuda.synchronize()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        plain, timed = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.stream(side):
            with torch.cuda.graph(plain, stream=side):
                tkv.topk_decode_attention(q, K, V, nc, k, **kw)
            lib.tkv_debug_timeline(ctypes.c_void_p(buf.data_ptr()))
            with torch.cuda.graph(timed, stream=side):
                tkv.topk_decode_attention(q, K, V, nc, k, **kw)
            lib.tkv_debug_timeline(None)
        torch.cuda.current_stream().wait_stream(side)
        graphs = (plain, timed)
    for it in range(args.steps + 3):
        buf.copy_(init)
        if graphs:
            graphs[0].replay()  # previous step in flight: realistic
            graphs[1].replay()
        else:
            tkv.topk_decode_attention(q, K, V, nc, k, **kw)  # previous step in flight: realistic
            lib.tkv_debug_timeline(ctypes.c_void_p(buf.data_ptr()))
            tkv.topk_decode_attention(q, K, V, nc, k, **kw)
            lib.tkv_debug_timeline(None)
        torch.cuda.synchronize()
        raw = buf.cpu().numpy().view(np.uint64)
        t = raw.astype(np.float64)
        t0 = t[0]
        if it >= 3:
            for j in range(len(PHASES)):
                e = len(NAMES) + j
                if t[2 * e + 1] > 0:
                    ph[j] += t[2 * e] / t[2 * e + 1] / 1e3
            for e in range(len(NAMES)):
                s, en = t[2 * e], t[2 * e + 1]
                acc[e, 0] += (s - t0) / 1e3 if s < 1.8e19 else np.nan
                acc[e, 1] += (en - t0) / 1e3 if en > 0 else np.nan
            for e in EXTRA_EVENTS:
                s, en = t[2 * e], t[2 * e + 1]
                xe[e][0] += (s - t0) / 1e3 if s < 1.8e19 else np.nan
                xe[e][1] += (en - t0) / 1e3 if en > 0 else np.nan
            for e in EXTRA_PHASES:
                if t[2 * e + 1] > 0:
                    xp[e] += t[2 * e] / t[2 * e + 1] / 1e3
    acc /= args.steps

    def sms(w):  # SM bitmask words (tl_smid) of the last step
        return {64 * i + b for i in range(3) for b in range(64) if (int(raw[w + i]) >> b) & 1}

    thr_sms, late_sms, scan_sms = sms(240), sms(243), sms(246)
    if scan_sms:
        print(f"  SMs: scan CTAs on {len(scan_sms)}, threshold CTAs on {len(thr_sms)}, scan CTAs starting "
              f">6 us late on {len(late_sms)} (of which {len(late_sms & thr_sms)} host a threshold CTA)")
    clus_sms = sms(249)
    if clus_sms:
        print(f"  SMs hosting a cluster k-th + gather CTA: {len(clus_sms)}")
    for e, nm in enumerate(NAMES):
        print(f"  {nm:26s} start {acc[e, 0]:8.1f}  end {acc[e, 1]:8.1f} us")
    for j, nm in enumerate(PHASES):
        if ph[j] > 0:
            print(f"  {nm:34s} {ph[j] / args.steps:8.2f} us (mean)")
    for e, nm in EXTRA_EVENTS.items():
        print(f"  {nm:34s} first {xe[e][0] / args.steps:8.1f}  last {xe[e][1] / args.steps:8.1f} us")
    for e, nm in EXTRA_PHASES.items():
        if xp[e] > 0:
            print(f"  {nm:34s} {xp[e] / args.steps:8.2f} us (mean)")


if __name__ == "__main__":
    main()
