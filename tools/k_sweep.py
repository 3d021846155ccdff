"""batched decode B=16, N=262,144 with the k sweep 0.5-10 % (cfg5 family).
Per k: µs per layer-step (CUDA events, back-to-back calls; default = 4 overlapped parts at
this size, and with one part), the step roofline (K + selected V + q/out + ids bytes at the
measured copy peak) and, for the one-part run, the kernel split (scan, k-th, gather) from
tkv_debug_timeline.

    python tools/k_sweep.py [--steps 20] [--out profiles/r1_cfg5_ksweep.json]
"""
import argparse
import ctypes
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
KS = [1310, 2621, 4096, 5242, 13107, 26214]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import numpy as np
    import torch

    import bench
    import paper_2502_06766_b200 as tkv
    from paper_2502_06766_b200 import _lib

    cfg = dict(bench.CONFIGS["cfg5"])
    dev = torch.device("cuda", 0)
    q, K, V, n = bench.make_inputs(cfg, cfg["N"] + 8, 0, dev)
    B = cfg["B"]
    nc = torch.full((B,), n, dtype=torch.int32, device=dev)
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    lib = _lib.load()
    rows = []
    for k in KS:
        out = torch.empty((B, 32, 128), dtype=torch.float32, device=dev)
        idx = torch.empty((B, 32, k), dtype=torch.int32, device=dev)
        sc = torch.empty((B, 32, k), dtype=torch.float32, device=dev)
        prob = tkv.ops.make_problem(B, 32, 8, K.shape[2], n, k)
        ws = tkv.Workspace(prob, dev)
        kw = dict(max_ctx=n, out=out, idx=idx, scores=sc, workspace=ws)

        def timed(**extra):
            for _ in range(3):
                tkv.topk_decode_attention(q, K, V, nc, k, **kw, **extra)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.steps):
                tkv.topk_decode_attention(q, K, V, nc, k, **kw, **extra)
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / args.steps * 1e3

        us = timed()             # default: 4 overlapped parts at this size (>= 4 GB of keys)
        us_p1 = timed(parts=1)   # one part: the plain kernel sequence, for the split below
        tl = torch.zeros(256, dtype=torch.int64, device=dev)  # TKV_TIMELINE_WORDS
        tl[0:20:2] = -1
        lib.tkv_debug_timeline(ctypes.c_void_p(tl.data_ptr()))
        tkv.topk_decode_attention(q, K, V, nc, k, **kw, parts=1)
        lib.tkv_debug_timeline(None)
        torch.cuda.synchronize()
        t = tl.cpu().numpy().view(np.uint64).astype(np.float64)
        span = lambda e: (t[2 * e + 1] - t[2 * e]) / 1e3  # noqa: E731
        kbytes = B * 8 * n * 128 * 2
        vbytes = B * 32 * k * 128 * 2
        other = B * 32 * 128 * (2 + 4) + B * 32 * k * 8
        roof_us = (kbytes + vbytes + other) / (peak * 1e3)
        row = {"k": k, "k_frac": round(k / n, 4), "us_per_step": round(us, 1), "roofline_us": round(roof_us, 1),
               "frac": round(roof_us / us, 3), "v_over_k_bytes": round(vbytes / kbytes, 3),
               "one_part_us_per_step": round(us_p1, 1),
               "one_part_split_us": {"scan": round(span(3), 1), "kth": round(span(5), 1), "gather": round(span(6), 1)}}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del ws
        torch.cuda.empty_cache()
    res = {"workload": "cfg5 family: B=16, N=262144, Hq=32, Hkv=8, d=128, bf16, standard-normal synthetic",
           "peak_gbs": peak, "steps": args.steps, "rows": rows}
    if args.out:
        Path(args.out).write_text(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    main()
