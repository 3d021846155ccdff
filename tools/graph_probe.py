"""Eager launches vs CUDA-graph replay of the same cfg3 layer step (device inputs), with the
cross-kernel timeline of each — where a graph loses time against eager PDL launches.
Diagnostic only:  python tools/graph_probe.py [--config cfg3]"""
import argparse
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
NAMES = ["sample", "threshold", "threshold past wait", "scan", "scan epilogue past wait", "k-th", "gather"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--steps", type=int, default=50)
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
    out = torch.empty((B, 32, 128), dtype=torch.float32, device=dev)
    idx = torch.empty((B, 32, k), dtype=torch.int32, device=dev)
    sc = torch.empty((B, 32, k), dtype=torch.float32, device=dev)
    prob = tkv.ops.make_problem(B, 32, 8, K.shape[2], n, k)
    ws = tkv.Workspace(prob, dev)
    lib = _lib.load()

    def call():
        tkv.topk_decode_attention(q, K, V, nc, k, max_ctx=n, out=out, idx=idx, scores=sc, workspace=ws)

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / args.steps * 1e3

    print(f"eager back-to-back:  {timed(call):.1f} us/step")
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            call()
    torch.cuda.current_stream().wait_stream(s)
    print(f"graph back-to-back:  {timed(g.replay):.1f} us/step")
    # timelines: eager (isolated step) and a graph captured with the timeline buffer baked in
    buf = torch.zeros(64, dtype=torch.int64, device=dev)
    lib.tkv_debug_timeline(ctypes.c_void_p(buf.data_ptr()))
    acc_e = []
    for it in range(13):
        buf[0:20:2] = -1
        buf[20:] = 0
        torch.cuda.synchronize()
        call()
        torch.cuda.synchronize()
        acc_e.append(buf.cpu().numpy().view(np.uint64).astype(np.float64))
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g2, stream=s):
            call()
    torch.cuda.current_stream().wait_stream(s)
    lib.tkv_debug_timeline(None)
    acc_g = []
    for it in range(13):
        buf[0:20:2] = -1
        buf[20:] = 0
        torch.cuda.synchronize()
        g2.replay()
        torch.cuda.synchronize()
        acc_g.append(buf.cpu().numpy().view(np.uint64).astype(np.float64))
    for label, rows in (("eager", acc_e[3:]), ("graph", acc_g[3:])):
        print(f"  {label} timeline (isolated step):")
        for e, nm in enumerate(NAMES):
            st = [(t[2 * e] - t[0]) / 1e3 for t in rows if t[2 * e] < 1.8e19]
            en = [(t[2 * e + 1] - t[0]) / 1e3 for t in rows if t[2 * e + 1] > 0]
            if st or en:
                print(f"    {nm:26s} start {np.mean(st) if st else float('nan'):8.1f}  "
                      f"end {np.mean(en) if en else float('nan'):8.1f} us")


if __name__ == "__main__":
    main()
