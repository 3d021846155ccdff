"""Time the layer step and its key-scan kernel (CUDA events around the scan launch) for one
config and scan variant:  python tools/scan_ab.py --config cfg3 [--scan tc|hmma] [--steps 50]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--scan", choices=["tc", "hmma"], default="tc")
    ap.add_argument("--label", default="")
    ap.add_argument("--no-filter", action="store_true", help="no sampled threshold: every score is a candidate")
    ap.add_argument("--n", type=int, default=0, help="override the context length")
    ap.add_argument("--k", type=int, default=0, help="override k")
    ap.add_argument("--head", default="auto", choices=["auto", "cluster", "head", "kth"],
                    help="k-th + gather kernels: automatic, cluster, per-head CTAs, k-th + candidate gather")
    args = ap.parse_args()
    args.tc = args.scan == "tc"
    import torch

    import bench
    import paper_2502_06766_b200 as tkv
    from paper_2502_06766_b200 import _lib

    cfg = dict(bench.CONFIGS[args.config])
    if args.n:
        cfg["N"] = args.n
    if args.k:
        cfg["k"] = args.k
    dev = torch.device("cuda", 0)
    q, K, V, n = bench.make_inputs(cfg, cfg["N"] + 8, 0, dev)
    B, k = cfg["B"], cfg["k"]
    nc = torch.full((B,), n, dtype=torch.int32, device=dev)
    out = torch.empty((B, 32, 128), dtype=torch.float32, device=dev)
    idx = torch.empty((B, 32, k), dtype=torch.int32, device=dev)
    sc = torch.empty((B, 32, k), dtype=torch.float32, device=dev)
    head = {"auto": None, "cluster": "cluster", "head": True, "kth": False}[args.head]
    prob = tkv.ops.make_problem(B, 32, 8, K.shape[2], n, k, tc_scan=args.tc, head=head,
                                no_filter=args.no_filter)
    ws = tkv.Workspace(prob, dev)
    kw = dict(max_ctx=n, out=out, idx=idx, scores=sc, workspace=ws, tc_scan=args.tc, head=head,
              no_filter=args.no_filter)
    for _ in range(5):
        tkv.topk_decode_attention(q, K, V, nc, k, **kw)
    torch.cuda.synchronize()
    lib = _lib.load()
    # step time: plain back-to-back calls (no profiling hooks, so programmatic dependent
    # launch between the kernels stays on); scan time: a second loop with the scan events
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        tkv.topk_decode_attention(q, K, V, nc, k, **kw)
    e1.record()
    torch.cuda.synchronize()
    step = e0.elapsed_time(e1) / args.steps * 1e3
    # the same call captured once into a CUDA graph and replayed (no host launch cost per kernel)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side), torch.cuda.graph(g, stream=side):
        tkv.topk_decode_attention(q, K, V, nc, k, **kw)
    torch.cuda.current_stream().wait_stream(side)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    step_graph = e0.elapsed_time(e1) / args.steps * 1e3
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a, b in ev:
        a.record(); b.record()
    torch.cuda.synchronize()
    for a, b in ev:
        lib.tkv_profile_scan_events(a.cuda_event, b.cuda_event)
        tkv.topk_decode_attention(q, K, V, nc, k, **kw)
    torch.cuda.synchronize()
    lib.tkv_profile_scan_events(None, None)
    scan = sum(a.elapsed_time(b) for a, b in ev) / args.steps * 1e3
    kbytes = B * 8 * n * 128 * 2
    print(f"{args.config} N={n} k={k} tc={int(args.tc)} head={args.head} nf={int(args.no_filter)} {args.label}: step {step:.1f} us (graph replay {step_graph:.1f} us), scan {scan:.1f} us "
          f"({kbytes / scan / 1e3:.0f} GB/s)", flush=True)


if __name__ == "__main__":
    main()
