"""Which part of the host-I/O decode step's CUDA graph costs time (cfg3): back-to-back replays
of graphs holding (a) the attention call alone, (b) + the window append folded into it
(topk_decode_step), (c) + the H2D staging copy, (d) + the output written to pinned host memory.
Diagnostic only:  python tools/e2e_graph_ab.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import bench
    import paper_2502_06766_b200 as tkv

    cfg = bench.CONFIGS["cfg3"]
    dev = torch.device("cuda", 0)
    q, K, V, n = bench.make_inputs(cfg, cfg["N"] + 4096, 0, dev)
    B, k = cfg["B"], cfg["k"]
    nc = torch.full((B,), n, dtype=torch.int32, device=dev)
    nw = torch.zeros((B,), dtype=torch.int32, device=dev)
    out = torch.empty((B, 32, 128), dtype=torch.float32, device=dev)
    out_h = torch.empty((B, 32, 128), dtype=torch.float32).pin_memory()
    idx = torch.empty((B, 32, k), dtype=torch.int32, device=dev)
    sc = torch.empty((B, 32, k), dtype=torch.float32, device=dev)
    kn = torch.randn((B, 8, 128), device=dev).bfloat16()
    vn = torch.randn((B, 8, 128), device=dev).bfloat16()
    in_h = torch.empty(q.numel() + kn.numel() + vn.numel(), dtype=torch.bfloat16).pin_memory()
    in_d = torch.empty_like(in_h, device=dev)
    qh, knh, vnh = q.cpu().pin_memory(), kn.cpu().pin_memory(), vn.cpu().pin_memory()
    prob = tkv.ops.make_problem(B, 32, 8, K.shape[2], n, k)
    ws = tkv.Workspace(prob, dev)
    kw = dict(max_ctx=n, idx=idx, scores=sc, workspace=ws)

    def attn(o=out):
        tkv.topk_decode_attention(q, K, V, nc, k, n_win=nw, out=o, **kw)

    def step(o=out):
        nw.zero_()  # keep the window short and constant across replays
        tkv.topk_decode_step(q, kn, vn, K, V, nc, nw, k, out=o, **kw)

    def step_copy(o=out):
        in_d.copy_(in_h, non_blocking=True)
        step(o)

    variants = {
        "attention only": attn,
        "attention, window reset": lambda: (nw.zero_(), attn()),
        "decode_step (fold append)": step,
        "H2D copy + decode_step": step_copy,
        "H2D copy + decode_step, out -> pinned host": lambda: step_copy(out_h),
        "attention, out -> pinned host": lambda: attn(out_h),
        "attention + D2H copy node of out": lambda: (attn(), out_h.copy_(out, non_blocking=True)),
        "H2D copy node + attention": lambda: (in_d.copy_(in_h, non_blocking=True), attn()),
        "attention, q from pinned host (staged in-call)": lambda: tkv.topk_decode_attention(
            qh, K, V, nc, k, n_win=nw, out=out, **kw),
        "decode_step, q/k/v from pinned host": lambda: (nw.zero_(), tkv.topk_decode_step(
            qh, knh, vnh, K, V, nc, nw, k, out=out, **kw)),
        "decode_step, q/k/v pinned host, out -> pinned host": lambda: (nw.zero_(), tkv.topk_decode_step(
            qh, knh, vnh, K, V, nc, nw, k, out=out_h, **kw)),
    }
    s = torch.cuda.Stream()
    for name, fn in variants.items():
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                fn()
        torch.cuda.current_stream().wait_stream(s)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        print(f"{name:45s} {e0.elapsed_time(e1) / 50 * 1e3:7.1f} us/step (graph, back-to-back)")


if __name__ == "__main__":
    main()
