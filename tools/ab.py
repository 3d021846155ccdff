"""A/B timing of the layer step: fused vs multi-kernel (CUDA events, K steps, cfg selectable)."""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

def main():
    ap = argparse.ArgumentParser(); ap.add_argument("--config", default="cfg3"); ap.add_argument("--steps", type=int, default=50)
    args = ap.parse_args()
    import torch, bench, paper_2502_06766_b200 as tkv
    cfg = bench.CONFIGS[args.config]; dev = torch.device("cuda", 0)
    q, K, V, n = bench.make_inputs(cfg, cfg["N"] + 8, 0, dev)
    B, k = cfg["B"], cfg["k"]
    nc = torch.full((B,), n, dtype=torch.int32, device=dev)
    out = torch.empty((B, 32, 128), dtype=torch.float32, device=dev)
    idx = torch.empty((B, 32, k), dtype=torch.int32, device=dev)
    sc = torch.empty((B, 32, k), dtype=torch.float32, device=dev)
    for fused in (True, False):
        prob = tkv.ops.make_problem(B, 32, 8, K.shape[2], n, k, fused=fused)
        ws = tkv.Workspace(prob, dev)
        kw = dict(max_ctx=n, fused=fused, out=out, idx=idx, scores=sc, workspace=ws)
        for _ in range(5):
            tkv.topk_decode_attention(q, K, V, nc, k, **kw)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            tkv.topk_decode_attention(q, K, V, nc, k, **kw)
        e1.record(); torch.cuda.synchronize()
        print(f"{args.config} fused={fused}: {e0.elapsed_time(e1) / args.steps * 1e3:.1f} us/step")

if __name__ == "__main__":
    main()
