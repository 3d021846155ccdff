"""Cost of the exactness fallback at cfg3: the step on the normal synthetic
cache, on a cache whose sampled rows of ONE kv group score far above everything else (the
sampled thresholds of that group's 4 heads admit < k rows → re-scan of the group), and on one
where every group's sampled rows do (all 32 heads fall back). CUDA events, µs per layer-step.

    python tools/fallback_cliff.py [--steps 20]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--config", default="cfg3")
    args = ap.parse_args()
    import torch

    import bench
    import paper_2502_06766_b200 as tkv
    from tests.conftest import sample_rows

    cfg = bench.CONFIGS[args.config]
    dev = torch.device("cuda", 0)
    B, N, k = cfg["B"], cfg["N"], cfg["k"]
    q, K, V, n = bench.make_inputs(cfg, N + 8, 0, dev)
    nc = torch.full((B,), n, dtype=torch.int32, device=dev)
    res = {}
    for mode in ("none", "one_group", "all_groups"):
        Km = K.clone() if mode != "none" else K
        if mode != "none":
            groups = [0] if mode == "one_group" else list(range(bench.HKV))
            for g in groups:
                rows = torch.from_numpy(sample_rows(n, g)).to(dev)
                boost = (2.0 * torch.sign(q[0, g * 4].float()))[None, :]
                Km[0, g, rows] = (Km[0, g, rows].float() * 0.01 + boost).to(torch.bfloat16)
        prob = tkv.ops.make_problem(B, 32, 8, Km.shape[2], n, k)
        ws = tkv.Workspace(prob, dev)
        kw = dict(max_ctx=n, workspace=ws)
        for _ in range(3):
            tkv.topk_decode_attention(q, Km, V, nc, k, **kw)
        torch.cuda.synchronize()
        f0 = ws.fallbacks(prob)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            tkv.topk_decode_attention(q, Km, V, nc, k, **kw)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / args.steps * 1e3
        res[mode] = {"us_per_step": round(us, 1), "fallback_heads_per_step": (ws.fallbacks(prob) - f0) / args.steps}
        print(mode, res[mode], flush=True)
        del Km
    print(json.dumps({"config": args.config, "steps": args.steps, **res}))


if __name__ == "__main__":
    main()
