"""BASELINE cfg4: full 32-layer Llama-3-8B-shaped random-init decode at a 1M-token context with
top-k attention in every layer — tokens/s of greedy decoding (batch 1, one CUDA graph per step).

    python tools/bench_cfg4.py [--n-ctx 1048576] [--k 16384] [--layers 32] [--steps 20]

All 32 layers' K/V (137 GB bf16 at 1M) plus the 16 GB of weights fit one B200 (HBM 180 GB),
so this runs on a single GPU; the token-range sharded variant is the multi-GPU path.
"""

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-ctx", type=int, default=1 << 20)
    ap.add_argument("--k", type=int, default=16384)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    import torch

    from paper_2502_06766_b200.model import LLAMA3_8B, TopkLlamaDecoder
    from dataclasses import replace

    shape = replace(LLAMA3_8B, n_layers=args.layers)
    dev = torch.device("cuda", 0)
    need = TopkLlamaDecoder.memory_bytes(shape, args.n_ctx)
    free, total = torch.cuda.mem_get_info(dev)
    dec = TopkLlamaDecoder(shape, args.n_ctx, args.k, device=dev, seed=0)
    dec.capture()
    tok = 1
    for _ in range(args.warmup):
        dec.step(tok)
        tok = None
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        dec.step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    print(json.dumps({
        "metric": "decode_tokens_per_s", "value": round(1e3 / ms, 2), "unit": "tokens/s", "ms_per_token": round(ms, 3),
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
        "config": {"workload": "cfg4", "model": "Llama-3-8B shape, random init", "layers": args.layers,
                   "n_ctx": args.n_ctx, "k": args.k, "batch": 1, "attention": "libtkv top-k per layer",
                   "cuda_graph": True, "hbm_needed_gb": round(need / 1e9, 1),
                   "hbm_free_gb_before": round(free / 1e9, 1)},
        "per_layer_us": round(ms * 1e3 / args.layers, 1),
    }))


if __name__ == "__main__":
    main()
