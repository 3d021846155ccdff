"""BASELINE cfg4: full 32-layer Llama-3-8B-shaped random-init decode at a 1M-token context with
top-k attention in every layer — tokens/s of greedy decoding (batch 1, one CUDA graph per step).

    python tools/bench_cfg4.py [--n-ctx 1048576] [--k 16384] [--layers 32] [--steps 20]
    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \\
        tools/bench_cfg4.py            # head-parallel tensor parallel over 8 GPUs (NCCL)

All 32 layers' K/V (137 GB bf16 at 1M) plus the 16 GB of weights fit one B200 (HBM 180 GB),
so one GPU runs it; under torchrun the model is head-parallel (TopkLlamaDecoder tp_group: each
rank holds Hkv/T kv heads' whole-context caches and 1/T of every layer's weights, two NCCL
all-reduces per layer) and the step time is the max over ranks.
"""

import argparse
import json
import os
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
    ap.add_argument("--tp-shard", type=int, default=0,
                    help="single GPU: build rank 0's shard of a T-way tensor-parallel model and time "
                         "its compute (the two all-reduces per layer are not run)")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    from paper_2502_06766_b200.model import LLAMA3_8B, TopkLlamaDecoder
    from dataclasses import replace

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD
    shape = replace(LLAMA3_8B, n_layers=args.layers)
    need = TopkLlamaDecoder.memory_bytes(shape, args.n_ctx, tp=world)
    free, total = torch.cuda.mem_get_info(dev)
    shard = (args.tp_shard, 0) if args.tp_shard > 1 and group is None else None
    if shard:
        need = TopkLlamaDecoder.memory_bytes(shape, args.n_ctx, tp=args.tp_shard)
    dec = TopkLlamaDecoder(shape, args.n_ctx, args.k, device=dev, seed=0, tp_group=group, tp_shard=shard)
    dec.capture()
    tok = 1
    for _ in range(args.warmup):
        dec.step(tok)
        tok = None
    torch.cuda.synchronize()
    if group is not None:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        dec.step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if group is not None:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        same = torch.tensor([int(dec.next_token.item())], device=dev)
        lo, hi = same.clone(), same.clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
        tokens_agree = bool(lo.item() == hi.item())
    else:
        tokens_agree = True
    if rank == 0:
        print(json.dumps({
            "metric": "decode_tokens_per_s", "value": round(1e3 / ms, 2), "unit": "tokens/s",
            "ms_per_token": round(ms, 3), "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "strong",
            "config": {"workload": "cfg4", "model": "Llama-3-8B shape, random init", "layers": args.layers,
                       "n_ctx": args.n_ctx, "k": args.k, "batch": 1, "attention": "libtkv top-k per layer",
                       "parallelism": (f"tp{world} (head-parallel)" if world > 1 else
                                       f"rank 0 of tp{args.tp_shard}, compute only (no all-reduce)" if shard
                                       else "single GPU"),
                       "cuda_graph": True, "hbm_needed_gb_per_rank": round(need / 1e9, 1),
                       "hbm_free_gb_before": round(free / 1e9, 1)},
            "per_layer_us": round(ms * 1e3 / args.layers, 1), "tokens_agree_across_ranks": tokens_agree,
        }))
    if group is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
