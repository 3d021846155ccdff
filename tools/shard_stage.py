"""Per-rank cost of the device-driven sharded step at cfg3 (one GPU, exchange emulated):
cfg3 (N = 1M, k = 16384) split into G token-range shards; every shard's lists are produced on
this GPU (LocalExchange), then rank 0's stages are timed with CUDA events: candidates2 (one scan,
local top-k' and top-k), the device merge over the G published lists (narrow or full chosen per
head on the device), the partial gather and the combine (sum of G partials + finish). Peer reads
are local here: NVLink time for the merge's list reads (G·k' composites per head) is not modelled.

    python tools/shard_stage.py [--shards 2 4 8] [--steps 20]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shards", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--c", type=float, default=1.5)
    ap.add_argument("--phases", action="store_true")
    args = ap.parse_args()
    import torch

    import bench
    import paper_2502_06766_b200 as tkv

    dev = torch.device("cuda", 0)
    cfg = bench.CONFIGS["cfg3"]
    N, k, B = cfg["N"], cfg["k"], cfg["B"]

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

    for G in args.shards:
        kk = tkv.narrow_k(k, G, args.c)
        exch = tkv.LocalExchange(G, B, 32, k, kk, dev)
        ranks = []
        for g in range(G):
            lo, hi = tkv.shard_range(N, G, g)
            q, K, V, n = bench.make_inputs(cfg, hi - lo + 8, 0, dev, lo, hi)
            nc = torch.full((B,), n, dtype=torch.int32, device=dev)
            st = tkv.CudaStages(B, 32, 8, K.shape[2], n, k, row_offset=lo, device=dev)
            step = tkv.DeviceShardedStep(st, exch, g, kk)
            step.publish_candidates(q, K, nc)
            ranks.append((step, q, K, V, nc))
            if g > 0:  # keep only rank 0's shard resident beyond its published lists
                del K, V
                ranks[-1] = (step, q, None, None, nc)
        torch.cuda.synchronize()
        step, q, K, V, nc = ranks[0]
        nw = torch.zeros(B, dtype=torch.int32, device=dev)
        t_cand = timed(lambda: step.publish_candidates(q, K, nc))
        t_merge = timed(lambda: step.merge_and_partial(q, K, V, nc))
        nar_p, full_p, bound_p, _ = exch.pointers()
        t_merge_only = timed(lambda: step.stages.exchange_merge(nar_p, full_p, bound_p, G, kk, step.used_full))
        t_comb = timed(lambda: step.combine(q, K, V, nc, nw))
        if args.phases:  # TKV_DIAG build: per-phase means of the merge kernel (tkv_debug_timeline)
            import ctypes
            import numpy as np
            from tools.timeline import EXTRA_PHASES
            buf = torch.zeros(256, dtype=torch.int64, device=dev)
            lib = tkv._lib.load()
            lib.tkv_debug_timeline(ctypes.c_void_p(buf.data_ptr()))
            for _ in range(args.steps):
                step.stages.exchange_merge(nar_p, full_p, bound_p, G, kk, step.used_full)
            lib.tkv_debug_timeline(None)
            torch.cuda.synchronize()
            t = buf.cpu().numpy().view(np.uint64).astype(np.float64)
            for e in range(47, 53):
                if t[2 * e + 1] > 0:
                    print(f"  G={G} {EXTRA_PHASES.get(e, e):40s} {t[2 * e] / t[2 * e + 1] / 1e3:7.2f} us", flush=True)
        t_step = t_cand + t_merge + t_comb
        used = int(step.used_full.sum().item())
        kbytes = B * 8 * (N // G) * 128 * 2
        rec = {"G": G, "rows_per_rank": N // G, "narrow_k": kk, "candidates2_us": round(t_cand, 1),
               "merge_us": round(t_merge_only, 1), "partial_us": round(t_merge - t_merge_only, 1),
               "combine_us": round(t_comb, 1), "rank_step_us": round(t_step, 1),
               "k_scan_roofline_us": round(kbytes / 6437.9e9 * 1e6, 1),
               "heads_merged_from_full": used,
               "narrow_list_bytes_read_per_rank": G * B * 32 * kk * 8}
        print(json.dumps(rec), flush=True)
        del ranks, exch
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
