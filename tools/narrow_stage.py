"""Per-rank cost of the sharded candidate stage, full-k vs narrow k' (one GPU, no collectives).

cfg3 (N = 1M, k = 16384) sharded G ways: every rank owns N/G rows. Times, with CUDA events over
`--steps` calls: tkv_shard_candidates at k and at k' = narrow_k(k, G); the exactness rule (device
kernel and the torch restatement) and tkv_shard_merge(_lists) over a G-rank gathered buffer (the
G lists are the G shards' real candidate lists, produced one after another on this GPU). Prints
the all-gather bytes each rank receives in both modes. Run: python tools/narrow_stage.py
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
    args = ap.parse_args()
    import torch

    import bench
    import paper_2502_06766_b200 as tkv
    from paper_2502_06766_b200.sharded import narrow_exchange_exact

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

    res = []
    for G in args.shards:
        kk = tkv.narrow_k(k, G, args.c)
        cands_full, cands_narrow, t_full, t_narrow = [], [], [], []
        for g in range(G):
            lo, hi = tkv.shard_range(N, G, g)
            q, K, V, n = bench.make_inputs(cfg, hi - lo, 0, dev, lo, hi)
            nc = torch.full((B,), n, dtype=torch.int32, device=dev)
            full = tkv.CudaStages(B, 32, 8, hi - lo, n, k, row_offset=lo, device=dev)
            nar = tkv.CudaStages(B, 32, 8, hi - lo, n, kk, row_offset=lo, device=dev)
            if g == 0:
                t_full.append(timed(lambda: full.candidates(q, K, nc)))
                t_narrow.append(timed(lambda: nar.candidates(q, K, nc)))
                st0 = full
            cands_full.append(full.candidates(q, K, nc).clone())
            cands_narrow.append(nar.candidates(q, K, nc).clone())
            del K, V
        gf, gn = torch.cat(cands_full), torch.cat(cands_narrow)
        exact = bool(narrow_exchange_exact(gn, G, k, kk).all())
        assert (st0.narrow_exact(gn, G, kk) != 0).tolist() == narrow_exchange_exact(gn, G, k, kk).tolist()
        t_rule_torch = timed(lambda: narrow_exchange_exact(gn, G, k, kk))
        t_rule = timed(lambda: st0.narrow_exact(gn, G, kk))
        t_merge = timed(lambda: st0.merge(gf, G))
        t_merge_n = timed(lambda: st0.merge(gn, G, kk))
        idx_f, _ = st0.merge(gf, G)
        idx_f = idx_f.clone()
        idx_n, _ = st0.merge(gn, G, kk)
        same = all(set(a.tolist()) == set(b.tolist())
                   for a, b in zip(idx_f.view(-1, k).cpu(), idx_n.view(-1, k).cpu()))
        r = {"G": G, "rows_per_rank": N // G, "k": k, "k_narrow": kk,
             "candidates_us_full": round(t_full[0], 1), "candidates_us_narrow": round(t_narrow[0], 1),
             "rule_kernel_us": round(t_rule, 1), "rule_torch_us": round(t_rule_torch, 1),
             "merge_us_full": round(t_merge, 1), "merge_us_narrow": round(t_merge_n, 1),
             "allgather_rx_MB_full": round((G - 1) * B * 32 * k * 8 / 1e6, 2),
             "allgather_rx_MB_narrow": round((G - 1) * B * 32 * kk * 8 / 1e6, 2),
             "narrow_exact": exact, "ids_equal": same}
        print(json.dumps(r), flush=True)
        res.append(r)


if __name__ == "__main__":
    main()
