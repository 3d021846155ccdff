"""Experiment: per-step time of the small-context configs under call-flag variants.

Usage (on a B200): python tools/exp_small.py [cfg1 cfg2 ...]
Prints one JSON line per (config, variant): device µs per step over 16 cycled layer caches
(CUDA events on the launching stream) and whether the variant's ids equal the default's.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2502_06766_b200 as tkv  # noqa: E402

VARIANTS = {
    "default": {},
    "no_filter": {"no_filter": True},
    "head": {"head": True},
    "kth_gather": {"head": False},
    "no_filter_kth_gather": {"no_filter": True, "head": False},
}


def run(cfg_name, variants, steps=200):
    cfg = bench.CONFIGS[cfg_name]
    dev = torch.device("cuda", 0)
    B, N, k = cfg["B"], cfg["N"], cfg["k"]
    rows = N + bench.WINDOW_CAP
    R = 16
    reps = [bench.make_inputs(cfg, rows, r, dev) for r in range(R)]
    n_ctx = torch.full((B,), N, dtype=torch.int32, device=dev)
    ref_idx = None
    for name in variants:
        kw = VARIANTS[name]
        out = torch.empty((B, bench.HQ, bench.D), dtype=torch.float32, device=dev)
        idx = torch.empty((B, bench.HQ, k), dtype=torch.int32, device=dev)
        sc = torch.empty((B, bench.HQ, k), dtype=torch.float32, device=dev)
        prob = tkv.ops.make_problem(B, bench.HQ, bench.HKV, rows, N, k,
                                    **kw)
        ws = tkv.Workspace(prob, dev)

        def step(i):
            q, K, V, _ = reps[i % R]
            tkv.topk_decode_attention(q, K, V, n_ctx, k, out=out, idx=idx, scores=sc, workspace=ws,
                                      max_ctx=N, **kw)
        for i in range(10):
            step(i)
        torch.cuda.synchronize()
        step(0)
        torch.cuda.synchronize()
        got = idx.clone()
        same = None
        if ref_idx is None:
            ref_idx = got
        else:
            same = bool(torch.equal(torch.sort(got, dim=-1)[0], torch.sort(ref_idx, dim=-1)[0]))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for i in range(steps):
            step(i)
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / steps
        print(json.dumps({"config": cfg_name, "variant": name, "us": round(us, 2), "ids_equal_default": same}),
              flush=True)


if __name__ == "__main__":
    cfgs = sys.argv[1:] or ["cfg1", "cfg2"]
    for c in cfgs:
        run(c, list(VARIANTS))
