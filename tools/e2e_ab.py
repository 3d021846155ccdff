"""A/B of the host-I/O decode step (cfg3): window append folded into the attention call vs a
separate append kernel. Same box, same process, alternating blocks of steps. Diagnostic only."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import bench
    from paper_2502_06766_b200.decoder import TopkDecoder

    cfg = bench.CONFIGS["cfg3"]
    dev = torch.device("cuda", 0)
    q, K, V, n = bench.make_inputs(cfg, cfg["N"] + 512, 0, dev)
    decs = {f: TopkDecoder(K, V, n, cfg["k"], max_ctx=n, fold_append=f) for f in (True, False)}
    qh = q.cpu().pin_memory()
    kh = torch.randn(1, 8, 128).bfloat16().pin_memory()
    vh = torch.randn(1, 8, 128).bfloat16().pin_memory()
    res = {True: [], False: []}
    for rnd in range(6):
        for f, dec in decs.items():
            dec.n_win.zero_()  # same window length for both arms
            for _ in range(3):
                dec.step(qh, kh, vh, return_idx=False)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(50):
                dec.step(qh, kh, vh, return_idx=False)
            res[f].append((time.perf_counter() - t0) / 50 * 1e6)
    for f in (True, False):
        v = sorted(res[f])
        print(f"fold_append={f}: median {v[len(v) // 2]:.1f} us  min {v[0]:.1f} us")


if __name__ == "__main__":
    main()
