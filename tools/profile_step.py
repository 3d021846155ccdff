"""Run a few layer steps of one BASELINE config (for ncu captures; prints nothing useful).

    ncu --set full -k regex:select_kernel -c 1 python tools/profile_step.py --config cfg3
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    import torch

    import bench
    import paper_2502_06766_b200 as tkv

    cfg = bench.CONFIGS[args.config]
    dev = torch.device("cuda", 0)
    q, K, V, n = bench.make_inputs(cfg, cfg["N"] + 8, 0, dev)
    for _ in range(args.steps):
        tkv.topk_decode_attention(q, K, V, n, cfg["k"], max_ctx=n)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
