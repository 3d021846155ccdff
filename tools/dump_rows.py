"""Dump the selected V-row list of one cfg3 layer step (output order, global row = kv head ·
rows + local row) for tools/micro/gather_bw. Diagnostic only."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    import bench
    import paper_2502_06766_b200 as tkv

    cfg = bench.CONFIGS["cfg3"]
    dev = torch.device("cuda", 0)
    q, K, V, n = bench.make_inputs(cfg, cfg["N"] + 8, 0, dev)
    _, idx, _ = tkv.topk_decode_attention(q, K, V, [n], cfg["k"], max_ctx=n)
    idx = idx.cpu().numpy()[0]  # [32, k]
    rows = n  # pack heads at N rows each: 8 × 1M × 256 B = the 2 GiB test buffer
    glob = (np.arange(32)[:, None] // 4) * rows + idx
    glob.astype(np.int32).tofile(sys.argv[1])
    print("rows", glob.size)


if __name__ == "__main__":
    main()
