"""CPU, world_size 2 and 4 over gloo: the token-range sharded protocol
(paper_2502_06766_b200.sharded.sharded_topk_attention) gives the unsharded oracle's ids and
outputs. The per-rank compute stages are the oracle's (oracle/shard_stages.py, test
infrastructure); the communication path is the product's."""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _data(seed=0, B=2, Hq=8, Hkv=2, N=997, W=3):
    sys.path.insert(0, str(ROOT))
    from oracle import oracle as O

    rng = np.random.default_rng(seed)
    q = O.to_bf16_f32(rng.standard_normal((B, Hq, 128), dtype=np.float32))
    K = O.to_bf16_f32(rng.standard_normal((B, Hkv, N + W, 128), dtype=np.float32))
    V = O.to_bf16_f32(rng.standard_normal((B, Hkv, N + W, 128), dtype=np.float32))
    K[:, :, 100:900:50] = K[:, :, 7:8]  # exact duplicates spread over shards: lower-id ties
    return q, K, V, N, W


def _worker(rank, world, port, k, combine, pinned, result_path):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.shard_stages import OracleStages
    from paper_2502_06766_b200.sharded import shard_range, sharded_topk_attention

    q, K, V, N, W = _data()
    B, Hq, Hkv = q.shape[0], q.shape[1], K.shape[1]
    lo, hi = shard_range(N, world, rank)
    ks = np.concatenate([K[:, :, lo:hi], K[:, :, N:N + W]], axis=2)
    vs = np.concatenate([V[:, :, lo:hi], V[:, :, N:N + W]], axis=2)
    st = OracleStages(B, Hq, Hkv, k, row_offset=lo, combine=combine, pinned_prefix=pinned)
    out, idx, sc = sharded_topk_attention(st, torch.from_numpy(q), torch.from_numpy(ks),
                                          torch.from_numpy(vs), [hi - lo] * B, [W] * B)
    np.savez(f"{result_path}.{rank}.npz", out=out.numpy(), idx=idx.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world,k,combine,pinned", [
    (2, 40, "joint", 0),
    (2, 7, "additive", 5),
    (4, 100, "joint", 3),
    (4, 2000, "joint", 0),  # k > N: every row, clamped
])
def test_sharded_equals_unsharded(tmp_path, world, k, combine, pinned):
    from oracle import oracle as O

    port = 29400 + world * 10 + (k % 7)
    res = str(tmp_path / "r")
    mp.start_processes(_worker, args=(world, port, k, combine, pinned, res), nprocs=world,
                       join=True, start_method="spawn")
    q, K, V, N, W = _data()
    ref_out, ref_ids = O.decode_layer(q, K, V, [N, N], k, n_win=[W, W], combine=combine,
                                      pinned_prefix=pinned)
    outs = [np.load(f"{res}.{r}.npz") for r in range(world)]
    for r in range(world):
        np.testing.assert_allclose(outs[r]["out"], outs[0]["out"], atol=0)  # identical on every rank
        np.testing.assert_array_equal(outs[r]["idx"], outs[0]["idx"])
    idx = outs[0]["idx"]
    for b in range(q.shape[0]):
        for h in range(q.shape[1]):
            got = set(idx[b, h][idx[b, h] >= 0].tolist())
            want = ref_ids[b][h]
            if pinned:
                got |= set(range(min(pinned, N)))
            assert got == set(want.tolist())
    np.testing.assert_allclose(outs[0]["out"], ref_out, atol=1e-5)


def test_shard_range_partitions():
    from paper_2502_06766_b200.sharded import shard_range

    for n in (1, 7, 1000, 1 << 20):
        for w in (1, 2, 3, 8):
            parts = [shard_range(n, w, r) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
