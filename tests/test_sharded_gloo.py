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


def _data(seed=0, B=2, Hq=8, Hkv=2, N=997, W=3, skew=False):
    sys.path.insert(0, str(ROOT))
    from oracle import oracle as O

    rng = np.random.default_rng(seed)
    q = O.to_bf16_f32(rng.standard_normal((B, Hq, 128), dtype=np.float32))
    K = O.to_bf16_f32(rng.standard_normal((B, Hkv, N + W, 128), dtype=np.float32))
    V = O.to_bf16_f32(rng.standard_normal((B, Hkv, N + W, 128), dtype=np.float32))
    K[:, :, 100:900:50] = K[:, :, 7:8]  # exact duplicates spread over shards: lower-id ties
    if skew:  # the relevant rows concentrate in the first quarter (rank 0's shard)
        K[:, :, :N // 4] *= 4.0
    return q, K, V, N, W


def _worker(rank, world, port, k, combine, pinned, result_path, c=None, skew=False):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.shard_stages import OracleStages
    from paper_2502_06766_b200.sharded import narrow_k, shard_range, sharded_topk_attention

    q, K, V, N, W = _data(skew=skew)
    B, Hq, Hkv = q.shape[0], q.shape[1], K.shape[1]
    lo, hi = shard_range(N, world, rank)
    ks = np.concatenate([K[:, :, lo:hi], K[:, :, N:N + W]], axis=2)
    vs = np.concatenate([V[:, :, lo:hi], V[:, :, N:N + W]], axis=2)
    st = OracleStages(B, Hq, Hkv, k, row_offset=lo, combine=combine, pinned_prefix=pinned)
    narrow = None
    if c is not None:
        narrow = OracleStages(B, Hq, Hkv, narrow_k(k, world, c), row_offset=lo, combine=combine,
                              pinned_prefix=pinned)
    stats = {}
    out, idx, sc = sharded_topk_attention(st, torch.from_numpy(q), torch.from_numpy(ks),
                                          torch.from_numpy(vs), [hi - lo] * B, [W] * B,
                                          narrow=narrow, stats=stats)
    np.savez(f"{result_path}.{rank}.npz", out=out.numpy(), idx=idx.numpy(),
             exact=np.array(stats.get("narrow_exact") is True))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,k,combine,pinned,c,skew,narrow_exact", [
    (2, 40, "joint", 0, None, False, False),
    (2, 7, "additive", 5, None, False, False),
    (4, 100, "joint", 3, None, False, False),
    (4, 2000, "joint", 0, None, False, False),  # k > N: every row, clamped
    # narrow exchange (each rank sends its top ceil(c·k/G)): exact on i.i.d. data ...
    (2, 40, "joint", 0, 1.5, False, True),
    (4, 100, "joint", 3, 2.0, False, True),
    # ... and falls back to the full-k exchange when one shard holds most of the top-k
    (4, 100, "joint", 0, 1.5, True, False),
    (4, 2000, "joint", 0, 1.5, False, True),  # k > N: each shard fits in k', nothing withheld
])
def test_sharded_equals_unsharded(tmp_path, world, k, combine, pinned, c, skew, narrow_exact):
    from oracle import oracle as O

    port = 29400 + world * 10 + (k % 7) + (0 if c is None else 3 + int(skew))
    res = str(tmp_path / "r")
    mp.start_processes(_worker, args=(world, port, k, combine, pinned, res, c, skew),
                       nprocs=world, join=True, start_method="spawn")
    q, K, V, N, W = _data(skew=skew)
    ref_out, ref_ids = O.decode_layer(q, K, V, [N, N], k, n_win=[W, W], combine=combine,
                                      pinned_prefix=pinned)
    outs = [np.load(f"{res}.{r}.npz") for r in range(world)]
    for r in range(world):
        np.testing.assert_allclose(outs[r]["out"], outs[0]["out"], atol=0)  # identical on every rank
        np.testing.assert_array_equal(outs[r]["idx"], outs[0]["idx"])
    assert all(bool(o["exact"]) == narrow_exact for o in outs)
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


def test_narrow_exchange_exact_rule():
    """The exactness rule on hand-made composites (unsigned 64-bit order; most real composites
    have the top bit set, so a signed compare would be wrong)."""
    from paper_2502_06766_b200.sharded import narrow_exchange_exact, narrow_k

    hi = 1 << 63

    def g(*ranks):  # ranks of one head each, kk slots, 0 = empty
        a = np.array([v for r in ranks for v in r], dtype=np.uint64)
        return torch.from_numpy(a.view(np.int64))

    # k = 3, kk = 2. Rank 0 full (floor hi+50), rank 1 full (floor hi+10): T = hi+50;
    # candidates >= T: hi+90, hi+50, hi+60 -> 3 >= k: exact
    assert bool(narrow_exchange_exact(g([hi + 90, hi + 50], [hi + 60, hi + 10]), 2, 3, 2).all())
    # rank 1's floor above rank 0's second: T = hi+60 -> only hi+90, hi+70, hi+60 ... count 3
    assert bool(narrow_exchange_exact(g([hi + 90, hi + 5], [hi + 70, hi + 60]), 2, 3, 2).all())
    # T = hi+80 (rank 0 floor); only hi+90, hi+80 >= T -> rank 0 may withhold a row above
    # rank 1's hi+10 which the merged top-3 would need: not exact
    assert not bool(narrow_exchange_exact(g([hi + 90, hi + 80], [5, 0]), 2, 3, 2).all())
    # no rank full: everything was sent
    assert bool(narrow_exchange_exact(g([hi + 90, 0], [7, 0]), 2, 3, 2).all())
    # negative-score composites (top bit clear) sort below positive ones: T = hi+2 (rank 1's
    # floor), only 2 candidates >= T, rank 1 may withhold rows above rank 0's 12
    assert not bool(narrow_exchange_exact(g([hi + 1, 12], [hi + 3, hi + 2]), 2, 3, 2).all())
    # per head: [world, BH=2, kk=2]; head 0 exact, head 1 not
    r0 = [hi + 90, hi + 50, hi + 90, hi + 80]
    r1 = [hi + 60, hi + 10, 5, 0]
    assert narrow_exchange_exact(g(r0, r1), 2, 3, 2).tolist() == [True, False]
    assert narrow_k(16384, 8) == 3072 and narrow_k(100, 1) == 100 and narrow_k(10, 4, 2.0) == 5


def test_publish_layout_views_tile_the_buffer():
    """DeviceShardedStep's publish buffer (narrow | full | bounds | partial): the views are
    disjoint, in order, and cover the buffer; the pointer arrays add the same offsets."""
    sys.path.insert(0, str(ROOT))
    from paper_2502_06766_b200.sharded import _PublishLayout, _pointer_arrays, _views

    B, Hq, k, kk = 2, 8, 100, 37
    lay = _PublishLayout(B, Hq, k, kk)
    buf = torch.zeros(lay.nbytes, dtype=torch.uint8)
    nar, full, bound, part = _views(buf, lay)
    assert nar.numel() == B * Hq * kk and full.numel() == B * Hq * k and bound.numel() == B * Hq * 3
    assert part.numel() == B * Hq * 129
    base = buf.data_ptr()
    offs = [t.data_ptr() - base for t in (nar, full, bound, part)]
    ends = [o + t.numel() * t.element_size() for o, t in zip(offs, (nar, full, bound, part))]
    assert offs[0] == 0 and all(ends[i] == offs[i + 1] for i in range(3)) and ends[3] == lay.nbytes
    ptrs = _pointer_arrays([base, base + 1000], lay, "cpu")
    for arr, o in zip(ptrs, offs):
        assert arr.tolist() == [base + o, base + 1000 + o]
