"""GPU: the device-driven sharded step (DeviceShardedStep) with the exchange emulated on one GPU
(LocalExchange: every rank's publish buffer in this process, the ranks' stages run one after
another — no kernel waits on another). Checks: ids and outputs equal the unsharded call; the
narrow-vs-full choice is made per head on the device (i.i.d. data → narrow everywhere; data
whose relevant rows sit in one shard → full lists for those heads, still exact); the whole
emulated step (all ranks, all stages) captures into one CUDA graph and replays exactly."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from tests.test_gpu_parity import _dev, _make

pytestmark = pytest.mark.gpu


def _setup(cuda, G, skew, N=40000, k=512, W=5, B=1, Hq=32, Hkv=8, seed=23):
    from paper_2502_06766_b200 import CudaStages, DeviceShardedStep, LocalExchange, narrow_k, shard_range

    rng = np.random.default_rng(seed)
    q, K, V = _make(rng, B, Hq, Hkv, N + W)
    if skew:
        K[:, :, : N // G] *= 4.0
    kk = narrow_k(k, G)
    exch = LocalExchange(G, B, Hq, k, kk, cuda)
    ranks = []
    for g in range(G):
        lo, hi = shard_range(N, G, g)
        ks = np.concatenate([K[:, :, lo:hi], K[:, :, N:N + W]], axis=2)
        vs = np.concatenate([V[:, :, lo:hi], V[:, :, N:N + W]], axis=2)
        st = CudaStages(B, Hq, Hkv, ks.shape[2], hi - lo, k, row_offset=lo, device=cuda)
        nc = torch.tensor([hi - lo] * B, dtype=torch.int32, device=cuda)
        ranks.append((DeviceShardedStep(st, exch, g, kk), _dev(ks, cuda), _dev(vs, cuda), nc))
    nw = torch.tensor([W] * B, dtype=torch.int32, device=cuda)
    return q, K, V, N, k, W, ranks, nw


def _emulated_step(qd, ranks, nw):
    """All ranks' device-driven stages, rank after rank per phase (the barriers' order)."""
    for st, ks, vs, nc in ranks:
        st.publish_candidates(qd, ks, nc)
    res = []
    for st, ks, vs, nc in ranks:
        res.append(st.merge_and_partial(qd, ks, vs, nc))
    outs = [st.combine(qd, ks, vs, nc, nw) for st, ks, vs, nc in ranks]
    return outs, res


@pytest.mark.parametrize("G,skew", [(2, False), (4, False), (8, False), (4, True), (8, True)])
def test_device_sharded_step_equals_unsharded(cuda, G, skew):
    from paper_2502_06766_b200 import topk_decode_attention

    q, K, V, N, k, W, ranks, nw = _setup(cuda, G, skew)
    qd = _dev(q, cuda)
    out1, idx1, _ = topk_decode_attention(qd, _dev(K, cuda), _dev(V, cuda), [N], k, n_win=[W])
    outs, res = _emulated_step(qd, ranks, nw)
    torch.cuda.synchronize()
    ref = idx1.cpu().numpy()
    for (st, *_), (idx, sc), out in zip(ranks, res, outs):
        a = idx.cpu().numpy()
        for h in range(a.shape[1]):
            assert set(a[0, h].tolist()) == set(ref[0, h].tolist())
        assert float((out - out1).abs().max()) < 1e-5
        used = st.used_full.cpu().numpy()
        if not skew:
            assert used.sum() == 0, "i.i.d. data must merge from the narrow lists"
    if skew:
        assert ranks[0][0].used_full.cpu().numpy().sum() > 0, "skewed data must trip the narrow rule"


def test_device_sharded_step_graph_capture(cuda):
    """The device-driven step has no host round trip: the whole emulated step (G = 4 ranks)
    captures into one CUDA graph; replays equal the eager results, including after the query
    changes in place."""
    from paper_2502_06766_b200 import topk_decode_attention

    G = 4
    q, K, V, N, k, W, ranks, nw = _setup(cuda, G, skew=False)
    qd = _dev(q, cuda)
    _emulated_step(qd, ranks, nw)  # warm-up (lazy library state outside the capture)
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side), torch.cuda.graph(g, stream=side):
        outs, res = _emulated_step(qd, ranks, nw)
    torch.cuda.current_stream().wait_stream(side)
    rng = np.random.default_rng(5)
    for rep in range(3):
        q2 = _make(rng, 1, 32, 8, 1)[0]
        qd.copy_(_dev(q2, cuda))
        g.replay()
        torch.cuda.synchronize()
        out1, idx1, _ = topk_decode_attention(qd, _dev(K, cuda), _dev(V, cuda), [N], k, n_win=[W])
        torch.cuda.synchronize()
        ref = idx1.cpu().numpy()
        for (idx, _), out in zip(res, outs):
            a = idx.cpu().numpy()
            for h in range(a.shape[1]):
                assert set(a[0, h].tolist()) == set(ref[0, h].tolist())
            assert float((out - out1).abs().max()) < 1e-5


# TKV_SHARD_FUZZ="start:count" widens the sweep (default 0:24)
_F0, _FN = (int(v) for v in __import__("os").environ.get("TKV_SHARD_FUZZ", "0:24").split(":"))


@pytest.mark.parametrize("seed", range(_F0, _F0 + _FN))
def test_device_sharded_step_fuzz(cuda, seed):
    """Random shard counts (uneven shards included), batch, GQA shapes, k from 1 to beyond a
    shard's rows and beyond N, windows, skew and exact cross-shard ties (duplicated rows): the
    emulated device-driven step gives the unsharded call's ids and outputs."""
    from paper_2502_06766_b200 import topk_decode_attention

    r = np.random.default_rng(seed)
    G = int(r.choice([2, 3, 4, 8]))
    B = int(r.integers(1, 3))
    Hkv = int(r.choice([1, 2, 8]))
    Hq = Hkv * int(r.choice([1, 4]))
    N = int(r.choice([3001, 20000, 70000]))
    k = int(r.choice([1, 50, 700, 4096, N + 5]))
    W = int(r.choice([0, 3]))
    skew = bool(r.random() < 0.3)
    q, K, V, N, k, W, ranks, nw = _setup(cuda, G, skew, N=N, k=k, W=W, B=B, Hq=Hq, Hkv=Hkv, seed=100 + seed)
    if r.random() < 0.3:  # duplicated rows across shard boundaries: ties resolved by the lower id
        src = r.integers(0, N, size=4)
        for b in range(B):
            for h in range(Hkv):
                K[b, h, r.integers(0, N, size=N // 5)] = K[b, h, r.choice(src)]
        q, K, V, N, k, W, ranks, nw = _rebuild(cuda, G, q, K, V, N, k, W, B, Hq, Hkv)
    qd = _dev(q, cuda)
    out1, idx1, _ = topk_decode_attention(qd, _dev(K, cuda), _dev(V, cuda), [N] * B, k, n_win=[W] * B)
    outs, res = _emulated_step(qd, ranks, nw)
    torch.cuda.synchronize()
    ref = idx1.cpu().numpy()
    for (idx, sc), out in zip(res, outs):
        a = idx.cpu().numpy()
        for b in range(B):
            for h in range(Hq):
                assert set(a[b, h].tolist()) == set(ref[b, h].tolist()), (b, h)
        assert float((out - out1).abs().max()) < 2e-5


def _rebuild(cuda, G, q, K, V, N, k, W, B, Hq, Hkv):
    """_setup's per-rank state for given arrays (after the data was modified)."""
    from paper_2502_06766_b200 import CudaStages, DeviceShardedStep, LocalExchange, narrow_k, shard_range

    kk = narrow_k(k, G)
    exch = LocalExchange(G, B, Hq, k, kk, cuda)
    ranks = []
    for g in range(G):
        lo, hi = shard_range(N, G, g)
        ks = np.concatenate([K[:, :, lo:hi], K[:, :, N:N + W]], axis=2)
        vs = np.concatenate([V[:, :, lo:hi], V[:, :, N:N + W]], axis=2)
        st = CudaStages(B, Hq, Hkv, ks.shape[2], hi - lo, k, row_offset=lo, device=cuda)
        nc = torch.tensor([hi - lo] * B, dtype=torch.int32, device=cuda)
        ranks.append((DeviceShardedStep(st, exch, g, kk), _dev(ks, cuda), _dev(vs, cuda), nc))
    nw = torch.tensor([W] * B, dtype=torch.int32, device=cuda)
    return q, K, V, N, k, W, ranks, nw
