"""GPU parity of the cluster k-th + gather kernel (clus_topk_kernel, select.cu; TKV_F_CLUSTER):
one 4-CTA thread-block cluster per head finds the exact k-th composite (members of the
threshold bucket exchanged over distributed shared memory), gathers the selected V rows and
finishes the head (pinned prefix, window, joint / additive) — against the CPU oracle, and
bit-for-bit against the k-th kernel + candidate gather on the selected ids."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from tests.conftest import sample_rows
from tests.test_gpu_parity import _check, _dev, _make, _run

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("B,Hq,Hkv,N,k,W,pin,combine", [
    (1, 32, 8, 16384, 256, 0, 0, "joint"),     # cfg1 shape
    (1, 32, 8, 131072, 2048, 0, 0, "joint"),   # cfg2 shape
    (1, 8, 2, 40000, 6000, 3, 0, "joint"),     # several compaction batches per CTA
    (2, 16, 4, 9000, 700, 4, 40, "joint"),     # pinned prefix + window
    (2, 16, 4, 9000, 700, 4, 40, "additive"),
    (3, 8, 2, 3000, 300, 5, 0, "joint"),       # ragged: k > n_ctx, an empty entry
    (1, 4, 1, 1000, 10, 0, 0, "joint"),        # GQA 4, tiny k
    (1, 16, 2, 5000, 1, 2, 0, "joint"),        # GQA 8, k = 1
    (1, 4, 4, 257, 257, 0, 0, "joint"),        # k == N: every candidate selected
])
def test_cluster_kernel_parity(cuda, B, Hq, Hkv, N, k, W, pin, combine):
    rng = np.random.default_rng(9100 + N + k + W)
    q, K, V = _make(rng, B, Hq, Hkv, N + W + 8)
    n_ctx = [N] + [max(1, N - 997 * i) for i in range(1, B)]
    if B == 3:
        n_ctx = [3000, 100, 0]
    n_win = [W] * B
    out, idx, sc = _run(q, K, V, n_ctx, k, cuda, n_win=n_win, pinned_prefix=pin, combine=combine,
                        head="cluster")
    torch.cuda.synchronize()
    _check(q, K, V, n_ctx, k, out, idx, sc, n_win=n_win, combine=combine, pinned=pin)


def test_cluster_matches_kth_path(cuda):
    """Same selected set (sorted ids) and the same outputs to fp32 summation order as the
    k-th kernel + candidate gather."""
    rng = np.random.default_rng(77)
    q, K, V = _make(rng, 2, 32, 8, 20000)
    qd, Kd, Vd = _dev(q, cuda), _dev(K, cuda), _dev(V, cuda)
    from paper_2502_06766_b200 import topk_decode_attention

    o1, i1, s1 = topk_decode_attention(qd, Kd, Vd, [20000, 17000], 1500, head="cluster", sorted=True)
    o2, i2, s2 = topk_decode_attention(qd, Kd, Vd, [20000, 17000], 1500, head=False, sorted=True)
    torch.cuda.synchronize()
    assert torch.equal(i1, i2) and torch.equal(s1, s2)
    assert float((o1 - o2).abs().max()) <= 1e-5


def test_cluster_duplicate_rows_tie_to_lower_id(cuda):
    """Many exactly equal scores straddle the k-th: the bucket's members decide by row id."""
    rng = np.random.default_rng(5)
    B, Hq, Hkv, N, k = 1, 8, 2, 12000, 900
    q, K, V = _make(rng, B, Hq, Hkv, N)
    K[0, :, 3000:6000] = K[0, :, 3000:3001]  # 3000 identical rows per kv head
    out, idx, sc = _run(q, K, V, [N], k, cuda, head="cluster")
    torch.cuda.synchronize()
    _check(q, K, V, [N], k, out, idx, sc)


@pytest.mark.parametrize("k", [512, 2048])
def test_cluster_kernel_fallback(cuda, k):
    """Sampled rows far above the rest: the sampled threshold admits < k rows; the cluster kernel
    flags the heads and tail-launches re-scan → k-th → candidate-mode gather over all heads."""
    from oracle import oracle as O
    from paper_2502_06766_b200 import ops

    rng = np.random.default_rng(31 + k)
    B, Hq, Hkv, N = 1, 8, 2, 65536
    q, K, V = _make(rng, B, Hq, Hkv, N)
    K = O.to_bf16_f32(K * 0.01)
    rr = sample_rows(N, 1, k)
    K[0, 1, rr] = O.to_bf16_f32(np.sign(q[0, 4])[None, :] * 2.0 + K[0, 1, rr])
    prob = ops.make_problem(B, Hq, Hkv, N, N, k, head="cluster")
    ws = ops.Workspace(prob, cuda)
    before = ws.fallbacks(prob)
    out, idx, sc = _run(q, K, V, [N], k, cuda, head="cluster", workspace=ws)
    torch.cuda.synchronize()
    assert ws.fallbacks(prob) > before, "the adversarial cache did not trigger the fallback"
    _check(q, K, V, [N], k, out, idx, sc)


def test_cluster_search_sorted(cuda):
    """topk_search (no gather) through the cluster kernel, TopKResult order, = the default path."""
    from paper_2502_06766_b200 import topk_search

    rng = np.random.default_rng(29)
    q, K, _ = _make(rng, 2, 16, 4, 20000)
    qd, Kd = _dev(q, cuda), _dev(K, cuda)
    i1, s1 = topk_search(qd, Kd, [20000, 15000], 3000, head="cluster")
    i2, s2 = topk_search(qd, Kd, [20000, 15000], 3000, head=False)
    torch.cuda.synchronize()
    assert torch.equal(i1, i2) and torch.equal(s1, s2)


def test_cluster_graph_replay(cuda):
    """Captured once into a CUDA graph and replayed: identical results every replay (the
    kernel leaves no per-call state behind: no tickets, output counters reset upstream)."""
    from paper_2502_06766_b200 import ops, topk_decode_attention

    rng = np.random.default_rng(3)
    q, K, V = _make(rng, 1, 32, 8, 30000)
    qd, Kd, Vd = _dev(q, cuda), _dev(K, cuda), _dev(V, cuda)
    nc = torch.tensor([30000], dtype=torch.int32, device=cuda)
    k = 1024
    out = torch.empty((1, 32, 128), dtype=torch.float32, device=cuda)
    idx = torch.empty((1, 32, k), dtype=torch.int32, device=cuda)
    sc = torch.empty((1, 32, k), dtype=torch.float32, device=cuda)
    prob = ops.make_problem(1, 32, 8, 30000, 30000, k, head="cluster")
    ws = ops.Workspace(prob, cuda)
    kw = dict(max_ctx=30000, out=out, idx=idx, scores=sc, workspace=ws, head="cluster", sorted=True)
    topk_decode_attention(qd, Kd, Vd, nc, k, **kw)
    torch.cuda.synchronize()
    ref = (out.clone(), idx.clone())
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side), torch.cuda.graph(g, stream=side):
        topk_decode_attention(qd, Kd, Vd, nc, k, **kw)
    torch.cuda.current_stream().wait_stream(side)
    for _ in range(5):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(idx, ref[1])
        # summation order follows the scan's candidate order (reservation atomics): fp32-close
        assert float((out - ref[0]).abs().max()) <= 1e-6
