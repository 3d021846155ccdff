"""GPU parity of the TMA + tcgen05 key scan (scan_tc.cu, the default; TKV_F_SCAN_HMMA selects scan.cu) against the oracle and
against the HMMA scan — same candidate contract, so the same selection must come out."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from tests.conftest import sample_rows
from tests.test_gpu_parity import _check, _dev, _make, _run

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("B,Hq,Hkv,N,k", [
    (1, 32, 8, 16384, 256),    # cfg1 shape
    (1, 4, 1, 1000, 10),       # partial last tile
    (2, 8, 8, 3000, 64),       # G = 1
    (1, 16, 2, 5000, 1),       # G = 8
    (1, 4, 4, 257, 257),       # k == N, unfiltered
    (64, 8, 8, 130, 17),       # many short segments per CTA: q-slot rotation
])
def test_tc_scan_parity(cuda, B, Hq, Hkv, N, k):
    rng = np.random.default_rng(3000 + N + k)
    q, K, V = _make(rng, B, Hq, Hkv, N)
    out, idx, sc = _run(q, K, V, [N] * B, k, cuda, tc_scan=True)
    torch.cuda.synchronize()
    _check(q, K, V, [N] * B, k, out, idx, sc)


@pytest.mark.parametrize("tc", [True, False])
def test_tc_scan_ragged_window(cuda, tc):
    rng = np.random.default_rng(77)
    B, Hq, Hkv, rows = 3, 8, 2, 4096
    q, K, V = _make(rng, B, Hq, Hkv, rows)
    n_ctx, n_win = [4090, 100, 1], [5, 0, 3]  # n_ctx + n_win <= rows (tkv.h precondition)
    out, idx, sc = _run(q, K, V, n_ctx, 300, cuda, n_win=n_win, tc_scan=tc)
    torch.cuda.synchronize()
    _check(q, K, V, n_ctx, 300, out, idx, sc, n_win=n_win)


@pytest.mark.parametrize("no_filter", [False, True])
def test_tc_scan_equals_hmma_scan(cuda, no_filter):
    rng = np.random.default_rng(123)
    q, K, V = _make(rng, 2, 32, 8, 65536)
    n_ctx = [65536, 40000]
    o1, i1, s1 = _run(q, K, V, n_ctx, 1024, cuda, tc_scan=True, no_filter=no_filter)
    o2, i2, s2 = _run(q, K, V, n_ctx, 1024, cuda, tc_scan=False, no_filter=no_filter)
    torch.cuda.synchronize()
    a, b = i1.cpu().numpy(), i2.cpu().numpy()
    diff = sum(len(set(a[x, h].tolist()) ^ set(b[x, h].tolist())) for x in range(2) for h in range(32))
    assert diff <= 4, diff  # only fp32 accumulation-order near-ties may differ
    assert float((o1 - o2).abs().max()) < 1e-3


def test_tc_scan_fallback(cuda):
    """Adversarial sample (see test_gpu_parity): the exactness fallback re-scans with the HMMA
    scan after the tcgen05 main pass; the result must still be exact."""
    from oracle import oracle as O

    rng = np.random.default_rng(9)
    B, Hq, Hkv, N, k = 1, 4, 1, 65536, 2048
    q, K, V = _make(rng, B, Hq, Hkv, N)
    K = O.to_bf16_f32(K * 0.01)
    rr = sample_rows(N, 0, k)  # the rows the sampled threshold scores (kv head 0)
    K[0, 0, rr] = O.to_bf16_f32(np.sign(q[0, 0])[None, :] * 2.0 + K[0, 0, rr])
    out, idx, sc = _run(q, K, V, [N], k, cuda, tc_scan=True)
    torch.cuda.synchronize()
    _check(q, K, V, [N], k, out, idx, sc)


def test_tc_scan_repeated_and_graph(cuda):
    """Persistent state (mbarriers, TMEM) is per launch: 20 back-to-back calls, then a graph."""
    from paper_2502_06766_b200 import ops

    rng = np.random.default_rng(5)
    q, K, V = _make(rng, 1, 32, 8, 32768)
    qd, Kd, Vd = _dev(q, cuda), _dev(K, cuda), _dev(V, cuda)
    n = torch.tensor([32768], dtype=torch.int32, device=cuda)
    prob = ops.make_problem(1, 32, 8, 32768, 32768, 512, tc_scan=True)
    ws = ops.Workspace(prob, cuda)
    ref = None
    for _ in range(20):
        out, idx, _ = ops.topk_decode_attention(qd, Kd, Vd, n, 512, workspace=ws, tc_scan=True, max_ctx=32768)
        if ref is None:
            ref = (out.clone(), idx.clone())
    torch.cuda.synchronize()
    same = lambda a, b: torch.equal(a.sort(-1).values, b.sort(-1).values)  # noqa: E731  (emission order varies)
    assert same(idx, ref[1]) and float((out - ref[0]).abs().max()) < 1e-5
    out_g = torch.empty_like(out)
    idx_g = torch.empty_like(idx)
    sc_g = torch.empty((1, 32, 512), dtype=torch.float32, device=cuda)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g):
            ops.topk_decode_attention(qd, Kd, Vd, n, 512, workspace=ws, tc_scan=True, max_ctx=32768,
                                      out=out_g, idx=idx_g, scores=sc_g)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert same(idx_g, ref[1]) and float((out_g - ref[0]).abs().max()) < 1e-5


@pytest.mark.parametrize("B,Hq,Hkv,N,k,parts", [
    (1, 32, 8, 16384, 256, 4),
    (2, 8, 4, 5000, 300, 3),     # uneven split of 8 segments, ragged below
    (1, 16, 2, 5000, 1, 2),
])
def test_overlapped_parts_parity(cuda, B, Hq, Hkv, N, k, parts):
    """The part-overlapped pipeline (scan of part i+1 beside k-th + gather of part i on a side
    stream) is exact, for every head range, also with sorted output and a window."""
    rng = np.random.default_rng(4000 + N + parts)
    q, K, V = _make(rng, B, Hq, Hkv, N + 8)
    n_ctx = [N] + [N - 777] * (B - 1)
    n_win = [3] * B
    out, idx, sc = _run(q, K, V, n_ctx, k, cuda, n_win=n_win, parts=parts, sorted=True)
    torch.cuda.synchronize()
    _check(q, K, V, n_ctx, k, out, idx, sc, n_win=n_win)
    out1, idx1, _ = _run(q, K, V, n_ctx, k, cuda, n_win=n_win, parts=1, sorted=True)
    torch.cuda.synchronize()
    assert torch.equal(idx, idx1)  # sorted: identical order
    assert float((out - out1).abs().max()) < 1e-5


def test_overlapped_parts_fallback_and_graph(cuda):
    """A failing head in a later part triggers that part's own device-side fallback; the whole
    overlapped layer is capturable in a CUDA graph (fork/join events)."""
    from oracle import oracle as O
    from paper_2502_06766_b200 import ops

    rng = np.random.default_rng(19)
    B, Hq, Hkv, N, k = 1, 16, 4, 65536, 2048
    q, K, V = _make(rng, B, Hq, Hkv, N)
    K = O.to_bf16_f32(K * 0.01)
    rr = sample_rows(N, 3, k)  # adversarial sample for kv head 3 only (the last part)
    K[0, 3, rr] = O.to_bf16_f32(np.sign(q[0, 12])[None, :] * 2.0 + K[0, 3, rr])
    out, idx, sc = _run(q, K, V, [N], k, cuda, parts=4)
    torch.cuda.synchronize()
    _check(q, K, V, [N], k, out, idx, sc)
    qd, Kd, Vd = _dev(q, cuda), _dev(K, cuda), _dev(V, cuda)
    n = torch.tensor([N], dtype=torch.int32, device=cuda)
    prob = ops.make_problem(B, Hq, Hkv, N, N, k, parts=4)
    ws = ops.Workspace(prob, cuda)
    out_g = torch.empty_like(out)
    idx_g = torch.empty_like(idx)
    sc_g = torch.empty_like(sc)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ops.topk_decode_attention(qd, Kd, Vd, n, k, workspace=ws, max_ctx=N, parts=4, out=out_g, idx=idx_g,
                                  scores=sc_g)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            ops.topk_decode_attention(qd, Kd, Vd, n, k, workspace=ws, max_ctx=N, parts=4, out=out_g,
                                      idx=idx_g, scores=sc_g)
    for _ in range(3):
        out_g.zero_()
        g.replay()
    torch.cuda.synchronize()
    _check(q, K, V, [N], k, out_g, idx_g, sc_g)


@pytest.mark.parametrize("B,Hq,Hkv,N,k,W,pin", [
    (1, 32, 8, 16384, 256, 0, 0),
    (3, 8, 2, 3000, 300, 5, 0),     # ragged, k > n_ctx for one entry, window
    (2, 16, 4, 9000, 700, 3, 40),   # pinned prefix
    (4, 4, 1, 2000, 1999, 0, 0),    # k = N - 1: heads span several CTA ranges
])
def test_list_gather_parity(cuda, B, Hq, Hkv, N, k, W, pin):
    """Filter pass + balanced list gather (TKV_F_GATHER_LIST) against the oracle, including an
    empty context (n_ctx = 0) whose heads must still be finalised."""
    rng = np.random.default_rng(5000 + N + k)
    q, K, V = _make(rng, B, Hq, Hkv, N + W + 8)
    n_ctx = [N] + [max(1, N - 700 * i) for i in range(1, B)]
    if B == 3:
        n_ctx = [3000, 100, 0]  # an empty context (the window alone is attended)
    n_win = [W] * B
    out, idx, sc = _run(q, K, V, n_ctx, k, cuda, n_win=n_win, pinned_prefix=pin, list_gather=True)
    torch.cuda.synchronize()
    _check(q, K, V, n_ctx, k, out, idx, sc, n_win=n_win, pinned=pin)
    out2, idx2, _ = _run(q, K, V, n_ctx, k, cuda, n_win=n_win, pinned_prefix=pin)
    torch.cuda.synchronize()
    assert float((out - out2).abs().max()) < 1e-5
