"""GPU parity of the per-head k-th + gather kernel (head_topk_kernel, select.cu; TKV_F_HEAD) at
any k — including the streamed case where one CTA's selected rows overflow its 8192-row shared
buffer — and of the kth_kernel + attend_cand path forced at small k (TKV_F_NO_HEAD)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from tests.conftest import sample_rows
from tests.test_gpu_parity import _check, _make, _run

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("B,Hq,Hkv,N,k,W,pin,head", [
    (1, 32, 8, 16384, 256, 0, 0, False),   # cfg1 shape on kth + attend_cand
    (1, 32, 8, 16384, 256, 0, 0, True),
    (1, 8, 2, 40000, 6000, 3, 0, True),    # C = 8 CTAs per head, large k
    (5, 32, 8, 24000, 9000, 0, 0, True),   # 160 heads → C = 1: 9000 selected rows stream through 8192
    (2, 16, 4, 9000, 700, 4, 40, True),    # pinned prefix + window
    (3, 8, 2, 3000, 300, 5, 0, True),      # ragged below (k > n_ctx for some entries)
])
def test_head_kernel_parity(cuda, B, Hq, Hkv, N, k, W, pin, head):
    rng = np.random.default_rng(7000 + N + k + int(head))
    q, K, V = _make(rng, B, Hq, Hkv, N + W + 8)
    n_ctx = [N] + [max(1, N - 997 * i) for i in range(1, B)]
    if B == 3:
        n_ctx = [3000, 100, 0]
    n_win = [W] * B
    out, idx, sc = _run(q, K, V, n_ctx, k, cuda, n_win=n_win, pinned_prefix=pin, head=head)
    torch.cuda.synchronize()
    _check(q, K, V, n_ctx, k, out, idx, sc, n_win=n_win, pinned=pin)


@pytest.mark.parametrize("k", [512, 2048])
def test_head_kernel_fallback(cuda, k):
    """Sampled rows far above the rest: the sampled threshold admits < k rows, the head kernel
    flags the heads and tail-launches re-scan → k-th → candidate-mode gather over all heads."""
    from oracle import oracle as O

    rng = np.random.default_rng(11 + k)
    B, Hq, Hkv, N = 1, 8, 2, 65536
    q, K, V = _make(rng, B, Hq, Hkv, N)
    K = O.to_bf16_f32(K * 0.01)
    rr = sample_rows(N, 1, k)  # the rows the sampled threshold scores (b = 0, kv head 1)
    K[0, 1, rr] = O.to_bf16_f32(np.sign(q[0, 4])[None, :] * 2.0 + K[0, 1, rr])
    out, idx, sc = _run(q, K, V, [N], k, cuda, head=True)
    torch.cuda.synchronize()
    _check(q, K, V, [N], k, out, idx, sc)


def test_head_kernel_search_sorted(cuda):
    """topk_search (no gather) through the head kernel, TopKResult order, = the default path."""
    from paper_2502_06766_b200 import topk_search
    from tests.test_gpu_parity import _dev

    rng = np.random.default_rng(23)
    q, K, _ = _make(rng, 2, 16, 4, 20000)
    qd, Kd = _dev(q, cuda), _dev(K, cuda)
    i1, s1 = topk_search(qd, Kd, [20000, 15000], 3000, head=True)
    i2, s2 = topk_search(qd, Kd, [20000, 15000], 3000, head=False)
    torch.cuda.synchronize()
    assert torch.equal(i1, i2) and torch.equal(s1, s2)
