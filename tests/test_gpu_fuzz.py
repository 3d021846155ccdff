"""GPU: seeded random configurations across every option of the layer call, each checked
against the CPU oracle (ids up to near-ties, outputs within the stated tolerances)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from tests.test_gpu_parity import _check, _make, _run

pytestmark = pytest.mark.gpu


def _config(seed: int):
    r = np.random.default_rng(seed)
    G = int(r.choice([1, 2, 4, 8]))
    Hkv = int(r.choice([1, 2, 4, 8])) if G < 8 else int(r.choice([1, 2]))
    B = int(r.integers(1, 4))
    N = int(r.choice([64, 300, 1000, 2500, 7000, 20000]))
    k = int(r.choice([1, 7, 64, 256, 1000, N - 1, N + 5]))
    k = max(1, k)
    W = int(r.choice([0, 0, 3, 40]))
    pin = int(r.choice([0, 0, 10, 300]))
    combine = str(r.choice(["joint", "additive"]))
    n_ctx = [N] + [int(r.integers(1, N + 1)) for _ in range(B - 1)]
    opts = dict(
        sorted=bool(r.random() < 0.3) and k <= 16384,
        parts=int(r.choice([0, 0, 2, 3])),
        list_gather=bool(r.random() < 0.3),
        tc_scan=bool(r.random() < 0.8),
        no_filter=bool(r.random() < 0.15),
    )
    return B, G * Hkv, Hkv, N, k, W, pin, combine, n_ctx, opts


@pytest.mark.parametrize("seed", range(30))
def test_fuzz_against_oracle(cuda, seed):
    B, Hq, Hkv, N, k, W, pin, combine, n_ctx, opts = _config(seed)
    rng = np.random.default_rng(10_000 + seed)
    q, K, V = _make(rng, B, Hq, Hkv, N + W + 4)
    n_win = [W] * B
    out, idx, sc = _run(q, K, V, n_ctx, k, cuda, n_win=n_win, pinned_prefix=pin, combine=combine, **opts)
    torch.cuda.synchronize()
    _check(q, K, V, n_ctx, k, out, idx, sc, n_win=n_win, combine=combine, pinned=pin)
