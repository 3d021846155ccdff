"""CPU shard stages — TEST INFRASTRUCTURE ONLY.

A numpy implementation of the four per-rank stages of the token-range sharded protocol
(paper_2502_06766_b200/sharded.py; C ABI tkv_shard_* in include/tkv.h), used to exercise the
protocol's communication logic over torch.distributed/gloo on CPU (tests/test_sharded_gloo.py).
Semantics follow the reference per head (ann.py:154-167 selection with lower-id ties,
attention.py:107-167 joint/additive softmax), with scores rounded to f32 like the device's
and candidates packed as the device's 64-bit composites.
"""

from __future__ import annotations

import numpy as np
import torch

from . import oracle as O


class OracleStages:
    def __init__(self, B, Hq, Hkv, k, *, row_offset=0, scale=None, combine="joint", pinned_prefix=0,
                 head_dim=128):
        self.B, self.Hq, self.Hkv, self.k = B, Hq, Hkv, k
        self.G = Hq // Hkv
        self.row_offset = row_offset
        self.scale = scale if scale is not None else 1.0 / np.sqrt(head_dim)
        self.combine = combine
        self.pinned = pinned_prefix
        self.d = head_dim

    def _scores(self, q, K, b, h, n):
        return (K[b, h // self.G, :n].astype(np.float64) @ q[b, h].astype(np.float64)).astype(np.float32)

    def candidates(self, q, k_shard, n_ctx):
        q, K = q.numpy(), k_shard.numpy()
        out = np.zeros((self.B * self.Hq, self.k), dtype=np.uint64)
        for b in range(self.B):
            n = int(n_ctx[b])
            for h in range(self.Hq):
                s = self._scores(q, K, b, h, n)
                comp = O.composite(s, np.arange(n) + self.row_offset)
                top = comp[O.topk_by_composite(comp, min(self.k, n))]
                out[b * self.Hq + h, :len(top)] = top
        return torch.from_numpy(out.reshape(-1).view(np.int64).copy())

    def merge(self, gathered, n_shards, list_len=None):
        L = self.k if list_len is None else list_len
        g = gathered.numpy().view(np.uint64).reshape(n_shards, self.B * self.Hq, L)
        self.idx = np.full((self.B, self.Hq, self.k), -1, dtype=np.int32)
        self.scores = np.full((self.B, self.Hq, self.k), -np.inf, dtype=np.float32)
        self.meta = {}
        for bh in range(self.B * self.Hq):
            c = g[:, bh].reshape(-1)
            c = c[c != 0]
            top = c[O.topk_by_composite(c, min(self.k, len(c)))]
            gid = (~top & np.uint64(0xFFFFFFFF)).astype(np.int64)
            key = (top >> np.uint64(32)).astype(np.uint32)
            s = _key_to_score(key)
            b, h = divmod(bh, self.Hq)
            self.idx[b, h, :len(top)] = gid
            self.scores[b, h, :len(top)] = s
            self.meta[bh] = (float(s.max()) if len(s) else -np.inf, top.min() if len(top) else None, len(top))
        return torch.from_numpy(self.idx), torch.from_numpy(self.scores)

    def partial_attend(self, q, k_shard, v_shard, n_ctx, idx, scores):
        q, K, V = q.numpy(), k_shard.numpy(), v_shard.numpy()
        part = np.zeros((self.B * self.Hq, self.d + 1), dtype=np.float64)
        for b in range(self.B):
            n = int(n_ctx[b])
            for h in range(self.Hq):
                bh = b * self.Hq + h
                M, kth, kb = self.meta[bh]
                if kb == 0:
                    continue
                ids = self.idx[b, h, :kb].astype(np.int64)
                s = self.scores[b, h, :kb].astype(np.float64)
                loc = ids - self.row_offset
                own = (loc >= 0) & (loc < n)
                w = np.exp((s[own] - M) * self.scale)
                part[bh, 0] += w.sum()
                part[bh, 1:] += w @ V[b, h // self.G, loc[own]].astype(np.float64)
                # pinned rows [0, p) of this shard that the top-k did not select
                lo, hi = max(0, -self.row_offset), min(n, self.pinned - self.row_offset)
                if hi > lo:
                    sp = self._scores(q, K, b, h, n)[lo:hi]
                    comp = O.composite(sp, np.arange(lo, hi) + self.row_offset)
                    extra = comp < kth
                    w = np.exp((sp[extra].astype(np.float64) - M) * self.scale)
                    part[bh, 0] += w.sum()
                    part[bh, 1:] += w @ V[b, h // self.G, lo:hi][extra].astype(np.float64)
        return torch.from_numpy(part.astype(np.float32).reshape(-1))

    def finalize(self, q, k_shard, v_shard, n_ctx, n_win, partial):
        q, K, V = q.numpy(), k_shard.numpy(), v_shard.numpy()
        part = partial.numpy().reshape(self.B * self.Hq, self.d + 1).astype(np.float64)
        out = np.zeros((self.B, self.Hq, self.d), dtype=np.float32)
        for b in range(self.B):
            n = int(n_ctx[b])
            w_n = int(n_win[b]) if n_win is not None else 0
            for h in range(self.Hq):
                bh = b * self.Hq + h
                M, _, kb = self.meta[bh]
                l_c, o_c = part[bh, 0], part[bh, 1:]
                zc = M * self.scale
                kv = h // self.G
                wk = K[b, kv, n:n + w_n].astype(np.float64)
                wv = V[b, kv, n:n + w_n].astype(np.float64)
                sw = wk @ q[b, h].astype(np.float64) * self.scale
                if self.combine == "joint":
                    m = max([zc] if kb else [] + [], default=-np.inf)
                    m = max(m, sw.max()) if w_n else m
                    L = (l_c * np.exp(zc - m) if kb else 0.0) + np.exp(sw - m).sum()
                    num = (o_c * np.exp(zc - m) if kb else 0.0) + np.exp(sw - m) @ wv
                    out[b, h] = num / L
                else:
                    acc = o_c / l_c if kb else 0.0
                    if w_n:
                        e = np.exp(sw - sw.max())
                        acc = acc + (e @ wv) / e.sum()
                    out[b, h] = acc
        return torch.from_numpy(out)


def _key_to_score(key: np.ndarray) -> np.ndarray:
    key = key.astype(np.uint32)
    neg = (key & 0x80000000) == 0
    b = np.where(neg, ~key, key & 0x7FFFFFFF).astype(np.uint32)
    return b.view(np.float32)
