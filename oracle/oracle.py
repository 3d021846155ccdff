"""CPU oracle — TEST INFRASTRUCTURE ONLY (never imported by the product package).

A plain numpy restatement of the reference's top-k decode-attention path
(/root/reference/pkg/src/topk_kv), used by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs as the checker. Every function cites the reference
file:line it restates. Parity of this restatement is pinned against golden vectors produced
by importing the live reference (tests/golden/make_golden.py → tests/golden/*.npz,
checked by tests/test_oracle_golden.py).

Numerics: like the reference, scores and softmax are float64 and outputs float32. The
reference's scan (ann_kernels.py:31-47) sums strictly left to right; `ip_scores_all` below
uses a BLAS f64 matvec. For bf16-representable inputs (all parity inputs) every product has
<= 16 significant bits and a 128-term f64 sum of such products is exact in any order, so the
two agree bit-for-bit; `ip_scores_strict` keeps the literal loop for the cross-check test.
"""

from __future__ import annotations

import numpy as np

DTYPE = np.float32


# ------------------------------------------------------------------------------ scan
def ip_scores_strict(keys: np.ndarray, q: np.ndarray) -> np.ndarray:
    """ann_kernels.py:31-47 — strict left-to-right f64 dot per row (small inputs only)."""
    n, d = keys.shape
    out = np.empty(n, dtype=np.float64)
    for i in range(n):
        s = 0.0
        for j in range(d):
            s += float(keys[i, j]) * float(q[j])
        out[i] = s
    return out


def ip_scores_all(keys: np.ndarray, q: np.ndarray) -> np.ndarray:
    """ann_kernels.py:40-47 — f64 inner product of q with every key row."""
    return np.asarray(keys, dtype=np.float64) @ np.asarray(q, dtype=np.float64)


# ------------------------------------------------------------------------------ select
def flat_topk_from_scores(s: np.ndarray, k: int) -> tuple[np.ndarray, np.ndarray]:
    """ann.py:154-167 (_flat_topk) on precomputed f64 scores: exact top-k, ties to the lower
    row id, ordered score-desc / id-asc. Returns (vals f32, ids i64)."""
    n = s.shape[0]
    k = min(k, n)
    if k == n:
        order = np.lexsort((np.arange(n), -s))  # ann.py:158-159
    else:
        part = np.argpartition(-s, k - 1)[:k]  # ann.py:161
        thresh = s[part].min()  # ann.py:162
        above = np.flatnonzero(s > thresh)  # ann.py:163
        ties = np.flatnonzero(s == thresh)[: k - above.size]  # ann.py:164
        cand = np.concatenate([above, ties])  # ann.py:165
        order = cand[np.lexsort((cand, -s[cand]))]  # ann.py:166
    return s[order].astype(DTYPE), order.astype(np.int64)


def flat_topk(keys: np.ndarray, q: np.ndarray, k: int) -> tuple[np.ndarray, np.ndarray]:
    """ann.py:154-167 (_flat_topk) including its scan."""
    return flat_topk_from_scores(ip_scores_all(keys, q), k)


# ------------------------------------------------------------------------------ attend
def joint_attend(s_ctx, v_ctx, s_gen, v_gen, combine: str) -> np.ndarray:
    """attention.py:107-122 (_joint_attend) — scores already scaled, f64 throughout."""
    if combine == "joint":
        scores = np.concatenate([s_ctx, s_gen])
        scores = scores - scores.max()
        w = np.exp(scores)
        num = w[: len(s_ctx)] @ v_ctx + w[len(s_ctx):] @ v_gen
        return (num / w.sum()).astype(DTYPE)
    if combine == "additive":
        out = np.zeros(v_ctx.shape[1] if len(v_ctx) else v_gen.shape[1])
        for s, v in ((s_ctx, v_ctx), (s_gen, v_gen)):
            if len(s):
                e = np.exp(s - s.max())
                out = out + (e @ v) / e.sum()
        return out.astype(DTYPE)
    raise ValueError(f"unknown combine mode {combine!r}")


def topk_attend(q, keys, values, win_keys, win_values, k: int, combine: str = "joint",
                pinned_prefix: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """attention.py:125-167 (topk_attend) for a flat index over `keys` with in-memory values.
    Returns (out f32 (d,), retrieved ids i64 as logged at attention.py:155-156)."""
    if k < 1:
        raise ValueError("k must be >= 1")
    n, d = keys.shape
    k = min(k, n)  # attention.py:147-149
    _, ids = flat_topk(keys, q, k)  # attention.py:150
    if pinned_prefix > 0:  # attention.py:152-154
        pinned = np.arange(min(pinned_prefix, n), dtype=np.int64)
        ids = np.unique(np.concatenate([pinned, ids]))
    q64 = np.asarray(q, dtype=np.float64)
    scale = 1.0 / np.sqrt(d)  # attention.py:159
    s_ctx = (np.asarray(keys, dtype=np.float64)[ids] @ q64) * scale  # attention.py:160
    v_ctx = np.asarray(values, dtype=np.float64)[ids]  # attention.py:161
    wk = np.asarray(win_keys, dtype=np.float64).reshape(-1, d)
    wv = np.asarray(win_values, dtype=np.float64).reshape(-1, d)
    s_gen = (wk @ q64) * scale  # attention.py:165
    return joint_attend(s_ctx, v_ctx, s_gen, wv, combine), ids


def attend_over_ids(q, keys, values, ids, win_keys, win_values, combine: str = "joint",
                    scale: float | None = None) -> np.ndarray:
    """attention.py:158-167 for a GIVEN id set (used to score the GPU's own selection)."""
    d = keys.shape[1]
    q64 = np.asarray(q, dtype=np.float64)
    sc = scale if scale is not None else 1.0 / np.sqrt(d)
    ids = np.asarray(ids, dtype=np.int64)
    s_ctx = (np.asarray(keys, dtype=np.float64)[ids] @ q64) * sc
    v_ctx = np.asarray(values, dtype=np.float64)[ids]
    wk = np.asarray(win_keys, dtype=np.float64).reshape(-1, d)
    wv = np.asarray(win_values, dtype=np.float64).reshape(-1, d)
    return joint_attend(s_ctx, v_ctx, (wk @ q64) * sc, wv, combine)


# ------------------------------------------------------------------------------ batched layer
def decode_layer(q, k_cache, v_cache, n_ctx, k: int, n_win=None, combine: str = "joint",
                 pinned_prefix: int = 0):
    """The per-head loop of decode_step (attention.py:213-230) for one layer, batched over b,
    with the GQA mapping q head h → kv head h // (Hq/Hkv) (the reference is MHA).
    Inputs f32 numpy: q [B,Hq,d], caches [B,Hkv,rows,d] (window rows after the context).
    Returns (out [B,Hq,d] f32, ids list[B][Hq] of i64 arrays)."""
    B, Hq, d = q.shape
    Hkv = k_cache.shape[1]
    G = Hq // Hkv
    out = np.zeros((B, Hq, d), dtype=DTYPE)
    ids_all = []
    for b in range(B):
        row = []
        n = int(n_ctx[b])
        w = int(n_win[b]) if n_win is not None else 0
        for h in range(Hq):
            kv = h // G
            keys = k_cache[b, kv, :n]
            vals = v_cache[b, kv, :n]
            wk = k_cache[b, kv, n:n + w]
            wv = v_cache[b, kv, n:n + w]
            o, ids = topk_attend(q[b, h], keys, vals, wk, wv, k, combine, pinned_prefix)
            out[b, h] = o
            row.append(ids)
        ids_all.append(row)
    return out, ids_all


# ------------------------------------------------------------------------------ parity helpers
def near_tie_set_diff(ids_gpu, ids_ref, scores64: np.ndarray, rel: float = 1e-3) -> tuple[int, int]:
    """Parity rule for index sets (north star): the symmetric difference may only contain rows
    whose oracle score is within rel·|s_k| of the oracle's k-th score s_k.
    Returns (n_diff, n_unexcused)."""
    a = set(int(x) for x in np.asarray(ids_gpu).ravel() if x >= 0)
    b = set(int(x) for x in np.asarray(ids_ref).ravel())
    diff = a ^ b
    if not diff:
        return 0, 0
    ref_sorted = np.sort(scores64[np.asarray(sorted(b), dtype=np.int64)])
    s_k = ref_sorted[0]
    tol = rel * abs(s_k)
    bad = [i for i in diff if abs(scores64[i] - s_k) >= tol]
    return len(diff), len(bad)


def to_bf16_f32(a: np.ndarray) -> np.ndarray:
    """Round f32 values to the nearest bf16 (RNE), returned as f32 — the values the GPU sees."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


# ------------------------------------------------------------------------------ sharding
def score_key(s32: np.ndarray) -> np.ndarray:
    """Order-preserving u32 key of f32 scores (-0.0 canonicalised to +0.0), the same map the
    kernels use for the (score desc, id asc) composite."""
    b = np.ascontiguousarray(s32, dtype=np.float32).view(np.uint32).copy()
    b[b == 0x80000000] = 0
    neg = (b & 0x80000000) != 0
    return np.where(neg, ~b, b | 0x80000000).astype(np.uint32)


def composite(s32: np.ndarray, gid: np.ndarray) -> np.ndarray:
    return (score_key(s32).astype(np.uint64) << np.uint64(32)) | (
        (~np.asarray(gid, dtype=np.uint64)) & np.uint64(0xFFFFFFFF))


def topk_by_composite(comp: np.ndarray, k: int) -> np.ndarray:
    """Indices of the k largest composites (unique), ordered descending."""
    comp = np.asarray(comp, dtype=np.uint64)
    order = np.argsort(comp)[::-1]
    return order[:k]


# ------------------------------------------------------------------------------ C port (ctypes)
_C = None


def c_lib():
    """oracle/build/libtkv_oracle.so (oracle/tkv_oracle.c, built by oracle/Makefile)."""
    global _C
    if _C is None:
        import ctypes
        from pathlib import Path

        path = Path(__file__).resolve().parent / "build" / "libtkv_oracle.so"
        if not path.exists():
            import subprocess

            subprocess.run(["make", "-C", str(path.parent.parent)], check=True, capture_output=True)
        lib = ctypes.CDLL(str(path))
        P = ctypes.c_void_p
        lib.tkv_oracle_layer.argtypes = [P, P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                         ctypes.c_int, P, P, ctypes.c_int64, ctypes.c_int, ctypes.c_int64,
                                         ctypes.c_int, P, P, P]
        lib.tkv_oracle_layer.restype = ctypes.c_int
        lib.tkv_oracle_max_threads.restype = ctypes.c_int
        _C = lib
    return _C


def c_decode_layer(q, k_cache, v_cache, n_ctx, k: int, n_win=None, combine: str = "joint",
                   pinned_prefix: int = 0, threads: int | None = None):
    """decode_layer() through the C port (strict left-to-right f64 scan, OpenMP)."""
    import ctypes

    lib = c_lib()
    q = np.ascontiguousarray(q, dtype=np.float32)
    kc = np.ascontiguousarray(k_cache, dtype=np.float32)
    vc = np.ascontiguousarray(v_cache, dtype=np.float32)
    B, Hq, d = q.shape
    Hkv, rows = kc.shape[1], kc.shape[2]
    nc = np.ascontiguousarray(n_ctx, dtype=np.int32)
    nw = np.ascontiguousarray(n_win if n_win is not None else np.zeros(B), dtype=np.int32)
    stride = k + max(0, pinned_prefix)
    out = np.zeros((B, Hq, d), dtype=np.float32)
    ids = np.zeros((B * Hq, stride), dtype=np.int64)
    cnt = np.zeros(B * Hq, dtype=np.int64)
    t = threads if threads is not None else lib.tkv_oracle_max_threads()
    vp = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    lib.tkv_oracle_layer(vp(q), vp(kc), vp(vc), B, Hq, Hkv, rows, d, vp(nc), vp(nw), k,
                         0 if combine == "joint" else 1, pinned_prefix, t, vp(out), vp(ids), vp(cnt))
    ids_all = [[ids[b * Hq + h, : cnt[b * Hq + h]].copy() for h in range(Hq)] for b in range(B)]
    return out, ids_all
