"""CPU: the oracle restatement (numpy and C port) reproduces the live reference's golden
vectors (tests/golden/make_golden.py) bit-for-bit on ids and to <= 1e-6 on outputs."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O

GOLDEN = Path(__file__).resolve().parent / "golden"
CASES = json.loads((GOLDEN / "index.json").read_text())["cases"]


def bits(b):
    return (np.asarray(b, dtype=np.uint32) << 16).view(np.float32)


def load(name):
    z = np.load(GOLDEN / "cases" / f"{name}.npz")
    return {k: z[k] for k in z.files}


@pytest.mark.parametrize("case", [c["name"] for c in CASES if c["kind"] == "search"])
def test_flat_topk_matches_reference(case):
    z = load(case)
    q, keys, k = bits(z["q"]), bits(z["keys"]), int(z["k"])
    vals, ids = O.flat_topk(keys, q, k)
    np.testing.assert_array_equal(ids, z["ids"])
    np.testing.assert_array_equal(vals, z["vals"])
    # strict left-to-right scan restatement agrees bit-for-bit with the BLAS one here
    if keys.shape[0] <= 1100:
        np.testing.assert_array_equal(O.ip_scores_strict(keys, q), O.ip_scores_all(keys, q))


@pytest.mark.parametrize("case", [c["name"] for c in CASES if c["kind"] == "attend"])
def test_topk_attend_matches_reference(case):
    z = load(case)
    q, keys, vals = bits(z["q"]), bits(z["keys"]), bits(z["values"])
    wk, wv = bits(z["win_keys"]), bits(z["win_values"])
    out, ids = O.topk_attend(q, keys, vals, wk, wv, int(z["k"]), str(z["combine"]), int(z["pinned"]))
    np.testing.assert_array_equal(ids, z["ids"])
    np.testing.assert_allclose(out, z["out"], rtol=0, atol=1e-6)


@pytest.mark.parametrize("case", [c["name"] for c in CASES if c["kind"] == "attend" and c["d"] == 128])
def test_c_port_matches_reference(case):
    z = load(case)
    q, keys, vals = bits(z["q"]), bits(z["keys"]), bits(z["values"])
    wk, wv = bits(z["win_keys"]), bits(z["win_values"])
    n, d = keys.shape
    w = wk.shape[0]
    K = np.concatenate([keys, wk])[None, None]
    V = np.concatenate([vals, wv])[None, None]
    out, ids = O.c_decode_layer(q[None, None], K, V, [n], int(z["k"]), n_win=[w],
                                combine=str(z["combine"]), pinned_prefix=int(z["pinned"]), threads=1)
    np.testing.assert_array_equal(ids[0][0], z["ids"])
    np.testing.assert_allclose(out[0, 0], z["out"], rtol=0, atol=1e-6)


def test_spec_known_answers():
    z = load("kat_knn_k1")
    assert z["ids"].tolist() == [0] and z["vals"].tolist() == [1.0]
    assert load("kat_ties")["ids"].tolist() == [1, 3, 0]  # lower-index ties
    assert load("kat_knn_k_gt_N")["ids"].tolist() == [0, 1, 2]  # k >= N: all, sorted
    z = load("kat_attend_N1")  # N=1, k=1: output == the single value row
    np.testing.assert_array_equal(z["out"], bits(z["values"])[0])


def test_softmax_known_answer():
    # softmax([1,2,3]) = [0.09003, 0.24473, 0.66524] ± 1e-5 via _joint_attend
    out = O.joint_attend(np.array([1.0, 2.0, 3.0]), np.eye(3), np.zeros(0), np.zeros((0, 3)), "joint")
    np.testing.assert_allclose(out, [0.09003, 0.24473, 0.66524], atol=1e-5)


def test_dense_equivalence_at_k_equals_n():
    # SPEC.md:255 / acceptance #1: k = N reduces to dense attention within 1e-5
    rng = np.random.default_rng(0)
    for _ in range(20):
        n, d = int(rng.integers(1, 300)), 16
        q = rng.standard_normal(d).astype(np.float32)
        K = rng.standard_normal((n, d)).astype(np.float32)
        V = rng.standard_normal((n, d)).astype(np.float32)
        out, _ = O.topk_attend(q, K, V, np.zeros((0, d)), np.zeros((0, d)), n)
        s = K.astype(np.float64) @ q / np.sqrt(d)
        w = np.exp(s - s.max())
        np.testing.assert_allclose(out, (w @ V) / w.sum(), atol=1e-5)


def test_flat_topk_equals_argsort_with_lower_index_ties():
    # acceptance #2: flat top-k == brute-force argsort, ties → lower index
    rng = np.random.default_rng(1)
    for _ in range(200):
        n = int(rng.integers(1, 400))
        k = int(rng.integers(1, n + 1))
        s = rng.integers(-5, 5, size=n).astype(np.float64)  # many exact ties
        _, ids = O.flat_topk_from_scores(s, k)
        ref = np.lexsort((np.arange(n), -s))[:k]
        np.testing.assert_array_equal(ids, ref)


def test_composite_order_is_reference_order():
    """The kernels' selection order (score key << 32 | ~id, descending) is the reference's
    (score desc, id asc) order, including -0.0 == +0.0 ties."""
    rng = np.random.default_rng(2)
    s = rng.integers(-3, 3, size=500).astype(np.float32)
    s[::7] = -0.0
    gid = np.arange(500)
    c = O.composite(s, gid)
    order = O.topk_by_composite(c, 500)
    ref = np.lexsort((gid, -s.astype(np.float64)))
    np.testing.assert_array_equal(order, ref)
