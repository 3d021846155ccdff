"""Generate golden vectors by running the LIVE reference (/root/reference/pkg/src/topk_kv).

Run in the development container (the reference tree does not exist on the GPU box):

    python tests/golden/make_golden.py

Each case is saved as tests/golden/cases/<name>.npz with bf16-representable inputs (stored
as uint16 bf16 bit patterns — the exact values the B200 kernels consume) and the
reference's outputs: topk_attend's return value, the retrieval log, the TierAccounting
counters and the index counters, and for search cases knn_search's TopKResult.
The reference is imported read-only; Numba's cache is redirected to /tmp so nothing is
written into the reference tree.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "numba_cache_golden"))
sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "cases"

import numpy as np  # noqa: E402


def bf16_bits(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    return (((u + 0x7FFF + ((u >> 16) & 1)) >> 16) & 0xFFFF).astype(np.uint16)


def from_bits(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


def rnd(rng, shape, scale=1.0):
    return from_bits(bf16_bits(rng.standard_normal(shape).astype(np.float32) * scale))


def main() -> None:
    sys.path.insert(0, str(REF))
    import topk_kv as ref  # noqa: E402  (the reference package)

    OUT.mkdir(parents=True, exist_ok=True)
    index = []

    def save_attend(name, q, keys, values, wk, wv, k, combine="joint", pinned=0):
        idx = ref.build_index(keys, "flat")
        acct = ref.TierAccounting()
        log: list = []
        out = ref.topk_attend(q, idx, lambda ids: values[ids], wk, wv, k, acct,
                              combine=combine, pinned_prefix=pinned, retrieval_log=log)
        np.savez_compressed(
            OUT / f"{name}.npz", kind="attend",
            q=bf16_bits(q), keys=bf16_bits(keys), values=bf16_bits(values),
            win_keys=bf16_bits(wk.reshape(-1, keys.shape[1])), win_values=bf16_bits(wv.reshape(-1, keys.shape[1])),
            k=k, combine=combine, pinned=pinned, out=out, ids=log[0],
            acct=np.array([acct.cold_reads, acct.hot_ops, acct.bytes_moved], dtype=np.int64),
            counters=np.array([idx.distance_evals, idx.queries], dtype=np.int64))
        index.append({"name": name, "kind": "attend", "N": int(keys.shape[0]), "d": int(keys.shape[1]),
                      "k": int(k), "n_gen": int(wk.shape[0]), "combine": combine, "pinned": int(pinned)})

    def save_search(name, q, keys, k):
        idx = ref.build_index(keys, "flat")
        res = ref.knn_search(idx, q, k)
        np.savez_compressed(OUT / f"{name}.npz", kind="search", q=bf16_bits(q), keys=bf16_bits(keys),
                            k=k, vals=res.vals, ids=res.ids,
                            counters=np.array([idx.distance_evals, idx.queries], dtype=np.int64))
        index.append({"name": name, "kind": "search", "N": int(keys.shape[0]), "d": int(keys.shape[1]),
                      "k": int(k)})

    # ---- SPEC known answers
    kat_keys = np.array([[1, 0], [0, 1], [-1, 0]], dtype=np.float32)
    save_search("kat_knn_k1", np.array([1, 0], dtype=np.float32), kat_keys, 1)
    save_search("kat_knn_kN", np.array([1, 0], dtype=np.float32), kat_keys, 3)
    save_search("kat_knn_k_gt_N", np.array([1, 0], dtype=np.float32), kat_keys, 5)
    # duplicate-score ties → lower ids first: scores [1,2,1,2,1], k=3 → ids [1,3,0]
    save_search("kat_ties", np.array([1.0], dtype=np.float32),
                np.array([[1], [2], [1], [2], [1]], dtype=np.float32), 3)
    one = np.array([[0.5, -1.25, 2.0, 0.125]], dtype=np.float32)
    save_attend("kat_attend_N1", np.array([1, 2, 3, 4], dtype=np.float32), one,
                np.array([[3.0, -1.0, 0.5, 8.0]], dtype=np.float32),
                np.zeros((0, 4), np.float32), np.zeros((0, 4), np.float32), 1)

    rng = np.random.default_rng(20250210)
    # ---- random cases, bf16-representable inputs (the GPU consumes exactly these values)
    cases = [
        ("rand_n512_d128_k16", 512, 128, 16, 0, "joint", 0),
        ("rand_n1000_d128_k100_w3", 1000, 128, 100, 3, "joint", 0),
        ("rand_n1000_d128_k100_w3_additive", 1000, 128, 100, 3, "additive", 0),
        ("rand_n700_d128_k50_w2_pin8", 700, 128, 50, 2, "joint", 8),
        ("rand_n300_d16_k20_w1", 300, 16, 20, 1, "joint", 0),
        ("rand_n2048_d64_k64", 2048, 64, 64, 0, "joint", 0),
        ("rand_n100_d128_kN_w4", 100, 128, 100, 4, "joint", 0),
        ("rand_n50_d128_k80_clamp", 50, 128, 80, 0, "joint", 0),
        ("rand_n1500_d128_k256_w5_pin3", 1500, 128, 256, 5, "joint", 3),
        ("rand_n64_d128_k1_w1_additive", 64, 128, 1, 1, "additive", 0),
    ]
    for name, n, d, k, w, comb, pin in cases:
        q = rnd(rng, (d,))
        keys = rnd(rng, (n, d))
        vals = rnd(rng, (n, d))
        save_attend(name, q, keys, vals, rnd(rng, (w, d)), rnd(rng, (w, d)), k, comb, pin)
    # exact duplicate rows: ties must resolve to the lower row id
    n, d = 1024, 128
    keys = rnd(rng, (n, d))
    keys[40:1000:40] = keys[7]
    keys[41:1000:40] = keys[9]
    q = rnd(rng, (d,))
    vals = rnd(rng, (n, d))
    for k in (5, 20, 26, 37):
        save_attend(f"ties_dup_rows_k{k}", q, keys, vals, np.zeros((0, d), np.float32),
                    np.zeros((0, d), np.float32), k)
        save_search(f"ties_search_k{k}", q, keys, k)
    # 10^3 Gaussian keys, d=16, k=8 equals the argsort oracle
    save_search("rand_search_n1000_d16_k8", rnd(rng, (16,)), rnd(rng, (1000, 16)), 8)
    save_search("rand_search_n4000_d128_k300", rnd(rng, (128,)), rnd(rng, (4000, 128)), 300)
    # k = N dense equivalence
    save_attend("dense_equiv_n256_d128", rnd(rng, (128,)), rnd(rng, (256, 128)), rnd(rng, (256, 128)),
                rnd(rng, (2, 128)), rnd(rng, (2, 128)), 256)

    # ---- TKKV cache file (cache.py:1-13) + header mutations with the reference's verdicts
    from topk_kv.cache import CacheFile, CacheMeta, KvCache, write_cache  # noqa: E402
    from topk_kv.errors import FormatError as RefFormatError  # noqa: E402

    meta = CacheMeta(2, 3, 50, 16, "f32", "golden-tiny")
    kv_rng = np.random.default_rng(7)
    cache = KvCache(meta, rnd(kv_rng, (2, 3, 50, 16)), rnd(kv_rng, (2, 3, 50, 16)))
    tk_path = OUT / "tkkv_small.tkkv"
    write_cache(cache, tk_path)
    blob = tk_path.read_bytes()
    mutations = []
    spots = [(0, b"XKKV"), (4, b"\x02"), (8, b"\x00"), (16, b"\x00"), (24, b"\x00"), (32, b"\x00"),
             (40, b"\x31"), (48, b"\x07"), (49, b"\xff\xff"), (53, b"\xff"), (49 + 4 + 11, b"\x01"),
             (49 + 4 + 11 + 8, b"\x00"), (len(blob) - 1, None), (len(blob), b"\x00"), (16, b"\x03"),
             (24, b"\x33"), (40, b"\x00\x01"), (49, b"\x00\x00\x00\x00"), (49 + 4 + 11 + 16, b"\x10"),
             (0, b"\x00")]
    for i, (at, new) in enumerate(spots):
        b2 = bytearray(blob)
        if new is None:
            b2 = b2[:at]
        elif at >= len(b2):
            b2 += new
        else:
            b2[at:at + len(new)] = new
        mp = OUT / f"tkkv_mut_{i:02d}.bin"
        mp.write_bytes(bytes(b2))
        try:
            with CacheFile(mp) as cf:
                verdict = {"ok": True, "meta_hash": cf.meta.meta_hash().hex()}
        except RefFormatError as e:
            verdict = {"ok": False, "error": "FormatError", "offset": e.offset}
        except Exception as e:  # noqa: BLE001
            verdict = {"ok": False, "error": type(e).__name__, "offset": None}
        mp.unlink()
        mutations.append({"at": at, "new": None if new is None else new.hex(), "verdict": verdict})
    index.append({"name": "tkkv_small", "kind": "tkkv", "meta_hash": meta.meta_hash().hex(),
                  "mutations": mutations})
    np.savez_compressed(OUT / "tkkv_small_values.npz", keys=bf16_bits(cache.keys), values=bf16_bits(cache.values))

    (OUT.parent / "index.json").write_text(json.dumps({"reference": str(REF), "cases": index}, indent=1))
    print(f"wrote {len(index)} cases to {OUT}")


if __name__ == "__main__":
    main()
