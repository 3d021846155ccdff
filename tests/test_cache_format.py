"""TKKV cache files (reference cache.py:1-13, 120-257): header validation with the reference's
exact verdicts on 20 mutated files (SPEC acceptance #10), zero-copy section views (CPU), and
the device loader into the bf16 scan layout (GPU)."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

from paper_2502_06766_b200 import cache as C
from paper_2502_06766_b200.errors import FormatError

GOLDEN = Path(__file__).resolve().parent / "golden"
CASE = [c for c in json.loads((GOLDEN / "index.json").read_text())["cases"] if c["kind"] == "tkkv"][0]
PATH = GOLDEN / "cases" / "tkkv_small.tkkv"


def golden_values():
    z = np.load(GOLDEN / "cases" / "tkkv_small_values.npz")
    bits = lambda b: (b.astype(np.uint32) << 16).view(np.float32)  # noqa: E731
    return bits(z["keys"]), bits(z["values"])


def test_header_and_meta_hash():
    meta, offsets = C.read_header(PATH)
    assert (meta.n_layers, meta.n_heads, meta.n_tokens, meta.head_dim) == (2, 3, 50, 16)
    assert meta.model_id == "golden-tiny"
    assert meta.meta_hash().hex() == CASE["meta_hash"]
    assert len(offsets) == 2 * 2 * 3


def test_sections_are_the_reference_arrays():
    K, V = golden_values()
    f = C.TkkvFile(PATH)
    for l in range(2):
        for h in range(3):
            np.testing.assert_array_equal(f.section(l, h, "keys"), K[l, h])
            np.testing.assert_array_equal(f.section(l, h, "values"), V[l, h])


@pytest.mark.parametrize("i", range(len(CASE["mutations"])))
def test_header_mutations_match_reference_verdicts(tmp_path, i):
    m = CASE["mutations"][i]
    blob = bytearray(PATH.read_bytes())
    at = m["at"]
    if m["new"] is None:
        blob = blob[:at]
    else:
        new = bytes.fromhex(m["new"])
        if at >= len(blob):
            blob += new
        else:
            blob[at:at + len(new)] = new
    p = tmp_path / "m.tkkv"
    p.write_bytes(bytes(blob))
    v = m["verdict"]
    if v["ok"]:
        meta, _ = C.read_header(p)
        assert meta.meta_hash().hex() == v["meta_hash"]
    elif v["error"] == "FormatError":
        with pytest.raises(FormatError) as e:
            C.read_header(p)
        assert e.value.offset == v["offset"]
    else:
        with pytest.raises(Exception) as e:
            C.read_header(p)
        assert type(e.value).__name__ == v["error"]


@pytest.mark.gpu
def test_load_layer_to_device(cuda):
    K, V = golden_values()
    f = C.TkkvFile(PATH, staging_rows=7)  # odd staging size: exercises the chunk loop
    for layer in range(2):
        kd, vd = f.load_layer(layer, cuda, capacity=64)
        assert kd.shape == (1, 3, 64, 128)
        kn = kd.float().cpu().numpy()
        np.testing.assert_array_equal(kn[0, :, :50, :16], K[layer])
        assert not kn[0, :, :, 16:].any() and not kn[0, :, 50:].any()
        np.testing.assert_array_equal(vd.float().cpu().numpy()[0, :, :50, :16], V[layer])
    # a token-range shard of a subset of heads
    kd, vd = f.load_layer(1, cuda, heads=[2, 0], row_range=(10, 35))
    np.testing.assert_array_equal(kd.float().cpu().numpy()[0, :, :, :16], K[1, [2, 0], 10:35])
