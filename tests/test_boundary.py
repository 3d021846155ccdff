"""CPU: the C-ABI library loads, exports every symbol include/tkv.h declares, and validates
problems with the reference's error taxonomy — all without a GPU (no compute calls)."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2502_06766_b200 import _lib, errors, ops

HEADER = Path(__file__).resolve().parents[1] / "include" / "tkv.h"


def header_functions() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tkv_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_header_symbols():
    lib = _lib.load()
    declared = header_functions()
    assert declared, "no functions parsed from include/tkv.h"
    for name in declared:
        assert hasattr(lib, name), f"libtkv.so does not export {name}"
    assert sorted(_lib.EXPORTS) == declared
    assert lib.tkv_version() == 1


def test_problem_struct_mirrors_header():
    text = HEADER.read_text()
    body = text[text.index("typedef struct tkv_problem"):text.index("} tkv_problem;")]
    fields = re.findall(r"^\s*(?:u?int\d+_t|float)\s+(\w+);", body, flags=re.M)
    assert fields == [f for f, _ in _lib.Problem._fields_]
    assert ctypes.sizeof(_lib.Problem) == 64


def _prob(**kw):
    base = dict(B=1, Hq=32, Hkv=8, cache_rows=1 << 20, max_ctx=1 << 20, k=16384)
    base.update(kw)
    return ops.make_problem(base["B"], base["Hq"], base["Hkv"], base["cache_rows"], base["max_ctx"], base["k"])


def test_workspace_sizing():
    n = _lib.workspace_bytes(_prob())
    # candidate buffer (B*Hq*N*8) dominates; everything else is small
    assert 32 * (1 << 20) * 8 <= n < 32 * (1 << 20) * 8 + 64 * (1 << 20)
    assert _lib.workspace_bytes(_prob(max_ctx=1000, cache_rows=1000, k=10)) < n


@pytest.mark.parametrize("kw,exc", [
    (dict(Hq=30), errors.ShapeError),          # not a multiple of Hkv
    (dict(Hq=96, Hkv=8), errors.ShapeError),   # group size 12
    (dict(k=0), errors.InputError),            # attention.py:144-145
    (dict(max_ctx=10, cache_rows=5), errors.ShapeError),
])
def test_validation_maps_to_reference_errors(kw, exc):
    with pytest.raises(exc):
        _lib.workspace_bytes(_prob(**kw))


def test_bad_head_dim_and_combine():
    p = _prob()
    p.head_dim = 64
    with pytest.raises(errors.ShapeError):
        _lib.workspace_bytes(p)
    p = _prob()
    p.combine = 7
    with pytest.raises(errors.ConfigError):
        _lib.workspace_bytes(p)
    with pytest.raises(errors.ConfigError):
        ops.make_problem(1, 1, 1, 1, 1, 1, combine="sum")
    # sorted output has no k limit (chunk sort + merge passes beyond one CTA's shared memory):
    # the workspace grows by the merge buffers instead
    p = _prob()
    p.k = 20000
    plain = _lib.workspace_bytes(p)
    p.flags = _lib.F_SORTED
    assert _lib.workspace_bytes(p) > plain


def test_compute_entry_rejects_bad_arguments_before_any_launch():
    lib = _lib.load()
    p = _prob(max_ctx=100, cache_rows=100, k=4)
    rc = lib.tkv_topk_decode_attention(ctypes.byref(p), None, None, None, None, None, None, None,
                                       None, None, 0, None)
    assert rc == errors.TKV_EWORKSPACE
    buf = np.zeros(_lib.workspace_bytes(p) + 512, dtype=np.uint8)
    ws = (buf.ctypes.data + 255) // 256 * 256
    rc = lib.tkv_topk_decode_attention(ctypes.byref(p), None, None, None, None, None, None, None,
                                       None, ctypes.c_void_p(ws), _lib.workspace_bytes(p), None)
    assert rc == errors.TKV_EBADSHAPE and "q is NULL" in _lib.last_error()
    rc = lib.tkv_kv_append(1, 8, 128, 10, None, None, None, None, None, None, 1, None)
    assert rc == errors.TKV_EBADSHAPE
    # the decode-step helpers validate before launching, with a message
    rc = lib.tkv_model_add_rmsnorm(None, None, None, 1e-5, None, 4096, None)
    assert rc == errors.TKV_EBADSHAPE and "tkv_model_add_rmsnorm" in _lib.last_error()
    rc = lib.tkv_model_qkv_rope_append(*([None] * 9), 10, 8, 2, 64, None)
    assert rc == errors.TKV_EBADSHAPE and "qkv_rope_append" in _lib.last_error()
    rc = lib.tkv_model_silu_mul(None, None, 0, None)
    assert rc == errors.TKV_EBADSHAPE and "silu_mul" in _lib.last_error()
    rc = lib.tkv_model_logits_argmax(None, 10, None, None, None, None)
    assert rc == errors.TKV_EBADSHAPE and "logits_argmax" in _lib.last_error()


def test_status_mapping():
    for code, exc in [(errors.TKV_EBADSHAPE, errors.ShapeError), (errors.TKV_EBADK, errors.InputError),
                      (errors.TKV_ECONFIG, errors.ConfigError), (errors.TKV_ECUDA, errors.DeviceError)]:
        with pytest.raises(exc):
            errors.raise_for_status(code, "x")
    assert issubclass(errors.InputError, ValueError) and issubclass(errors.InputError, errors.TopkKvError)


def test_product_path_has_no_cpu_fallback(monkeypatch):
    """Without the native library every entry point fails loudly (DeviceError)."""
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", Path("/nonexistent/libtkv.so"))
    with pytest.raises(errors.DeviceError):
        _lib.load()
    import torch

    with pytest.raises(errors.ShapeError):  # CPU tensors are rejected outright
        ops.topk_decode_attention(torch.zeros(1, 4, 128, dtype=torch.bfloat16),
                                  torch.zeros(1, 1, 8, 128, dtype=torch.bfloat16),
                                  torch.zeros(1, 1, 8, 128, dtype=torch.bfloat16), 8, 2)


def test_product_package_does_not_import_oracle():
    pkg = Path(__file__).resolve().parents[1] / "paper_2502_06766_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "import oracle" not in src and "from oracle" not in src, f"{f} imports the oracle"


def test_python_flag_constants_match_header():
    """The drop-in's flag constants (_lib.F_*) are the header's TKV_F_* values."""
    import re

    from paper_2502_06766_b200 import _lib

    hdr = (Path(__file__).resolve().parents[1] / "include" / "tkv.h").read_text()
    defs = {m.group(1): int(m.group(2)) for m in re.finditer(r"#define TKV_F_(\w+) (\d+)u", hdr)}
    for name in ("SORTED", "NO_FILTER", "GATHER_LIST", "HEAD", "NO_HEAD", "HOST_Q", "SCAN_HMMA", "CLUSTER",
                 "NO_CLUSTER"):
        assert getattr(_lib, "F_" + name) == defs[name], name
