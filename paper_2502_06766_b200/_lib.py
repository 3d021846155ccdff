"""ctypes binding of libtkv.so — the C ABI declared in include/tkv.h.

This is the only place the package touches the native library. There is no fallback: if
the shared object is missing or fails to load, every compute entry point raises
DeviceError (the product path never silently runs anything else).
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import DeviceError, raise_for_status

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libtkv.so"
if os.environ.get("TKV_LIB_PATH"):  # A/B experiments with an alternative build
    LIB_PATH = Path(os.environ["TKV_LIB_PATH"]).resolve()

# symbols the header declares (checked by tests/test_boundary.py against include/tkv.h)
EXPORTS = (
    "tkv_version",
    "tkv_last_error",
    "tkv_device_check",
    "tkv_workspace_bytes",
    "tkv_workspace_init",
    "tkv_topk_decode_attention",
    "tkv_topk_search",
    "tkv_topk_decode_step",
    "tkv_kv_append",
    "tkv_shard_candidates",
    "tkv_shard_merge",
    "tkv_shard_narrow_check",
    "tkv_shard_merge_lists",
    "tkv_shard_candidates2",
    "tkv_shard_exchange_merge",
    "tkv_shard_combine",
    "tkv_shard_partial",
    "tkv_shard_finalize",
    "tkv_last_launch_count",
    "tkv_workspace_fallbacks",
    "tkv_profile_scan_events",
    "tkv_debug_timeline",
    "tkv_convert_rows_f32",
    "tkv_model_add_rmsnorm",
    "tkv_model_qkv_rope_append",
    "tkv_model_silu_mul",
    "tkv_model_logits_argmax",
)

COMBINE_JOINT = 0
COMBINE_ADDITIVE = 1
F_SORTED = 1
F_NO_FILTER = 2
F_SCAN_HMMA = 8
F_PARTS_SHIFT = 8  # TKV_F_PARTS(n): bits 8..11
F_GATHER_LIST = 16
F_HEAD = 32
F_NO_HEAD = 64
F_HOST_Q = 128
F_CLUSTER = 4096
F_NO_CLUSTER = 8192


class Problem(ctypes.Structure):
    """Mirror of `tkv_problem` (include/tkv.h)."""

    _fields_ = [
        ("batch", ctypes.c_int32),
        ("n_q_heads", ctypes.c_int32),
        ("n_kv_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("cache_rows", ctypes.c_int64),
        ("max_ctx", ctypes.c_int64),
        ("k", ctypes.c_int32),
        ("pinned_prefix", ctypes.c_int32),
        ("scale", ctypes.c_float),
        ("combine", ctypes.c_int32),
        ("flags", ctypes.c_uint32),
        ("row_offset", ctypes.c_int64),
    ]

    def key(self) -> tuple:
        return tuple(getattr(self, f) for f, _ in self._fields_)


_P = ctypes.c_void_p
_I = ctypes.c_int
_SIG = {
    "tkv_version": ([], _I),
    "tkv_last_error": ([], ctypes.c_char_p),
    "tkv_device_check": ([], _I),
    "tkv_last_launch_count": ([], _I),
    "tkv_workspace_fallbacks": ([ctypes.POINTER(Problem), _P, ctypes.c_size_t, _P], _I),
    "tkv_profile_scan_events": ([_P, _P], _I),
    "tkv_debug_timeline": ([_P], _I),
    "tkv_convert_rows_f32": ([_P, ctypes.c_int64, ctypes.c_int32, _P, _P], _I),
    "tkv_workspace_bytes": ([ctypes.POINTER(Problem), ctypes.POINTER(ctypes.c_size_t)], _I),
    "tkv_workspace_init": ([ctypes.POINTER(Problem), _P, ctypes.c_size_t, _P], _I),
    "tkv_topk_decode_attention": (
        [ctypes.POINTER(Problem), _P, _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P], _I),
    "tkv_topk_search": ([ctypes.POINTER(Problem), _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P], _I),
    "tkv_topk_decode_step": (
        [ctypes.POINTER(Problem), _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P], _I),
    "tkv_kv_append": (
        [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, _P, _P, _P, _P, _P, _P,
         ctypes.c_int32, _P], _I),
    "tkv_shard_candidates": ([ctypes.POINTER(Problem), _P, _P, _P, _P, _P, ctypes.c_size_t, _P], _I),
    "tkv_shard_merge": (
        [ctypes.POINTER(Problem), _P, ctypes.c_int32, _P, _P, _P, ctypes.c_size_t, _P], _I),
    "tkv_shard_narrow_check": (
        [ctypes.POINTER(Problem), _P, ctypes.c_int32, ctypes.c_int32, _P, _P], _I),
    "tkv_shard_merge_lists": (
        [ctypes.POINTER(Problem), _P, ctypes.c_int32, ctypes.c_int32, _P, _P, _P, ctypes.c_size_t,
         _P], _I),
    "tkv_shard_candidates2": (
        [ctypes.POINTER(Problem), ctypes.c_int32, _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P], _I),
    "tkv_shard_exchange_merge": (
        [ctypes.POINTER(Problem), _P, _P, _P, ctypes.c_int32, ctypes.c_int32, _P, _P, _P, _P, ctypes.c_size_t,
         _P], _I),
    "tkv_shard_combine": (
        [ctypes.POINTER(Problem), _P, ctypes.c_int32, _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P], _I),
    "tkv_shard_partial": (
        [ctypes.POINTER(Problem), _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P], _I),
    "tkv_shard_finalize": (
        [ctypes.POINTER(Problem), _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P], _I),
    "tkv_model_add_rmsnorm": ([_P, _P, _P, ctypes.c_float, _P, ctypes.c_int32, _P], _I),
    "tkv_model_qkv_rope_append": (
        [_P, _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _P],
        _I),
    "tkv_model_silu_mul": ([_P, _P, ctypes.c_int32, _P], _I),
    "tkv_model_logits_argmax": ([_P, ctypes.c_int32, _P, _P, _P, _P], _I),
}

_lock = threading.Lock()
_lib = None


def load(build_if_missing: bool = False) -> ctypes.CDLL:
    """Load libtkv.so (building it first only when asked). Raises DeviceError if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            if build_if_missing:
                from .build import build

                build()
            else:
                raise DeviceError(
                    f"native library {LIB_PATH} is missing: run `python -m paper_2502_06766_b200.build`"
                )
        try:
            lib = ctypes.CDLL(str(LIB_PATH))
        except OSError as e:  # pragma: no cover - depends on the host
            raise DeviceError(f"cannot load {LIB_PATH}: {e}") from e
        for name, (args, res) in _SIG.items():
            if os.environ.get("TKV_LIB_PATH") and not hasattr(lib, name):
                continue  # A/B against an older experiment build: newer entry points absent
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def last_error() -> str:
    return load().tkv_last_error().decode(errors="replace")


def check(code: int) -> None:
    if code != 0:
        raise_for_status(code, last_error())


def call(name: str, *args) -> None:
    lib = load()
    check(getattr(lib, name)(*args))


def launches() -> int:
    return int(load().tkv_last_launch_count())


def workspace_bytes(p: Problem) -> int:
    n = ctypes.c_size_t(0)
    check(load().tkv_workspace_bytes(ctypes.byref(p), ctypes.byref(n)))
    return int(n.value)
