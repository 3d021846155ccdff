"""TKKV cache files → HBM (SURVEY §8f "next" #3).

Reads the reference's on-disk KV cache (topk_kv/cache.py:1-13: magic "TKKV", version 1,
little-endian fixed header L, H, N, d, D, dtype; model_id; 2·L·H u64 section offsets; row-major
f32 (N, d) sections ordered (layer, head, keys|values)) with the same validation and the same
FormatError byte offsets as the reference's `_read_header` / `CacheFile` (cache.py:160-211),
and streams sections straight into the scan-friendly device layout: bf16 rows of 128 values
([1, H, rows, 128] per layer, zero-padded for d < 128), optionally only a token range
[lo, hi) for a shard. Bytes go file → pinned staging (double-buffered) → H2D → the
`tkv_convert_rows_f32` kernel; no full f32 copy of a layer ever exists on the host or device.
`CacheMeta.meta_hash` pairs a cache with its index exactly as cache.py:59-70 does.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, ops
from .errors import FormatError, InputError

CACHE_MAGIC = b"TKKV"
CACHE_VERSION = 1
_DTYPE_CODES = {"f32": 1}
_DTYPE_NAMES = {v: k for k, v in _DTYPE_CODES.items()}
_SCALAR_BYTES = 4
_FIXED_HEADER = struct.Struct("<4sIQQQQQB")  # magic, version, L, H, N, d, D, dtype (cache.py:34)


@dataclass(frozen=True)
class CacheMeta:
    """Shape card of a cache (cache.py:37-73)."""

    n_layers: int
    n_heads: int
    n_tokens: int
    head_dim: int
    dtype: str = "f32"
    model_id: str = ""

    @property
    def model_dim(self) -> int:
        return self.n_heads * self.head_dim

    def meta_hash(self) -> bytes:
        """sha256 of the packed fixed header + model_id (cache.py:59-70)."""
        blob = _FIXED_HEADER.pack(CACHE_MAGIC, CACHE_VERSION, self.n_layers, self.n_heads,
                                  self.n_tokens, self.head_dim, self.model_dim,
                                  _DTYPE_CODES[self.dtype])
        return hashlib.sha256(blob + self.model_id.encode()).digest()


def _section_offsets(meta: CacheMeta, header_len: int) -> np.ndarray:
    """cache.py:143-148."""
    n_sections = 2 * meta.n_layers * meta.n_heads
    data_base = header_len + 8 * n_sections
    section_bytes = meta.n_tokens * meta.head_dim * _SCALAR_BYTES
    return data_base + section_bytes * np.arange(n_sections, dtype=np.uint64)


def section_index(meta: CacheMeta, layer: int, head: int, kind: str) -> int:
    """cache.py:151-156."""
    if kind not in ("keys", "values"):
        raise InputError(f"unknown section kind {kind!r}")
    if not (0 <= layer < meta.n_layers and 0 <= head < meta.n_heads):
        raise InputError(f"(layer={layer}, head={head}) out of range")
    return (layer * meta.n_heads + head) * 2 + (0 if kind == "keys" else 1)


def _read_exact(f, n: int, what: str) -> bytes:
    blob = f.read(n)
    if len(blob) < n:
        raise FormatError(f"file truncated reading {what}", offset=f.tell())
    return blob


def read_header(path) -> tuple[CacheMeta, np.ndarray]:
    """Validate a TKKV file exactly like the reference (cache.py:166-192 and the size check of
    CacheFile.__init__, cache.py:198-211); returns (meta, section offsets)."""
    path = os.fspath(path)
    with open(path, "rb") as f:
        fixed = _read_exact(f, _FIXED_HEADER.size, "header")
        magic, version, L, H, N, d, D, dtype_code = _FIXED_HEADER.unpack(fixed)
        if magic != CACHE_MAGIC:
            raise FormatError(f"bad magic {magic!r}", offset=0)
        if version != CACHE_VERSION:
            raise FormatError(f"unsupported cache version {version}", offset=4)
        if dtype_code not in _DTYPE_NAMES:
            raise FormatError(f"unknown dtype code {dtype_code}", offset=_FIXED_HEADER.size - 1)
        if min(L, H, N, d) < 1 or D != H * d:
            raise FormatError(f"invalid meta L={L} H={H} N={N} d={d} D={D}", offset=8)
        (mid_len,) = struct.unpack("<I", _read_exact(f, 4, "model_id length"))
        if mid_len > 4096:
            raise FormatError(f"implausible model_id length {mid_len}", offset=f.tell() - 4)
        model_id = _read_exact(f, mid_len, "model_id").decode()
        meta = CacheMeta(L, H, N, d, _DTYPE_NAMES[dtype_code], model_id)
        table_at = f.tell()
        table = np.frombuffer(_read_exact(f, 8 * 2 * L * H, "offset table"), dtype="<u8")
        expected = _section_offsets(meta, table_at)
        if not np.array_equal(table, expected):
            raise FormatError("offset table does not match meta-derived layout", offset=table_at)
        f.seek(0, os.SEEK_END)
        size = f.tell()
    section_bytes = N * d * _SCALAR_BYTES
    want = int(table[-1]) + section_bytes
    if size != want:
        raise FormatError(f"file size {size} != expected {want}", offset=min(size, want))
    return meta, table.astype(np.int64)


class TkkvFile:
    """Validated TKKV file, loadable into device caches layer by layer."""

    def __init__(self, path, *, staging_rows: int = 1 << 16):
        self.path = os.fspath(path)
        self.meta, self.offsets = read_header(self.path)
        if self.meta.head_dim > ops.HEAD_DIM:
            raise InputError(f"head_dim {self.meta.head_dim} > {ops.HEAD_DIM} is not supported")
        self._mm = np.memmap(self.path, dtype=np.uint8, mode="r")
        self.staging_rows = staging_rows

    def section(self, layer: int, head: int, kind: str) -> np.ndarray:
        """The (N, d) f32 section as a zero-copy view of the file."""
        m = self.meta
        base = int(self.offsets[section_index(m, layer, head, kind)])
        nbytes = m.n_tokens * m.head_dim * _SCALAR_BYTES
        return self._mm[base:base + nbytes].view("<f4").reshape(m.n_tokens, m.head_dim)

    def load_layer(self, layer: int, device, *, heads=None, row_range=None, capacity: int | None = None,
                   out=None):
        """(K, V) bf16 [1, len(heads), capacity, 128] device caches for one layer; rows
        [lo, hi) of every section land at rows [0, hi - lo). capacity >= hi - lo leaves headroom
        for the generation window (GenWindow rows after the context)."""
        m = self.meta
        heads = list(range(m.n_heads)) if heads is None else list(heads)
        lo, hi = (0, m.n_tokens) if row_range is None else row_range
        if not (0 <= lo <= hi <= m.n_tokens):
            raise InputError(f"row range {(lo, hi)} outside [0, {m.n_tokens}]")
        n = hi - lo
        cap = n if capacity is None else capacity
        if cap < n:
            raise InputError("capacity smaller than the row range")
        dev = torch.device(device)
        if out is None:
            K = torch.zeros((1, len(heads), cap, ops.HEAD_DIM), dtype=torch.bfloat16, device=dev)
            V = torch.zeros_like(K)
        else:
            K, V = out
        lib = _lib.load()
        stream = torch.cuda.current_stream(dev)
        rows = max(1, min(self.staging_rows, n))
        stage = [torch.empty((rows, m.head_dim), dtype=torch.float32, pin_memory=True) for _ in range(2)]
        dstage = [torch.empty((rows, m.head_dim), dtype=torch.float32, device=dev) for _ in range(2)]
        done = [torch.cuda.Event() for _ in range(2)]
        slot = 0
        for hi_, h in enumerate(heads):
            for kind, dst in (("keys", K), ("values", V)):
                sec = self.section(layer, h, kind)
                for r0 in range(lo, hi, rows):
                    r1 = min(hi, r0 + rows)
                    done[slot].synchronize()  # staging slot free again (its H2D + convert finished)
                    stage[slot][: r1 - r0].numpy()[...] = sec[r0:r1]
                    dstage[slot][: r1 - r0].copy_(stage[slot][: r1 - r0], non_blocking=True)
                    target = dst[0, hi_, r0 - lo:r1 - lo]
                    _lib.check(lib.tkv_convert_rows_f32(ctypes.c_void_p(dstage[slot].data_ptr()), r1 - r0,
                                                        m.head_dim, ctypes.c_void_p(target.data_ptr()),
                                                        ctypes.c_void_p(stream.cuda_stream)))
                    done[slot].record(stream)
                    slot ^= 1
        stream.synchronize()
        return K, V
