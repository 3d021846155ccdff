"""Flat maximum-inner-product index with device-resident keys (drop-in for ann.py's flat kind).

Mirrors the reference's flat-index surface — `build_index` (ann.py:107-137), `MipsIndex`
(ann.py:58-89), `TopKResult` (ann.py:47-55), `knn_search` (ann.py:203-221) — with the scan and
the exact selection running on the B200 (libtkv: tkv_topk_search). The keys are validated
like the reference (tensor.py:17-28), kept as the reference's f32 host copy for `row_keys`,
and uploaded once as a bf16 [1, 1, rows, 128] cache (zero-padded when d < 128; zero columns
do not change any dot product).

The approximate "graph" index kind (ann.py:92-151, ann_kernels.py:50-320) is out of scope for
this hot path: exact top-k is the north star.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import ops
from .errors import ConfigError, DomainError, InputError, ShapeError

DTYPE = np.float32


def as_matrix(a) -> np.ndarray:
    """tensor.py:17-28: C-contiguous f32 2-d, finite."""
    m = np.ascontiguousarray(a, dtype=DTYPE)
    if m.ndim != 2:
        raise ShapeError(f"expected 2-d matrix, got ndim={m.ndim}")
    if not np.isfinite(m).all():
        raise DomainError("matrix entries must be finite")
    return m


def as_vector(a) -> np.ndarray:
    """tensor.py:31-40: C-contiguous f32 1-d, finite."""
    v = np.ascontiguousarray(a, dtype=DTYPE)
    if v.ndim != 1:
        raise ShapeError(f"expected 1-d vector, got ndim={v.ndim}")
    if not np.isfinite(v).all():
        raise DomainError("vector entries must be finite")
    return v


@dataclass(frozen=True)
class TopKResult:
    """Scores (descending) and the cache rows they belong to (ann.py:47-55)."""

    vals: np.ndarray  # float32
    ids: np.ndarray  # int64

    def __len__(self) -> int:
        return len(self.ids)


def _default_device() -> torch.device:
    if not torch.cuda.is_available():
        from .errors import DeviceError

        raise DeviceError("no CUDA device: the B200 index has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _pad_rows(a: np.ndarray, width: int = ops.HEAD_DIM) -> np.ndarray:
    n, d = a.shape
    if d == width:
        return a
    out = np.zeros((n, width), dtype=DTYPE)
    out[:, :d] = a
    return out


@dataclass
class MipsIndex:
    """Flat index over one head's keys; K lives in HBM as bf16 rows (+ window headroom)."""

    kind: str
    dim: int
    n_keys: int
    keys: np.ndarray  # reference-compatible f32 host copy (ann.py:114)
    device: torch.device
    k_dev: torch.Tensor = field(repr=False)  # [1, 1, rows, 128] bf16
    v_dev: torch.Tensor | None = field(default=None, repr=False)
    distance_evals: int = 0
    queries: int = 0

    @property
    def n_nodes(self) -> int:
        return self.n_keys

    @property
    def capacity(self) -> int:
        return int(self.k_dev.shape[2])

    def row_keys(self, ids: np.ndarray) -> np.ndarray:
        """ann.py:81-85."""
        return self.keys[ids]

    def reset_counters(self) -> None:
        self.distance_evals = 0
        self.queries = 0

    def ensure_capacity(self, rows: int) -> None:
        """Grow the device buffers so rows [n_keys, rows) can hold window rows."""
        if rows <= self.capacity:
            return
        new = max(rows, self.capacity + max(64, self.capacity // 8))
        for name in ("k_dev", "v_dev"):
            t = getattr(self, name)
            if t is None:
                continue
            g = torch.zeros((1, 1, new, ops.HEAD_DIM), dtype=torch.bfloat16, device=self.device)
            g[:, :, : self.n_keys] = t[:, :, : self.n_keys]
            setattr(self, name, g)

    def attach_values(self, values) -> "DeviceValues":
        """Upload the head's value rows next to its keys; the returned handle is a valid
        `fetch_values` for topk_attend and keeps V resident in HBM (no host gather)."""
        v = as_matrix(values)
        if v.shape != (self.n_keys, self.dim):
            raise ShapeError(f"values shape {v.shape} != {(self.n_keys, self.dim)}")
        buf = torch.zeros((1, 1, self.capacity, ops.HEAD_DIM), dtype=torch.bfloat16, device=self.device)
        buf[0, 0, : self.n_keys] = torch.from_numpy(_pad_rows(v)).to(self.device, torch.bfloat16)
        self.v_dev = buf
        return DeviceValues(self, v)


class DeviceValues:
    """Device-resident value rows bound to one MipsIndex; callable like fetch_values."""

    def __init__(self, index: MipsIndex, host_values: np.ndarray):
        self.index = index
        self.host_values = host_values

    def __call__(self, ids: np.ndarray) -> np.ndarray:
        return self.host_values[ids]


def build_index(keys, kind: str = "flat", params=None, *, device=None,
                window_capacity: int = 64) -> MipsIndex:
    """Index one (N, d) key matrix (ann.py:107-137); flat only on this path."""
    k = as_matrix(keys)
    if k.shape[0] < 1:
        raise InputError("cannot index an empty key matrix")
    if kind == "graph":
        raise ConfigError("graph (approximate) indexes are not part of the B200 exact top-k path")
    if kind != "flat":
        raise InputError(f"unknown index kind {kind!r}")
    n, d = k.shape
    if d > ops.HEAD_DIM:
        raise ShapeError(f"head dim {d} > {ops.HEAD_DIM} is not supported by this build")
    dev = torch.device(device) if device is not None else _default_device()
    buf = torch.zeros((1, 1, n + max(0, window_capacity), ops.HEAD_DIM), dtype=torch.bfloat16, device=dev)
    buf[0, 0, :n] = torch.from_numpy(_pad_rows(k)).to(dev, torch.bfloat16)
    return MipsIndex("flat", d, n, k, dev, buf)


def _device_q(idx: MipsIndex, qv: np.ndarray) -> torch.Tensor:
    qp = np.zeros((1, 1, ops.HEAD_DIM), dtype=DTYPE)
    qp[0, 0, : qv.shape[0]] = qv
    return torch.from_numpy(qp).to(idx.device, torch.bfloat16)


def device_search(idx: MipsIndex, qv: np.ndarray, k: int) -> tuple[np.ndarray, np.ndarray]:
    """Exact top-min(k, N) on the device; returns (ids int64, vals f32) TopKResult-ordered
    (score desc, id asc, ann.py:166 — ordered on the device for every k)."""
    k = min(k, idx.n_keys)
    q = _device_q(idx, qv)
    ids_t, sc_t = ops.topk_search(q, idx.k_dev, idx.n_keys, k, sorted=True, max_ctx=idx.n_keys)
    ids = ids_t[0, 0].cpu().numpy().astype(np.int64)
    vals = sc_t[0, 0].cpu().numpy().astype(DTYPE)
    return ids, vals


def knn_search(idx: MipsIndex, q, k: int, ef_search: int | None = None) -> TopKResult:
    """Top-k rows by inner product (ann.py:203-218): exact, ties to the lower row id."""
    qv = as_vector(q)
    if qv.shape[0] != idx.dim:
        raise ShapeError(f"query dim {qv.shape[0]} != index dim {idx.dim}")
    if k < 1:
        raise InputError("k must be >= 1")
    ids, vals = device_search(idx, qv, k)
    idx.distance_evals += idx.n_keys
    idx.queries += 1
    return TopKResult(vals, ids)


def recall_at_k(approx: TopKResult, exact: TopKResult) -> float:
    """ann.py:224-229."""
    if len(exact) == 0:
        raise InputError("exact result is empty")
    return np.intersect1d(approx.ids, exact.ids).size / len(exact)


def default_scale(d: int) -> float:
    return 1.0 / math.sqrt(d)
