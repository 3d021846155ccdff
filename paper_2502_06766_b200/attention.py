"""Drop-in `topk_attend` (reference attention.py:125-167) backed by the B200 kernels.

Same signature, argument meaning, side effects and error behaviour as the reference:

* k < 1 → InputError (attention.py:144-145); k > N → warning + clamp (attention.py:147-149);
  q must be a finite 1-d vector of the index dim (ShapeError / DomainError, ann.py:209-211).
* index counters distance_evals += N, queries += 1 (ann.py:216-217); retrieval_log gets the
  retrieved ids — score-desc/id-asc, or ascending-unique with a pinned prefix
  (attention.py:152-156); accounting cold_reads/bytes_moved/hot_ops (attention.py:162-166).
* unknown combine → ConfigError raised after the retrieval side effects (attention.py:122).
* returns the (d,) float32 output of the joint (or additive) softmax over the retrieved rows
  and the window rows (attention.py:107-122).

Two value paths:
  - `fetch_values` is a DeviceValues handle (index.attach_values(V)): V is resident in HBM,
    the window rows are copied into the index's headroom rows and ONE device call does scan,
    select, gather and softmax (tkv_topk_decode_attention).
  - any other callable (e.g. the reference's ValueTier lambda): the exact top-k is computed on
    the device, fetch_values(ids) is called once like in the reference, and the attention over
    the retrieved rows + window runs on the device over a compact cache of those rows
    (k = len(ids) selects them all; scores are recomputed by the same kernel).
Numerics: inputs are stored as bf16 on the device; scores accumulate in fp32.
"""

from __future__ import annotations

import logging
from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .ann import DTYPE, DeviceValues, MipsIndex, _pad_rows, as_vector, default_scale, device_search
from .errors import ConfigError, InputError, ShapeError

logger = logging.getLogger(__name__)

SCORE_BYTES = 4


def VALUE_ROW_BYTES(d: int) -> int:  # noqa: N802 - reference name (attention.py:33)
    return (d + 1) * SCORE_BYTES


@dataclass
class TierAccounting:
    """Per-step movement counters between the cold cache tier and the hot tier (attention.py:36-49)."""

    cold_reads: int = 0
    hot_ops: int = 0
    bytes_moved: int = 0

    def snapshot(self) -> dict:
        return {"cold_reads": self.cold_reads, "hot_ops": self.hot_ops, "bytes_moved": self.bytes_moved}


def _window(win_keys, win_values, d: int) -> tuple[np.ndarray, np.ndarray]:
    wk = np.asarray(win_keys, dtype=DTYPE).reshape(-1, d) if np.size(win_keys) else np.zeros((0, d), DTYPE)
    wv = np.asarray(win_values, dtype=DTYPE).reshape(-1, d) if np.size(win_values) else np.zeros((0, d), DTYPE)
    if wk.shape != wv.shape:
        raise ShapeError(f"window keys {wk.shape} and values {wv.shape} differ")
    return wk, wv


def _to_dev(a: np.ndarray, dev) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(_pad_rows(a))).to(dev, torch.bfloat16)


def topk_attend(q, index: MipsIndex, fetch_values, win_keys, win_values, k: int,
                accounting: TierAccounting, ef_search: int | None = None, combine: str = "joint",
                pinned_prefix: int = 0, retrieval_log: list | None = None) -> np.ndarray:
    """One head's attention output over retrieved cache rows plus the window."""
    if k < 1:
        raise InputError("k must be >= 1")
    d = index.dim
    N = index.n_keys
    if k > N:
        logger.warning("k=%d exceeds cache size %d; clamping", k, N)
        k = N
    qv = as_vector(q)
    if qv.shape[0] != d:
        raise ShapeError(f"query dim {qv.shape[0]} != index dim {d}")
    wk, wv = _window(win_keys, win_values, d)
    n_gen = wk.shape[0]
    scale = default_scale(d)
    dev = index.device
    resident = isinstance(fetch_values, DeviceValues) and fetch_values.index is index and index.v_dev is not None
    good_combine = combine in ("joint", "additive")

    if resident and good_combine:
        index.ensure_capacity(N + n_gen)
        if n_gen:
            index.k_dev[0, 0, N:N + n_gen] = _to_dev(wk, dev)
            index.v_dev[0, 0, N:N + n_gen] = _to_dev(wv, dev)
        qd = torch.from_numpy(_pad_rows(qv[None, :])[None]).to(dev, torch.bfloat16)
        out, idx_t, sc_t = ops.topk_decode_attention(
            qd, index.k_dev, index.v_dev, N, k, n_win=n_gen, scale=scale, combine=combine,
            pinned_prefix=pinned_prefix, sorted=True, max_ctx=N)
        ids = idx_t[0, 0].cpu().numpy().astype(np.int64)
        result = out[0, 0, :d].cpu().numpy().astype(DTYPE)
    else:
        ids, _ = device_search(index, qv, k)
        result = None
    index.distance_evals += N
    index.queries += 1
    if pinned_prefix > 0:
        pinned = np.arange(min(pinned_prefix, N), dtype=np.int64)
        ids = np.unique(np.concatenate([pinned, ids]))
    if retrieval_log is not None:
        retrieval_log.append(ids)

    if result is None:
        # generic fetch_values: one call with the retrieved ids, as the reference does
        v_ctx = np.asarray(fetch_values(ids), dtype=DTYPE).reshape(len(ids), d)
    accounting.cold_reads += len(ids)
    accounting.bytes_moved += len(ids) * VALUE_ROW_BYTES(d)
    accounting.hot_ops += n_gen
    if not good_combine:
        raise ConfigError(f"unknown combine mode {combine!r}")
    if result is not None:
        return result

    # attention over exactly the retrieved rows + window on the device
    m = len(ids)
    rows = m + n_gen
    kc = np.zeros((rows, d), dtype=DTYPE)
    vc = np.zeros((rows, d), dtype=DTYPE)
    kc[:m] = index.row_keys(ids)
    vc[:m] = v_ctx
    kc[m:] = wk
    vc[m:] = wv
    kd = _to_dev(kc, dev)[None, None]
    vd = _to_dev(vc, dev)[None, None]
    qd = torch.from_numpy(_pad_rows(qv[None, :])[None]).to(dev, torch.bfloat16)
    out, _, _ = ops.topk_decode_attention(qd, kd, vd, m, m, n_win=n_gen, scale=scale,
                                          combine=combine, max_ctx=m, no_filter=True)
    return out[0, 0, :d].cpu().numpy().astype(DTYPE)
