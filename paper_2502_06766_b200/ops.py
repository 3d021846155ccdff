"""Batched device API over libtkv: one call = one layer's top-k decode attention.

    out, idx, scores = topk_decode_attention(q, k_cache, v_cache, n_ctx, k)

replaces the per-(layer, head) loop of the reference decode step (attention.py:213-230, each
iteration a `topk_attend`, attention.py:125-167) for every head and batch entry at once.
Tensors are torch CUDA tensors (torch is used only for device memory and streams); the work
is done by the sm_100a kernels behind the C ABI (include/tkv.h). There is no CPU path: CPU
tensors are rejected, a missing native library raises DeviceError.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import torch

from . import _lib
from .errors import ConfigError, InputError, ShapeError

HEAD_DIM = 128
_COMBINE = {"joint": _lib.COMBINE_JOINT, "additive": _lib.COMBINE_ADDITIVE}


def _vp(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(device: torch.device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def combine_code(combine: str) -> int:
    try:
        return _COMBINE[combine]
    except KeyError:
        raise ConfigError(f"unknown combine mode {combine!r}") from None


def make_problem(B: int, Hq: int, Hkv: int, cache_rows: int, max_ctx: int, k: int, *,
                 pinned_prefix: int = 0, scale: float | None = None, combine: str = "joint",
                 sorted: bool = False, no_filter: bool = False, row_offset: int = 0,
                 head_dim: int = HEAD_DIM,
                 tc_scan: bool | None = None, parts: int = 0, list_gather: bool = False,
                 head: bool | str | None = None, host_q: bool = False) -> _lib.Problem:
    p = _lib.Problem()
    p.batch, p.n_q_heads, p.n_kv_heads, p.head_dim = B, Hq, Hkv, head_dim
    p.cache_rows, p.max_ctx, p.k = cache_rows, max_ctx, k
    p.pinned_prefix = pinned_prefix
    p.scale = float(scale) if scale is not None else 1.0 / math.sqrt(head_dim)
    p.combine = combine_code(combine)
    p.flags = (_lib.F_SORTED if sorted else 0) | (_lib.F_NO_FILTER if no_filter else 0)
    if tc_scan is None:  # the tcgen05 scan is the default; TKV_SCAN=hmma selects the mma.sync scan
        tc_scan = os.environ.get("TKV_SCAN", "") != "hmma"
    if not tc_scan:
        p.flags |= _lib.F_SCAN_HMMA
    if not 0 <= parts <= 15:
        raise ConfigError("parts must be in 0..15 (0 = automatic)")
    p.flags |= parts << _lib.F_PARTS_SHIFT
    if list_gather:
        p.flags |= _lib.F_GATHER_LIST
    # k-th + gather kernel: True = per-head CTAs (head_topk_kernel), "cluster" = one 4-CTA cluster
    # per head (clus_topk_kernel), False = k-th kernel + candidate gather; None: automatic
    if head == "cluster":
        p.flags |= _lib.F_CLUSTER
    elif head is not None:
        p.flags |= (_lib.F_HEAD | _lib.F_NO_CLUSTER) if head else (_lib.F_NO_HEAD | _lib.F_NO_CLUSTER)
    if host_q:  # q in pinned host memory, staged on device inside the call
        p.flags |= _lib.F_HOST_Q
    p.row_offset = row_offset
    return p


class Workspace:
    """Device scratch for one problem layout, zeroed once (tkv_workspace_init).

    One workspace per stream: the kernels keep self-resetting control words in it.
    """

    def __init__(self, problem: _lib.Problem, device: torch.device):
        self.device = torch.device(device)
        self.nbytes = _lib.workspace_bytes(problem)
        self._buf = torch.empty(self.nbytes + 256, dtype=torch.uint8, device=self.device)
        base = self._buf.data_ptr()
        self.ptr = ctypes.c_void_p((base + 255) // 256 * 256)
        _lib.call("tkv_workspace_init", ctypes.byref(problem), self.ptr, self.nbytes,
                  _stream(self.device))

    def fits(self, problem: _lib.Problem) -> bool:
        return _lib.workspace_bytes(problem) <= self.nbytes

    def fallbacks(self, problem: _lib.Problem) -> int:
        """Selections that needed the exactness fallback on this workspace (synchronous read)."""
        n = ctypes.c_uint32(0)
        _lib.call("tkv_workspace_fallbacks", ctypes.byref(problem), self.ptr, self.nbytes, ctypes.byref(n))
        return int(n.value)


_WS_CACHE: dict[tuple, Workspace] = {}


def workspace_for(problem: _lib.Problem, device: torch.device) -> Workspace:
    dev = torch.device(device)
    key = (dev.index, torch.cuda.current_stream(dev).cuda_stream, problem.batch, problem.n_q_heads,
           problem.n_kv_heads)
    ws = _WS_CACHE.get(key)
    if ws is None or not ws.fits(problem):
        ws = Workspace(problem, dev)
        _WS_CACHE[key] = ws
    return ws


def _is_host_pinned(t) -> bool:
    return isinstance(t, torch.Tensor) and not t.is_cuda and t.is_pinned()


def _check_cuda_bf16(name: str, t: torch.Tensor, ndim: int, allow_pinned: bool = False) -> None:
    if not isinstance(t, torch.Tensor):
        raise ShapeError(f"{name} must be a torch tensor")
    if not t.is_cuda and not (allow_pinned and t.is_pinned()):
        raise ShapeError(f"{name} must be a CUDA tensor{' or pinned host memory' if allow_pinned else ''} "
                         "(the B200 path has no CPU fallback)")
    if t.dtype != torch.bfloat16:
        raise ShapeError(f"{name} must be bfloat16, got {t.dtype}")
    if t.dim() != ndim or not t.is_contiguous():
        raise ShapeError(f"{name} must be a contiguous {ndim}-d tensor, got shape {tuple(t.shape)}")


def _as_counts(name: str, v, B: int, device) -> torch.Tensor:
    if isinstance(v, torch.Tensor):
        if v.dtype != torch.int32 or v.numel() != B or not v.is_cuda:
            raise ShapeError(f"{name} must be an int32 CUDA tensor of {B} entries")
        return v.contiguous()
    vals = [int(v)] * B if isinstance(v, int) else [int(x) for x in v]
    if len(vals) != B:
        raise ShapeError(f"{name} needs {B} entries, got {len(vals)}")
    return torch.tensor(vals, dtype=torch.int32, device=device)


def _host_max(v) -> int:
    """Largest context length of a host-side n_ctx (int or sequence): no device reduction and
    no device→host read on the call path."""
    return int(v) if isinstance(v, int) else max(int(x) for x in v)


@dataclass
class Shapes:
    B: int
    Hq: int
    Hkv: int
    cache_rows: int


def check_shapes(q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor | None) -> Shapes:
    """q may be a pinned host tensor (TKV_F_HOST_Q: staged on device by the call itself)."""
    _check_cuda_bf16("q", q, 3, allow_pinned=True)
    _check_cuda_bf16("k_cache", k_cache, 4)
    B, Hq, d = q.shape
    if d != HEAD_DIM:
        raise ShapeError(f"head_dim {d} unsupported (this build: {HEAD_DIM})")
    Bk, Hkv, rows, dk = k_cache.shape
    if Bk != B or dk != d:
        raise ShapeError(f"k_cache shape {tuple(k_cache.shape)} incompatible with q {tuple(q.shape)}")
    if v_cache is not None:
        _check_cuda_bf16("v_cache", v_cache, 4)
        if v_cache.shape != k_cache.shape:
            raise ShapeError("v_cache shape must equal k_cache shape")
    if Hq % Hkv:
        raise ShapeError(f"Hq={Hq} is not a multiple of Hkv={Hkv}")
    if q.is_cuda and q.device != k_cache.device:
        raise ShapeError("q and k_cache live on different devices")
    return Shapes(B, Hq, Hkv, rows)


def topk_decode_attention(q, k_cache, v_cache, n_ctx, k: int, *, n_win=None, scale=None,
                          combine: str = "joint", pinned_prefix: int = 0, sorted: bool = False,
                          max_ctx: int | None = None, no_filter: bool = False, row_offset: int = 0,
                          out=None, idx=None, scores=None, workspace: Workspace | None = None,
                          tc_scan: bool | None = None, parts: int = 0,
                          list_gather: bool = False, head: bool | str | None = None):
    """Exact top-k decode attention for every (batch, q head) of one layer.

    q [B, Hq, 128] bf16; k_cache/v_cache [B, Hkv, rows, 128] bf16 with the context in rows
    [0, n_ctx[b]) and the generation window in [n_ctx[b], n_ctx[b] + n_win[b]).
    Returns (out [B, Hq, 128] f32, idx [B, Hq, k] int32, scores [B, Hq, k] f32):
    selected global row ids (-1 pads when k > n_ctx[b]) and their raw dot products.
    """
    if k < 1:
        raise InputError("k must be >= 1")
    s = check_shapes(q, k_cache, v_cache)
    dev = k_cache.device
    n_ctx_t = _as_counts("n_ctx", n_ctx, s.B, dev)
    n_win_t = None if n_win is None else _as_counts("n_win", n_win, s.B, dev)
    if max_ctx is None:
        max_ctx = s.cache_rows if isinstance(n_ctx, torch.Tensor) else _host_max(n_ctx)
    prob = make_problem(s.B, s.Hq, s.Hkv, s.cache_rows, max_ctx, k, pinned_prefix=pinned_prefix,
                        scale=scale, combine=combine, sorted=sorted, no_filter=no_filter,
                        row_offset=row_offset, tc_scan=tc_scan, parts=parts,
                        list_gather=list_gather, head=head,
                        host_q=not q.is_cuda)
    ws = workspace or workspace_for(prob, dev)
    out = out if out is not None else torch.empty((s.B, s.Hq, HEAD_DIM), dtype=torch.float32, device=dev)
    idx = idx if idx is not None else torch.empty((s.B, s.Hq, k), dtype=torch.int32, device=dev)
    scores = scores if scores is not None else torch.empty((s.B, s.Hq, k), dtype=torch.float32, device=dev)
    _lib.call("tkv_topk_decode_attention", ctypes.byref(prob), _vp(q), _vp(k_cache), _vp(v_cache),
              _vp(n_ctx_t), _vp(n_win_t), _vp(out), _vp(idx), _vp(scores), ws.ptr, ws.nbytes,
              _stream(dev))
    return out, idx, scores


def topk_decode_step(q, k_new, v_new, k_cache, v_cache, n_ctx, n_win, k: int, *, scale=None,
                     combine: str = "joint", pinned_prefix: int = 0, sorted: bool = False,
                     max_ctx: int | None = None, out=None, idx=None, scores=None,
                     workspace: Workspace | None = None, tc_scan: bool | None = None,
                     parts: int = 0, list_gather: bool = False, head: bool | str | None = None):
    """One decode step of one layer (decode_step, attention.py:203-230): append this token's
    k_new/v_new [B, Hkv, 128] to the window (GenWindow.append, attention.py:210; n_win is a
    device int32 counter advanced in place) and attend over context + window, in one call."""
    if k < 1:
        raise InputError("k must be >= 1")
    s = check_shapes(q, k_cache, v_cache)
    dev = k_cache.device
    n_ctx_t = _as_counts("n_ctx", n_ctx, s.B, dev)
    if not (isinstance(n_win, torch.Tensor) and n_win.dtype == torch.int32 and n_win.is_cuda and n_win.numel() == s.B):
        raise ShapeError("n_win must be a device int32 tensor of B counters (advanced in place)")
    for name, t in (("k_new", k_new), ("v_new", v_new)):
        _check_cuda_bf16(name, t, 3, allow_pinned=True)
        if tuple(t.shape) != (s.B, s.Hkv, HEAD_DIM):
            raise ShapeError(f"{name} must be [B, Hkv, {HEAD_DIM}]")
    if max_ctx is None:
        max_ctx = s.cache_rows if isinstance(n_ctx, torch.Tensor) else _host_max(n_ctx)
    prob = make_problem(s.B, s.Hq, s.Hkv, s.cache_rows, max_ctx, k, pinned_prefix=pinned_prefix,
                        scale=scale, combine=combine, sorted=sorted, tc_scan=tc_scan,
                        parts=parts, list_gather=list_gather, head=head,
                        host_q=not q.is_cuda)
    ws = workspace or workspace_for(prob, dev)
    out = out if out is not None else torch.empty((s.B, s.Hq, HEAD_DIM), dtype=torch.float32, device=dev)
    idx = idx if idx is not None else torch.empty((s.B, s.Hq, k), dtype=torch.int32, device=dev)
    _lib.call("tkv_topk_decode_step", ctypes.byref(prob), _vp(q), _vp(k_new), _vp(v_new), _vp(k_cache),
              _vp(v_cache), _vp(n_ctx_t), _vp(n_win), _vp(out), _vp(idx), _vp(scores), ws.ptr, ws.nbytes,
              _stream(dev))
    return out, idx, scores


def topk_search(q, k_cache, n_ctx, k: int, *, sorted: bool = True, max_ctx: int | None = None,
                no_filter: bool = False, row_offset: int = 0, workspace: Workspace | None = None,
                tc_scan: bool | None = None, parts: int = 0, head: bool | str | None = None):
    """Exact top-k rows per (batch, q head) without attention (knn_search flat, ann.py:203-218).

    Returns (idx [B, Hq, k] int32, scores [B, Hq, k] f32), TopKResult-ordered when sorted.
    """
    if k < 1:
        raise InputError("k must be >= 1")
    s = check_shapes(q, k_cache, None)
    dev = k_cache.device
    n_ctx_t = _as_counts("n_ctx", n_ctx, s.B, dev)
    if max_ctx is None:
        max_ctx = s.cache_rows if isinstance(n_ctx, torch.Tensor) else _host_max(n_ctx)
    prob = make_problem(s.B, s.Hq, s.Hkv, s.cache_rows, max_ctx, k, sorted=sorted,
                        no_filter=no_filter, row_offset=row_offset, tc_scan=tc_scan,
                        parts=parts, head=head, host_q=not q.is_cuda)
    ws = workspace or workspace_for(prob, dev)
    idx = torch.empty((s.B, s.Hq, k), dtype=torch.int32, device=dev)
    scores = torch.empty((s.B, s.Hq, k), dtype=torch.float32, device=dev)
    _lib.call("tkv_topk_search", ctypes.byref(prob), _vp(q), _vp(k_cache), _vp(n_ctx_t), _vp(idx),
              _vp(scores), ws.ptr, ws.nbytes, _stream(dev))
    return idx, scores


def kv_append(k_cache, v_cache, k_new, v_new, count, *, base=None, advance: bool = True) -> None:
    """Write this token's k/v rows ([B, Hkv, 128] bf16) at row base[b] + count[b] (GenWindow.append,
    attention.py:94-100; base = n_ctx, count = n_win grows the window after the context).
    With advance, count[b] += 1 on device (no host sync)."""
    _check_cuda_bf16("k_cache", k_cache, 4)
    _check_cuda_bf16("v_cache", v_cache, 4)
    _check_cuda_bf16("k_new", k_new, 3)
    _check_cuda_bf16("v_new", v_new, 3)
    B, Hkv, rows, d = k_cache.shape
    if k_new.shape != (B, Hkv, d) or v_new.shape != (B, Hkv, d) or v_cache.shape != k_cache.shape:
        raise ShapeError("k_new/v_new must be [B, Hkv, d] matching the caches")
    for name, t in (("count", count), ("base", base)):
        if t is None and name == "base":
            continue
        if not (isinstance(t, torch.Tensor) and t.dtype == torch.int32 and t.is_cuda and t.numel() == B):
            raise ShapeError(f"{name} must be an int32 CUDA tensor of B entries")
    _lib.call("tkv_kv_append", B, Hkv, d, rows, _vp(k_cache), _vp(v_cache), _vp(k_new), _vp(v_new),
              _vp(base), _vp(count), 1 if advance else 0, _stream(k_cache.device))
