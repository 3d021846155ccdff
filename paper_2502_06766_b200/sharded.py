"""Token-range sharded exact top-k decode attention (decode-time context parallelism).

The reference is single-process; the scaling story here is to shard the
context of every KV head by token range across the GPUs of one node: rank g holds global
rows [row_offset_g, row_offset_g + n_local). One layer step is

  1. local scan + exact local top-k            (tkv_shard_candidates, no communication)
  2. all-gather of k packed (score key, ~global id) candidates per q head
  3. exact global top-k over G·k candidates   (tkv_shard_merge; ties → lower global id, which
     is the lower rank because shards are contiguous — identical to the unsharded order)
  4. each rank gathers the V rows it owns       (tkv_shard_partial, weights against the
     global max known to every rank, so partials add without rescaling)
  5. all-reduce SUM of (l, o[128]) per q head  (16.5 KB per rank at Hq=32)
  6. window rows + normalisation               (tkv_shard_finalize, window replicated)

Global top-k ⊆ ∪ local top-k, so the result equals the single-GPU one exactly (same ids;
outputs up to fp32 summation order). The communication goes through torch.distributed
(NCCL over NVLink on B200; gloo for the CPU tests). The compute stages are pluggable so the
protocol itself can be tested on CPU with the oracle's stages (tests only); the product
default is `CudaStages` (libtkv), which fails loudly without the native library.
"""

from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from . import _lib, ops
from .errors import InputError


class CudaStages:
    """libtkv shard stages for one problem layout; owns the workspace shared by the stages."""

    def __init__(self, B: int, Hq: int, Hkv: int, cache_rows: int, max_ctx: int, k: int, *,
                 row_offset: int, device, scale=None, combine="joint", pinned_prefix=0,
                 sorted=False):
        self.prob = ops.make_problem(B, Hq, Hkv, cache_rows, max_ctx, k, row_offset=row_offset,
                                     scale=scale, combine=combine, pinned_prefix=pinned_prefix,
                                     sorted=sorted)
        self.device = torch.device(device)
        self.ws = ops.Workspace(self.prob, self.device)
        self.B, self.Hq, self.k = B, Hq, k
        D = ops.HEAD_DIM
        self.cand = torch.empty(B * Hq * k, dtype=torch.int64, device=self.device)
        self.idx = torch.empty((B, Hq, k), dtype=torch.int32, device=self.device)
        self.scores = torch.empty((B, Hq, k), dtype=torch.float32, device=self.device)
        self.partial = torch.empty(B * Hq * (D + 1), dtype=torch.float32, device=self.device)
        self.out = torch.empty((B, Hq, D), dtype=torch.float32, device=self.device)

    def _s(self):
        return ops._stream(self.device)

    def candidates(self, q, k_cache, n_ctx):
        _lib.call("tkv_shard_candidates", ctypes.byref(self.prob), ops._vp(q), ops._vp(k_cache),
                  ops._vp(n_ctx), ops._vp(self.cand), self.ws.ptr, self.ws.nbytes, self._s())
        return self.cand

    def merge(self, gathered, n_shards: int, list_len: int | None = None):
        """Exact global top-k over n_shards lists of list_len (default k) candidates per head."""
        _lib.call("tkv_shard_merge_lists", ctypes.byref(self.prob), ops._vp(gathered), n_shards,
                  self.k if list_len is None else list_len, ops._vp(self.idx),
                  ops._vp(self.scores), self.ws.ptr, self.ws.nbytes, self._s())
        return self.idx, self.scores

    def narrow_exact(self, gathered, n_shards: int, list_len: int) -> torch.Tensor:
        """Per-head exactness of a narrow exchange (int32 [B*Hq], 1 = exact); device kernel
        for narrow_exchange_exact."""
        ok = torch.empty(self.B * self.Hq, dtype=torch.int32, device=self.device)
        _lib.call("tkv_shard_narrow_check", ctypes.byref(self.prob), ops._vp(gathered), n_shards,
                  list_len, ops._vp(ok), self._s())
        return ok

    def partial_attend(self, q, k_cache, v_cache, n_ctx, idx, scores):
        _lib.call("tkv_shard_partial", ctypes.byref(self.prob), ops._vp(q), ops._vp(k_cache),
                  ops._vp(v_cache), ops._vp(n_ctx), ops._vp(idx), ops._vp(scores),
                  ops._vp(self.partial), self.ws.ptr, self.ws.nbytes, self._s())
        return self.partial

    def finalize(self, q, k_cache, v_cache, n_ctx, n_win, partial):
        _lib.call("tkv_shard_finalize", ctypes.byref(self.prob), ops._vp(q), ops._vp(k_cache),
                  ops._vp(v_cache), ops._vp(n_ctx), ops._vp(n_win), ops._vp(partial),
                  ops._vp(self.out), self.ws.ptr, self.ws.nbytes, self._s())
        return self.out


_U64_TO_I64 = torch.iinfo(torch.int64).min  # x ^ this maps unsigned order onto signed order


def narrow_k(k: int, world: int, c: float = 1.5) -> int:
    """Candidates each rank sends in the narrow exchange: ceil(c·k/world), at most k (SURVEY
    §8e mitigation; c ≈ 1.25–2). With i.i.d. relevance each shard holds ≈ k/world of the
    global top-k, so c·k/world covers it with margin."""
    if world < 1 or k < 1 or c <= 0:
        raise InputError(f"bad narrow_k arguments k={k} world={world} c={c}")
    return min(k, -(-int(c * k) // world))


def narrow_exchange_exact(gathered: torch.Tensor, world: int, k: int, kk: int) -> torch.Tensor:
    """Per (b, q head): is the global top-k over the narrow gathered lists exact?

    gathered: [world * BH * kk] packed composites (uint64 bit patterns in int64; 0 = empty
    slot), rank-major. A rank whose list is full may have withheld rows; each withheld row's
    composite is below that rank's smallest sent one (its floor t'_g — composites are unique).
    The merged k-th composite is ≥ T = max over full ranks of t'_g iff at least k gathered
    candidates are ≥ T; then no withheld row can enter the top-k and the result is exact.
    Conservative (a rank with exactly kk rows counts as full), never optimistic. Every rank
    evaluates this on identical data, so all ranks take the same branch without a collective."""
    g = (gathered ^ _U64_TO_I64).view(world, -1, kk)                 # [world, BH, kk]
    empty = torch.tensor(_U64_TO_I64, dtype=torch.int64, device=gathered.device)
    full = (g != empty).all(dim=2)                                   # [world, BH]
    floor = torch.where(full, g.min(dim=2).values, empty)             # [world, BH]
    T = floor.max(dim=0).values                                       # [BH]
    count = (g >= T.view(1, -1, 1)).sum(dim=(0, 2))                   # [BH]
    return (~full.any(dim=0)) | (count >= k)


def sharded_topk_attention(stages, q, k_shard, v_shard, n_ctx_local, n_win=None, *, group=None,
                           gathered: torch.Tensor | None = None, narrow=None,
                           stats: dict | None = None):
    """One layer's exact top-k attention with the context sharded by token range across the
    ranks of `group`. Every rank passes its shard (rows [row_offset, row_offset + n_local) in
    rows [0, n_local) of k_shard/v_shard, window rows after them, replicated) and receives the
    full result: (out [B, Hq, 128] f32, idx [B, Hq, k] global ids, scores).

    narrow: optional stages object of the same layout built with k' = narrow_k(k, world) < k
    (only its `candidates` and `k` are used). Each rank then all-gathers only its local
    top-k' (traffic ÷ k/k'); if `narrow_exchange_exact` fails for any head (skewed data: one
    shard holds more than k' of the global top-k) every rank re-runs the full-k exchange, so
    the result is always exact. Costs one device→host read of the exactness flag. `stats`,
    when given, receives {"narrow": bool used, "narrow_exact": bool}."""
    world = dist.get_world_size(group)
    if narrow is not None and narrow.k < stages.k:
        cand = narrow.candidates(q, k_shard, n_ctx_local)
        small = torch.empty(world * cand.numel(), dtype=cand.dtype, device=cand.device)
        dist.all_gather_into_tensor(small, cand, group=group)
        if hasattr(stages, "narrow_exact"):
            ok = stages.narrow_exact(small, world, narrow.k)
        else:
            ok = narrow_exchange_exact(small, world, stages.k, narrow.k)
        exact = bool(ok.all())
        if stats is not None:
            stats.update(narrow=True, narrow_exact=exact)
        if exact:
            return _finish(stages, world, small, q, k_shard, v_shard, n_ctx_local, n_win, group,
                           list_len=narrow.k)
    elif stats is not None:
        stats.update(narrow=False, narrow_exact=None)
    cand = stages.candidates(q, k_shard, n_ctx_local)
    if gathered is None:
        gathered = torch.empty(world * cand.numel(), dtype=cand.dtype, device=cand.device)
    dist.all_gather_into_tensor(gathered, cand, group=group)
    return _finish(stages, world, gathered, q, k_shard, v_shard, n_ctx_local, n_win, group)


def _finish(stages, world, gathered, q, k_shard, v_shard, n_ctx_local, n_win, group,
            list_len=None):
    idx, scores = stages.merge(gathered, world, list_len)
    partial = stages.partial_attend(q, k_shard, v_shard, n_ctx_local, idx, scores)
    dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)
    out = stages.finalize(q, k_shard, v_shard, n_ctx_local, n_win, partial)
    return out, idx, scores


def shard_range(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous token range [lo, hi) of rank `rank` (balanced, lower ranks take the remainder)."""
    if world < 1 or not 0 <= rank < world:
        raise InputError(f"bad rank {rank} of world {world}")
    base, rem = divmod(n_total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)
