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

    def merge(self, gathered, n_shards: int):
        _lib.call("tkv_shard_merge", ctypes.byref(self.prob), ops._vp(gathered), n_shards,
                  ops._vp(self.idx), ops._vp(self.scores), self.ws.ptr, self.ws.nbytes, self._s())
        return self.idx, self.scores

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


def sharded_topk_attention(stages, q, k_shard, v_shard, n_ctx_local, n_win=None, *, group=None,
                           gathered: torch.Tensor | None = None):
    """One layer's exact top-k attention with the context sharded by token range across the
    ranks of `group`. Every rank passes its shard (rows [row_offset, row_offset + n_local) in
    rows [0, n_local) of k_shard/v_shard, window rows after them, replicated) and receives the
    full result: (out [B, Hq, 128] f32, idx [B, Hq, k] global ids, scores)."""
    world = dist.get_world_size(group)
    cand = stages.candidates(q, k_shard, n_ctx_local)
    if gathered is None:
        gathered = torch.empty(world * cand.numel(), dtype=cand.dtype, device=cand.device)
    dist.all_gather_into_tensor(gathered, cand, group=group)
    idx, scores = stages.merge(gathered, world)
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
