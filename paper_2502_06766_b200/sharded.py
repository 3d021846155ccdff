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
outputs up to fp32 summation order). `sharded_topk_attention` runs the exchange through
torch.distributed collectives (NCCL over NVLink; gloo in the CPU tests), with the compute stages
pluggable so the protocol can be tested on CPU with the oracle's stages (tests only).

`DeviceShardedStep` is the device-driven form: every rank publishes its narrow AND full lists in
memory its peers read directly (torch symmetric memory over NVLink — `SymmetricExchange` — or,
in the one-GPU emulation, `LocalExchange`), the merge kernel picks narrow or full per head on the
device (tkv_shard_exchange_merge), and the partials are summed by the finishing kernel reading
every rank's buffer (tkv_shard_combine). No host round trip: the step is CUDA-graph capturable.
The product default is `CudaStages` (libtkv), which fails loudly without the native library.
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

    def candidates2(self, q, k_cache, n_ctx, narrow_k: int, narrow_out, full_out, bounds_out):
        """One scan: the exact local top-k list, the narrow list (its entries above a bound t2,
        fewer than narrow_k) and the bounds {t2, local k-th, max} into the given buffers."""
        _lib.call("tkv_shard_candidates2", ctypes.byref(self.prob), narrow_k, ops._vp(q), ops._vp(k_cache),
                  ops._vp(n_ctx), ops._vp(narrow_out), ops._vp(full_out), ops._vp(bounds_out), self.ws.ptr,
                  self.ws.nbytes, self._s())

    def exchange_merge(self, narrow_ptrs, full_ptrs, bound_ptrs, n_shards: int, narrow_k: int, used_full=None):
        """Exact global top-k over every rank's published lists (device arrays of pointers)."""
        _lib.call("tkv_shard_exchange_merge", ctypes.byref(self.prob), ops._vp(narrow_ptrs), ops._vp(full_ptrs),
                  ops._vp(bound_ptrs), n_shards, narrow_k, ops._vp(self.idx), ops._vp(self.scores),
                  ops._vp(used_full), self.ws.ptr, self.ws.nbytes, self._s())
        return self.idx, self.scores

    def partial_into(self, q, k_cache, v_cache, n_ctx, idx, scores, partial_out):
        _lib.call("tkv_shard_partial", ctypes.byref(self.prob), ops._vp(q), ops._vp(k_cache),
                  ops._vp(v_cache), ops._vp(n_ctx), ops._vp(idx), ops._vp(scores),
                  ops._vp(partial_out), self.ws.ptr, self.ws.nbytes, self._s())

    def combine(self, partial_ptrs, n_shards: int, q, k_cache, v_cache, n_ctx, n_win):
        """Sum every rank's partial (device array of pointers) + window + normalisation."""
        _lib.call("tkv_shard_combine", ctypes.byref(self.prob), ops._vp(partial_ptrs), n_shards, ops._vp(q),
                  ops._vp(k_cache), ops._vp(v_cache), ops._vp(n_ctx), ops._vp(n_win), ops._vp(self.out),
                  self.ws.ptr, self.ws.nbytes, self._s())
        return self.out

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


# ---------------------------------------------------------------------- device-driven exchange
class _PublishLayout:
    """Byte layout of one rank's publish buffer: narrow list | full list | bounds | partial."""

    def __init__(self, B: int, Hq: int, k: int, narrow_k: int):
        bh = B * Hq
        self.narrow = (0, bh * narrow_k)                      # int64 elements
        self.full = (bh * narrow_k, bh * k)
        self.bound = (bh * narrow_k + bh * k, bh * 3)
        self.partial_off_bytes = (bh * narrow_k + bh * k + bh * 3) * 8
        self.partial_len = bh * (ops.HEAD_DIM + 1)             # float32 elements
        self.nbytes = self.partial_off_bytes + self.partial_len * 4


class LocalExchange:
    """The exchange emulated on one GPU: all `world` ranks' publish buffers live in this process
    (tests, tools/narrow_stage.py). Barriers are no-ops: the emulated ranks run their stages one
    after another in stream order, so no kernel ever waits on another."""

    def __init__(self, world: int, B: int, Hq: int, k: int, narrow_k: int, device):
        self.world, self.layout = world, _PublishLayout(B, Hq, k, narrow_k)
        self.device = torch.device(device)
        self.bufs = [torch.zeros(self.layout.nbytes, dtype=torch.uint8, device=self.device) for _ in range(world)]
        self._ptrs = _pointer_arrays([b.data_ptr() for b in self.bufs], self.layout, self.device)

    def views(self, rank: int):
        return _views(self.bufs[rank], self.layout)

    def pointers(self):
        return self._ptrs

    def barrier(self):
        pass


class SymmetricExchange:
    """torch symmetric memory, one rank per GPU: every rank allocates its publish buffer from the
    symmetric pool and rendezvous with the group, so each rank's kernels read the peers' buffers
    directly over NVLink through device pointers; barriers run on the symmetric signal pads
    (stream-ordered kernels, CUDA-graph capturable). Needs an NCCL process group on CUDA."""

    def __init__(self, B: int, Hq: int, k: int, narrow_k: int, device, group=None):
        import torch.distributed._symmetric_memory as symm_mem

        self.layout = _PublishLayout(B, Hq, k, narrow_k)
        self.device = torch.device(device)
        grp = group if group is not None else dist.group.WORLD
        self.world = dist.get_world_size(grp)
        self.rank = dist.get_rank(grp)
        self.buf = symm_mem.empty(self.layout.nbytes, dtype=torch.uint8, device=self.device)
        self.handle = symm_mem.rendezvous(self.buf, grp)
        bases = [int(p) + int(getattr(self.handle, "offset", 0)) for p in self.handle.buffer_ptrs]
        self._ptrs = _pointer_arrays(bases, self.layout, self.device)

    def views(self, rank: int):
        if rank != self.rank:
            raise InputError("a rank writes only its own publish buffer")
        return _views(self.buf, self.layout)

    def pointers(self):
        return self._ptrs

    def barrier(self):
        self.handle.barrier(channel=0)


def _views(buf: torch.Tensor, layout: _PublishLayout):
    i64 = buf[: layout.partial_off_bytes].view(torch.int64)
    narrow = i64[layout.narrow[0]: layout.narrow[0] + layout.narrow[1]]
    full = i64[layout.full[0]: layout.full[0] + layout.full[1]]
    bound = i64[layout.bound[0]: layout.bound[0] + layout.bound[1]]
    partial = buf[layout.partial_off_bytes: layout.nbytes].view(torch.float32)
    return narrow, full, bound, partial


def _pointer_arrays(bases, layout: _PublishLayout, device):
    """Device int64 arrays of every rank's narrow list, full list, bounds and partial addresses."""
    nar = [b + layout.narrow[0] * 8 for b in bases]
    full = [b + layout.full[0] * 8 for b in bases]
    bound = [b + layout.bound[0] * 8 for b in bases]
    part = [b + layout.partial_off_bytes for b in bases]
    return tuple(torch.tensor(x, dtype=torch.int64, device=device) for x in (nar, full, bound, part))


class DeviceShardedStep:
    """One layer step of the token-range sharded attention for rank `rank`, device-driven:

      candidates2  → this rank's narrow (top-k') and full (top-k) lists into its publish buffer
      barrier      (every rank's lists published)
      merge        exact global top-k, narrow or full per head chosen on the device
      partial      this rank's (l, o) over the selected rows it owns → its publish buffer
      barrier      (every partial published)
      combine      sum of all partials (read from the peers) + window + normalisation
      barrier      (peers done reading before the next step overwrites the buffers)

    Returns (out, idx, scores) — identical on every rank; `used_full` [B*Hq] int32 records the
    heads merged from the full lists."""

    def __init__(self, stages: "CudaStages", exchange, rank: int, narrow_k: int):
        self.stages, self.exch, self.rank, self.narrow_k = stages, exchange, rank, narrow_k
        self.used_full = torch.zeros(stages.B * stages.Hq, dtype=torch.int32, device=stages.device)

    def publish_candidates(self, q, k_shard, n_ctx):
        narrow, full, bound, _ = self.exch.views(self.rank)
        self.stages.candidates2(q, k_shard, n_ctx, self.narrow_k, narrow, full, bound)

    def merge_and_partial(self, q, k_shard, v_shard, n_ctx):
        nar_p, full_p, bound_p, _ = self.exch.pointers()
        idx, sc = self.stages.exchange_merge(nar_p, full_p, bound_p, self.exch.world, self.narrow_k,
                                             self.used_full)
        partial = self.exch.views(self.rank)[3]
        self.stages.partial_into(q, k_shard, v_shard, n_ctx, idx, sc, partial)
        return idx, sc

    def combine(self, q, k_shard, v_shard, n_ctx, n_win):
        part_p = self.exch.pointers()[3]
        return self.stages.combine(part_p, self.exch.world, q, k_shard, v_shard, n_ctx, n_win)

    def __call__(self, q, k_shard, v_shard, n_ctx, n_win=None):
        self.publish_candidates(q, k_shard, n_ctx)
        self.exch.barrier()
        idx, sc = self.merge_and_partial(q, k_shard, v_shard, n_ctx)
        self.exch.barrier()
        out = self.combine(q, k_shard, v_shard, n_ctx, n_win)
        self.exch.barrier()
        return out, idx, sc
