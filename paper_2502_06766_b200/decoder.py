"""Decode-loop session over one layer's device-resident KV cache.

`TopkDecoder` is the user-facing object for the paper's decode step on B200: it owns the
layer's bf16 K/V cache in HBM (context rows [0, n_ctx) followed by the generation window,
the reference's GenWindow, attention.py:76-104), the libtkv workspace, and pinned host
staging buffers. `step(q, k_new, v_new)` mirrors one layer of `decode_step`
(attention.py:203-230): append the token's k/v to the window (attention.py:210), then top-k
attention for every q head. With host tensors it is the end-to-end path: q/k/v go into pinned
staging buffers that the call reads itself (TKV_F_HOST_Q: one small kernel stages them on the
device) and the output is written straight into pinned host memory; the whole device part of
a step (staging, KV append, the attention kernels) is captured once into a CUDA graph and
replayed, so a step costs one graph launch plus the host-side copies into the staging buffers.
"""

from __future__ import annotations

import torch

from . import ops
from .errors import InputError, ShapeError


class TopkDecoder:
    def __init__(self, k_cache: torch.Tensor, v_cache: torch.Tensor, n_ctx, k: int, *,
                 n_win=0, scale: float | None = None, combine: str = "joint",
                 pinned_prefix: int = 0, sorted: bool = False, max_ctx: int | None = None,
                 use_graph: bool = True, parts: int = 0, list_gather: bool = False,
                 head: bool | None = None, fold_append: bool = True):
        if k < 1:
            raise InputError("k must be >= 1")
        ops._check_cuda_bf16("k_cache", k_cache, 4)
        ops._check_cuda_bf16("v_cache", v_cache, 4)
        if v_cache.shape != k_cache.shape:
            raise ShapeError("v_cache shape must equal k_cache shape")
        self.k_cache, self.v_cache = k_cache, v_cache
        self.B, self.Hkv, self.rows, d = k_cache.shape
        self.device = k_cache.device
        self.n_ctx = ops._as_counts("n_ctx", n_ctx, self.B, self.device)
        self.n_win = ops._as_counts("n_win", n_win, self.B, self.device)
        # host mirrors of the counters (one read at construction): the window's capacity is
        # checked before a step is enqueued, as GenWindow.append does (attention.py:96-97)
        self._ctx_host = [int(x) for x in self.n_ctx.tolist()]
        self._win_host = [int(x) for x in self.n_win.tolist()]
        self.max_ctx = int(max_ctx if max_ctx is not None else self.rows)
        self.k = k
        self.kw = dict(scale=scale, combine=combine, pinned_prefix=pinned_prefix, sorted=sorted,
                       max_ctx=self.max_ctx, parts=parts, list_gather=list_gather, head=head)
        ops.combine_code(combine)
        self.use_graph = use_graph
        self.fold_append = fold_append
        self.Hq = None
        self._bufs = None
        self.ws = None
        self._graphs: dict[tuple, torch.cuda.CUDAGraph] = {}
        self._last_direct = None  # (q, k_new, v_new, data pointers) of the last validated direct step

    def _ensure(self, Hq: int) -> None:
        if self.Hq == Hq:
            return
        if Hq % self.Hkv:
            raise ShapeError(f"Hq={Hq} is not a multiple of Hkv={self.Hkv}")
        self.Hq = Hq
        dev = self.device
        prob = ops.make_problem(self.B, Hq, self.Hkv, self.rows, self.max_ctx, self.k,
                                pinned_prefix=self.kw["pinned_prefix"], scale=self.kw["scale"],
                                combine=self.kw["combine"], sorted=self.kw["sorted"],
                                parts=self.kw["parts"], list_gather=self.kw["list_gather"],
                                head=self.kw["head"])
        self.ws = ops.Workspace(prob, dev)
        D = ops.HEAD_DIM
        bf, f32, i32 = torch.bfloat16, torch.float32, torch.int32
        # q, k_new and v_new share one staging buffer on each side, so a step moves its inputs
        # with a single host→device copy
        nq, nkv = self.B * Hq * D, self.B * self.Hkv * D
        in_d = torch.empty(nq + 2 * nkv, dtype=bf, device=dev)
        in_h = torch.empty(nq + 2 * nkv, dtype=bf, pin_memory=True)

        def views(buf):
            return (buf[:nq].view(self.B, Hq, D), buf[nq:nq + nkv].view(self.B, self.Hkv, D),
                    buf[nq + nkv:].view(self.B, self.Hkv, D))

        q_d, k_d, v_d = views(in_d)
        q_h, k_h, v_h = views(in_h)
        self._bufs = dict(
            in_d=in_d, in_h=in_h, nq=nq,
            q=q_d, k_new=k_d, v_new=v_d,
            out=torch.empty((self.B, Hq, D), dtype=f32, device=dev),
            idx=torch.empty((self.B, Hq, self.k), dtype=i32, device=dev),
            scores=torch.empty((self.B, Hq, self.k), dtype=f32, device=dev),
            q_h=q_h, k_h=k_h, v_h=v_h,
            out_h=torch.empty((self.B, Hq, D), dtype=f32, pin_memory=True),
            idx_h=torch.empty((self.B, Hq, self.k), dtype=i32, pin_memory=True),
        )
        self._graphs.clear()
        self._last_direct = None

    # ------------------------------------------------------------------ device-side pieces
    def _reserve_row(self) -> None:
        if any(c + w + 1 > self.rows for c, w in zip(self._ctx_host, self._win_host)):
            raise InputError("generation window capacity exceeded")
        self._win_host = [w + 1 for w in self._win_host]

    def append(self, k_new: torch.Tensor, v_new: torch.Tensor) -> None:
        """GenWindow.append (attention.py:94-100) on device: rows n_ctx + n_win, n_win += 1."""
        if self._bufs is None:
            raise InputError("call step() (or attend()) once before append-only use")
        self._reserve_row()
        kd, vd = self._bufs["k_new"], self._bufs["v_new"]
        kd.copy_(k_new, non_blocking=True)
        vd.copy_(v_new, non_blocking=True)
        ops.kv_append(self.k_cache, self.v_cache, kd, vd, self.n_win, base=self.n_ctx, advance=True)

    def attend(self, q: torch.Tensor):
        """Top-k attention of q [B, Hq, 128] over context + window. Device tensors out."""
        self._ensure(q.shape[1])
        b = self._bufs
        qd = q if (q.is_cuda and q.dtype == torch.bfloat16 and q.is_contiguous()) else b["q"].copy_(q, non_blocking=True)
        ops.topk_decode_attention(qd, self.k_cache, self.v_cache, self.n_ctx, self.k, n_win=self.n_win,
                                  out=b["out"], idx=b["idx"], scores=b["scores"], workspace=self.ws,
                                  **self.kw)
        return b["out"], b["idx"], b["scores"]

    def _host_step_body(self, with_kv: bool, with_idx: bool, src=None) -> None:
        """Everything a host-I/O step enqueues, reading/writing the pinned staging buffers (or,
        with src = (q, k_new, v_new), the caller's own pinned tensors)."""
        b = self._bufs
        q_h, k_h, v_h = src if src is not None else (b["q_h"], b["k_h"], b["v_h"])
        # inputs: read straight from the pinned host staging buffer by the call itself
        # (TKV_F_HOST_Q: one small kernel stages q, the window append reads k/v over PCIe) —
        # no H2D copy node; only the unfolded append path copies q | k_new | v_new first.
        # The head-finishing CTAs write the output straight into the pinned host buffer (mapped
        # memory, 512 B per head): no device->host copy node on the step's critical path
        if with_kv and not self.fold_append:
            b["in_d"].copy_(b["in_h"], non_blocking=True)
            ops.kv_append(self.k_cache, self.v_cache, b["k_new"], b["v_new"], self.n_win,
                          base=self.n_ctx, advance=True)
            q_in = b["q"]
        else:
            q_in = q_h
        # the selected ids likewise go straight into pinned host memory, written by the gather
        # as it finds them (coalesced 128-byte PCIe writes overlapping the gather) instead of a
        # device->host copy of the whole list after it — unless the ids are sorted afterwards
        # (the sort kernel would then work over PCIe)
        direct_idx = with_idx and not self.kw["sorted"]
        idx_buf = b["idx_h"] if direct_idx else b["idx"]
        if with_kv and self.fold_append:  # window append folded into the attention call
            ops.topk_decode_step(q_in, k_h, v_h, self.k_cache, self.v_cache, self.n_ctx,
                                 self.n_win, self.k, out=b["out_h"], idx=idx_buf, scores=b["scores"],
                                 workspace=self.ws, **self.kw)
        else:
            ops.topk_decode_attention(q_in, self.k_cache, self.v_cache, self.n_ctx, self.k,
                                      n_win=self.n_win, out=b["out_h"], idx=idx_buf, scores=b["scores"],
                                      workspace=self.ws, **self.kw)
        if with_idx and not direct_idx:
            b["idx_h"].copy_(b["idx"], non_blocking=True)

    # ------------------------------------------------------------------ user API
    def step(self, q: torch.Tensor, k_new: torch.Tensor | None = None, v_new: torch.Tensor | None = None,
             return_idx: bool = True):
        """One decode step for this layer. Host inputs → host outputs (out f32[, idx int32]);
        device inputs → device outputs (out, idx)."""
        self._ensure(q.shape[1])
        if q.is_cuda:
            if k_new is not None:
                self.append(k_new, v_new)
            out, idx, _ = self.attend(q)
            return (out, idx) if return_idx else out
        b = self._bufs
        with_kv = k_new is not None
        if with_kv:
            self._reserve_row()
        Hq = q.shape[1]
        # pinned bf16 inputs of the right shape are read in place by the call (no host copy);
        # the step's graph is then keyed by their addresses (a few cached). The same live tensor
        # objects as the previous step skip the checks (Tensor.is_pinned() queries the driver: a
        # few µs per tensor on the end-to-end path)
        last = self._last_direct
        if (last is not None and q is last[0] and k_new is last[1] and v_new is last[2]
                and last[3] == (q.data_ptr(), k_new.data_ptr() if with_kv else 0,
                                v_new.data_ptr() if with_kv else 0) and last[4] == q.shape):
            direct = True
        else:
            direct = ((self.fold_append or not with_kv) and self._pinned_ok(q, (self.B, Hq, ops.HEAD_DIM))
                      and (not with_kv or (self._pinned_ok(k_new, (self.B, self.Hkv, ops.HEAD_DIM))
                                           and self._pinned_ok(v_new, (self.B, self.Hkv, ops.HEAD_DIM)))))
            self._last_direct = (q, k_new, v_new, (q.data_ptr(), k_new.data_ptr() if with_kv else 0,
                                                   v_new.data_ptr() if with_kv else 0), q.shape) if direct else None
        if direct:
            src = (q, k_new, v_new)
            key = (with_kv, return_idx, q.data_ptr(), k_new.data_ptr() if with_kv else 0,
                   v_new.data_ptr() if with_kv else 0)
        else:
            b["q_h"].copy_(q)
            if with_kv:
                b["k_h"].copy_(k_new)
                b["v_h"].copy_(v_new)
            src, key = None, (with_kv, return_idx)
        if self.use_graph:
            g = self._graphs.get(key)
            if g is None:
                g = self._capture(key, src)
            g.replay()
        else:
            self._host_step_body(with_kv, return_idx, src)
        torch.cuda.current_stream(self.device).synchronize()
        return (b["out_h"], b["idx_h"]) if return_idx else b["out_h"]

    @staticmethod
    def _pinned_ok(t, shape) -> bool:
        return (isinstance(t, torch.Tensor) and not t.is_cuda and t.is_pinned() and t.dtype == torch.bfloat16
                and t.is_contiguous() and tuple(t.shape) == shape)

    def _capture(self, key, src=None) -> torch.cuda.CUDAGraph:
        with_kv, with_idx = key[0], key[1]
        if src is not None:  # graphs bound to caller tensors: keep only the most recent few
            direct = [kk for kk in self._graphs if len(kk) > 2]
            for kk in direct[:max(0, len(direct) - 7)]:
                del self._graphs[kk]
        stream = torch.cuda.current_stream(self.device)
        # capture on a side stream; one eager run first so every lazy attribute/occupancy
        # query inside libtkv has happened before capture. The eager run's KV append is undone
        # by rewinding n_win, so the capture does not double-append.
        saved = self.n_win.clone()
        self._host_step_body(with_kv, with_idx, src)
        self.n_win.copy_(saved)
        stream.synchronize()
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(self.device)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                self._host_step_body(with_kv, with_idx, src)
        stream.wait_stream(side)
        self._graphs[key] = g
        return g
