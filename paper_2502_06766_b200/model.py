"""Decode-step integration: a random-init Llama-3-8B-shaped decoder whose attention is the
B200 top-k decode attention (SURVEY §8f "next" #2, BASELINE cfg4).

Mirrors the reference's `decode_step` (attention.py:170-236) layer by layer — RMSNorm, Q/K/V
projections, RoPE at the token's absolute position (model.py:178-191), append of the token's
k/v to the generation window (attention.py:210), top-k attention of every head jointly with
the window (here ONE libtkv call per layer instead of the per-head loop, attention.py:213-230),
W_O, residual, RMSNorm, MLP, residual; final norm and logits. Differences to the desk-scale
reference model, as SURVEY §8f notes: GQA (32 q / 8 kv heads), and the Llama SwiGLU MLP
instead of the reference's non-gated SiLU (model.py:263). Weights and the prefilled KV cache
are random (no checkpoints offline). The dense projections are plain cuBLAS GEMMs through
torch; the whole step is captured in one CUDA graph.
"""

from __future__ import annotations

import math
import zlib
from dataclasses import dataclass

import torch

from . import _lib, ops
from .budget import LayerBudget
from .errors import ConfigError, InputError


@dataclass(frozen=True)
class LlamaShape:
    n_layers: int = 32
    d_model: int = 4096
    n_heads: int = 32
    n_kv_heads: int = 8
    head_dim: int = 128
    ffn: int = 14336
    vocab: int = 128256
    rope_theta: float = 500000.0
    eps: float = 1e-5


LLAMA3_8B = LlamaShape()


def rope_tables(shape: LlamaShape, max_pos: int, device) -> tuple[torch.Tensor, torch.Tensor]:
    inv = 1.0 / (shape.rope_theta ** (torch.arange(0, shape.head_dim, 2, device=device, dtype=torch.float64)
                                      / shape.head_dim))
    pos = torch.arange(max_pos, device=device, dtype=torch.float64)
    ang = torch.outer(pos, inv)
    return torch.cos(ang).float(), torch.sin(ang).float()


def apply_rope(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    """Rotate-half RoPE of x [..., H, 128] (f32) with cos/sin [64] for one position."""
    x1, x2 = x[..., 0::2], x[..., 1::2]
    out = torch.empty_like(x)
    out[..., 0::2] = x1 * cos - x2 * sin
    out[..., 1::2] = x1 * sin + x2 * cos
    return out


def rmsnorm(x: torch.Tensor, w: torch.Tensor, eps: float) -> torch.Tensor:
    xf = x.float()
    return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps) * w).to(torch.bfloat16)


class TopkLlamaDecoder:
    """Batch-1 decode with every layer's KV cache resident in HBM ([1, Hkv, rows, 128] bf16).

    Tensor parallel over `tp_group` (torch.distributed, one rank per GPU, NCCL): head-parallel
    Megatron-style sharding — rank r owns q heads [r·Hq/T, (r+1)·Hq/T) and their KV heads (whole
    context: the top-k attention of its heads is local, no cross-GPU selection), the matching
    columns of W_QKV and rows of W_O, 1/T of the MLP's gate/up columns and down rows. Two
    all-reduces per layer (after W_O and after the MLP down projection) sum the partial outputs;
    the residual stream, norms, embedding and LM head are replicated. With T = 1 this is the
    single-GPU model. Weights and caches are generated from per-(layer, head) seeds, so every T
    builds the same model."""

    def __init__(self, shape: LlamaShape, n_ctx: int, k: "int | LayerBudget", *, device="cuda", seed: int = 0,
                 window_capacity: int = 256, init_std: float = 0.02, retrieval_hook=None, tp_group=None,
                 tp_shard: "tuple[int, int] | None" = None):
        """k: one k for every layer, or a per-layer LayerBudget (budget.py; the reference's
        decode_step takes `budget[l]`, attention.py:202-221 — its layer count must match,
        attention.py:190-191). retrieval_hook(layer, idx): called after each layer's attention
        with the selected ids (device tensor [1, Hq_local, k_layer], -1 pads), like the
        reference's per-head hook (attention.py:229-230); eager steps only. tp_shard=(T, r)
        without a tp_group builds rank r's shard with no collectives: one rank's compute,
        for timing a tensor-parallel rank on a single GPU (tools/bench_cfg4.py --tp-shard)."""
        if shape.head_dim != ops.HEAD_DIM:
            raise InputError(f"head_dim must be {ops.HEAD_DIM}")
        if isinstance(k, LayerBudget):
            if k.n_layers != shape.n_layers:
                raise ConfigError(f"budget has {k.n_layers} layers, model has {shape.n_layers}")
            self.budget = k
        else:
            self.budget = LayerBudget(tuple([int(k)] * shape.n_layers))
        self.shape, self.n, self.k = shape, n_ctx, self.budget.k_max
        self.retrieval_hook = retrieval_hook
        self.device = torch.device(device)
        self.tp_group = tp_group
        if tp_group is not None:
            import torch.distributed as dist

            self.tp, self.tp_rank = dist.get_world_size(tp_group), dist.get_rank(tp_group)
        else:
            self.tp, self.tp_rank = tp_shard if tp_shard is not None else (1, 0)
        dev, s, T, r = self.device, shape, self.tp, self.tp_rank
        if s.n_kv_heads % T or s.n_heads % T or s.ffn % T:
            raise ConfigError(f"tensor parallel degree {T} must divide the kv heads, heads and ffn")
        self.hq, self.hkv, self.ffn = s.n_heads // T, s.n_kv_heads // T, s.ffn // T
        hd, bf = s.head_dim, torch.bfloat16

        def gen(*tags):  # process-independent seed per tag (str hash() is salted per process)
            g = torch.Generator(device=dev)
            g.manual_seed((seed * 0x9E3779B1 + zlib.crc32(repr(tags).encode())) & 0x7FFFFFFFFFFFFFFF)
            return g

        def w(g, *dims):
            return (torch.randn(dims, generator=g, device=dev) * init_std).to(bf)

        self.embed = w(gen("embed"), s.vocab, s.d_model)
        self.lm_head = w(gen("lm_head"), s.d_model, s.vocab)
        self.norm_f = torch.ones(s.d_model, device=dev)
        q_cols = slice(r * self.hq * hd, (r + 1) * self.hq * hd)
        k_cols = slice(s.n_heads * hd + r * self.hkv * hd, s.n_heads * hd + (r + 1) * self.hkv * hd)
        v_cols = slice((s.n_heads + s.n_kv_heads) * hd + r * self.hkv * hd,
                       (s.n_heads + s.n_kv_heads) * hd + (r + 1) * self.hkv * hd)
        f_cols = slice(r * self.ffn, (r + 1) * self.ffn)
        self.layers = []
        rows = n_ctx + window_capacity
        self.rows = rows
        for layer in range(s.n_layers):
            g = gen("layer", layer)
            wqkv = w(g, s.d_model, (s.n_heads + 2 * s.n_kv_heads) * hd)
            wo = w(g, s.n_heads * hd, s.d_model)
            wgu = w(g, s.d_model, 2 * s.ffn)
            wd = w(g, s.ffn, s.d_model)
            lw = dict(wqkv=torch.cat([wqkv[:, q_cols], wqkv[:, k_cols], wqkv[:, v_cols]], dim=1).contiguous(),
                      wo=wo[q_cols].contiguous(),
                      wgu=torch.cat([wgu[:, f_cols], wgu[:, s.ffn + f_cols.start: s.ffn + f_cols.stop]], 1).contiguous(),
                      wd=wd[f_cols].contiguous(),
                      n1=torch.ones(s.d_model, device=dev), n2=torch.ones(s.d_model, device=dev))
            del wqkv, wo, wgu, wd
            # prefilled context of this rank's kv heads: random post-RoPE keys / values per head
            K = torch.empty((1, self.hkv, rows, hd), dtype=bf, device=dev)
            V = torch.empty_like(K)
            for j in range(self.hkv):
                gk = gen("kv", layer, r * self.hkv + j)
                for r0 in range(0, rows, 1 << 16):
                    r1 = min(rows, r0 + (1 << 16))
                    K[0, j, r0:r1] = torch.randn((r1 - r0, hd), generator=gk, device=dev).to(bf)
                    V[0, j, r0:r1] = torch.randn((r1 - r0, hd), generator=gk, device=dev).to(bf)
            lw["K"], lw["V"] = K, V
            self.layers.append(lw)
        self.n_ctx = torch.tensor([n_ctx], dtype=torch.int32, device=dev)
        self.n_win = torch.zeros(1, dtype=torch.int32, device=dev)
        self.pos = torch.zeros(1, dtype=torch.int64, device=dev)  # absolute position of the token
        self.cos, self.sin = rope_tables(s, rows, dev)
        # one workspace sized for the largest k serves every layer: its control words sit at
        # k-independent offsets (api.cu make_layout)
        self.ws = ops.Workspace(ops.make_problem(1, self.hq, self.hkv, rows, n_ctx, self.k), dev) \
            if dev.type == "cuda" else None
        self.token = torch.zeros(1, dtype=torch.int64, device=dev)
        self.next_token = torch.zeros(1, dtype=torch.int64, device=dev)
        self.logits = torch.zeros((1, s.vocab), dtype=torch.float32, device=dev)  # last step's
        self.attn_out = torch.empty((1, self.hq, hd), dtype=torch.float32, device=dev)
        self._sel = {kl: (torch.empty((1, self.hq, kl), dtype=torch.int32, device=dev),
                          torch.empty((1, self.hq, kl), dtype=torch.float32, device=dev))
                     for kl in sorted(set(self.budget.k_per_layer))}
        self.idx, self.scores = self._sel[self.k]
        self.graph = None
        self.pos.fill_(n_ctx)
        self.win_used = 0  # host mirror of n_win: capacity is checked before a step is enqueued
        if dev.type == "cuda":  # persistent activations of the fused CUDA step (_step_body_cuda)
            nqkv = (self.hq + 2 * self.hkv) * hd
            self._x = torch.empty((1, s.d_model), dtype=bf, device=dev)  # residual stream
            self._h = torch.empty((1, s.d_model), dtype=bf, device=dev)
            self._qkv = torch.empty((1, nqkv), dtype=bf, device=dev)
            self._q = torch.empty((1, self.hq, hd), dtype=bf, device=dev)
            self._a = torch.empty((1, self.hq * hd), dtype=bf, device=dev)
            self._o = torch.empty((1, s.d_model), dtype=bf, device=dev)
            self._gu = torch.empty((1, 2 * self.ffn), dtype=bf, device=dev)
            self._act = torch.empty((1, self.ffn), dtype=bf, device=dev)
            self._d = torch.empty((1, s.d_model), dtype=bf, device=dev)
            self._lg = torch.empty((1, s.vocab), dtype=bf, device=dev)
            self._am = torch.zeros(2, dtype=torch.int64, device=dev)  # argmax scratch (self-resetting)
            self._n_win_next = torch.empty_like(self.n_win)

    def _attend(self, layer: int, lw: dict, q: torch.Tensor, kk, v) -> torch.Tensor:
        """Window append of this token's k/v (attention.py:210; n_win advances once per step,
        after the last layer; kk = v = None: already appended by the fused RoPE kernel) + top-k
        attention of this rank's heads (libtkv, one call)."""
        if kk is not None:
            ops.kv_append(lw["K"], lw["V"], kk, v, self.n_win, base=self.n_ctx, advance=False)
        kl = self.budget[layer]
        idx, scores = self._sel[kl]
        ops.topk_decode_attention(q, lw["K"], lw["V"], self.n_ctx, kl, n_win=self._n_win_next,
                                  out=self.attn_out, idx=idx, scores=scores, workspace=self.ws, max_ctx=self.n)
        if self.retrieval_hook is not None:
            self.retrieval_hook(layer, idx)
        return self.attn_out

    def _reduce(self, part: torch.Tensor) -> torch.Tensor:
        """Sum of the ranks' partial projections (fp32 on the wire), back to bf16."""
        if self.tp == 1:
            return part
        t = part.float()
        if self.tp_group is not None:  # (tp_shard timing runs: the same casts, no collective)
            import torch.distributed as dist

            dist.all_reduce(t, group=self.tp_group)
        return t.to(torch.bfloat16)

    def _layer(self, x: torch.Tensor, lw: dict, layer: int = 0) -> torch.Tensor:
        s = self.shape
        h = rmsnorm(x, lw["n1"], s.eps)
        qkv = (h @ lw["wqkv"]).float()
        nq, nk = self.hq * s.head_dim, self.hkv * s.head_dim
        q = qkv[:, :nq].view(1, self.hq, s.head_dim)
        kk = qkv[:, nq:nq + nk].view(1, self.hkv, s.head_dim)
        v = qkv[:, nq + nk:].view(1, self.hkv, s.head_dim)
        cos = self.cos.index_select(0, self.pos)
        sin = self.sin.index_select(0, self.pos)
        q = apply_rope(q, cos, sin).to(torch.bfloat16).contiguous()
        kk = apply_rope(kk, cos, sin).to(torch.bfloat16).contiguous()
        v = v.to(torch.bfloat16).contiguous()
        attn = self._attend(layer, lw, q, kk, v)
        x = x + self._reduce(attn.reshape(1, -1).to(torch.bfloat16) @ lw["wo"])
        h2 = rmsnorm(x, lw["n2"], s.eps)
        gu = h2 @ lw["wgu"]
        gate, up = gu[:, :self.ffn], gu[:, self.ffn:]
        x = x + self._reduce((torch.nn.functional.silu(gate.float()) * up.float()).to(torch.bfloat16) @ lw["wd"])
        return x

    def _step_body(self) -> None:
        if self.device.type == "cuda":
            self._step_body_cuda()
            return
        x = self.embed.index_select(0, self.token)
        self._n_win_next = self.n_win + 1  # the token attends to itself (attention.py:210)
        for layer, lw in enumerate(self.layers):
            x = self._layer(x, lw, layer)
        logits = rmsnorm(x, self.norm_f, self.shape.eps) @ self.lm_head
        self.logits.copy_(logits)
        self.next_token.copy_(logits.argmax(-1))
        self.n_win.add_(1)
        self.pos.add_(1)

    def _step_body_cuda(self) -> None:
        """One step on the device, ~14 launches per layer: fused residual-add + RMSNorm, the QKV
        GEMV, fused RoPE + window append, top-k attention (libtkv), O projection (+ the TP
        all-reduce), fused residual-add + RMSNorm, gate/up GEMV, fused SiLU·up, down GEMV (+ the
        all-reduce); then the final norm, LM head and a fused logits copy + argmax
        (csrc/model_glue.cu). Same numerics as the eager path (bf16 storage, fp32 math)."""
        s, dev = self.shape, self.device
        st = ops._stream(dev)
        vp = ops._vp
        torch.index_select(self.embed, 0, self.token, out=self._x)
        torch.add(self.n_win, 1, out=self._n_win_next)  # the token attends to itself (attention.py:210)
        delta = None
        for layer, lw in enumerate(self.layers):
            _lib.call("tkv_model_add_rmsnorm", vp(self._x), vp(delta), vp(lw["n1"]), s.eps, vp(self._h),
                      s.d_model, st)
            torch.mm(self._h, lw["wqkv"], out=self._qkv)
            _lib.call("tkv_model_qkv_rope_append", vp(self._qkv), vp(self.cos), vp(self.sin), vp(self.pos),
                      vp(self._q), vp(lw["K"]), vp(lw["V"]), vp(self.n_ctx), vp(self.n_win), self.rows, self.hq,
                      self.hkv, s.head_dim, st)
            attn = self._attend(layer, lw, self._q, None, None)
            self._a.copy_(attn.view(1, -1))
            torch.mm(self._a, lw["wo"], out=self._o)
            delta = self._reduce(self._o)
            _lib.call("tkv_model_add_rmsnorm", vp(self._x), vp(delta), vp(lw["n2"]), s.eps, vp(self._h),
                      s.d_model, st)
            torch.mm(self._h, lw["wgu"], out=self._gu)
            _lib.call("tkv_model_silu_mul", vp(self._gu), vp(self._act), self.ffn, st)
            torch.mm(self._act, lw["wd"], out=self._d)
            delta = self._reduce(self._d)
        _lib.call("tkv_model_add_rmsnorm", vp(self._x), vp(delta), vp(self.norm_f), s.eps, vp(self._h),
                  s.d_model, st)
        torch.mm(self._h, self.lm_head, out=self._lg)
        _lib.call("tkv_model_logits_argmax", vp(self._lg), s.vocab, vp(self.logits), vp(self.next_token),
                  vp(self._am), st)
        self.n_win.add_(1)
        self.pos.add_(1)

    def step(self, token: int | None = None) -> torch.Tensor:
        """One decode step for every layer; returns the greedy next token (device tensor)."""
        if self.n + self.win_used + 1 > self.rows:
            # GenWindow.append raises on a full window (attention.py:96-97)
            raise InputError("generation window capacity exceeded")
        self.win_used += 1
        if token is not None:
            self.token.fill_(token)
        if self.graph is not None:
            self.graph.replay()
        else:
            self._step_body()
        self.token.copy_(self.next_token)
        return self.next_token

    def capture(self) -> None:
        """Capture one step into a CUDA graph (window and position advance on device)."""
        if self.retrieval_hook is not None:
            raise ConfigError("retrieval_hook runs host code per layer: eager steps only, no graph capture")
        torch.cuda.synchronize(self.device)
        saved = (self.n_win.clone(), self.pos.clone(), self.token.clone())
        self._step_body()  # warm-up: lazy libtkv / cuBLAS setup outside the capture
        self.n_win.copy_(saved[0])
        self.pos.copy_(saved[1])
        self.token.copy_(saved[2])
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._step_body()
        self.graph = g

    @staticmethod
    def memory_bytes(shape: LlamaShape, n_ctx: int, window_capacity: int = 256, tp: int = 1) -> int:
        """HBM of one rank at tensor-parallel degree tp (layer weights and KV split tp ways,
        embedding / LM head replicated)."""
        s = shape
        per_layer_w = (s.d_model * (s.n_heads + 2 * s.n_kv_heads) * s.head_dim + s.n_heads * s.head_dim * s.d_model
                       + 3 * s.d_model * s.ffn) * 2
        kv = 2 * s.n_kv_heads * (n_ctx + window_capacity) * s.head_dim * 2
        return s.n_layers * (per_layer_w + kv) // tp + 2 * s.vocab * s.d_model * 2


def dense_reference_step(dec: TopkLlamaDecoder, token: int) -> torch.Tensor:
    """fp32 reference of the same step with DENSE attention over context + window (k = N is the
    exact-equivalence case). Test helper: does not touch the decoder's state."""
    s = dec.shape
    x = dec.embed[token].float()[None]
    pos = dec.pos.clone()
    nwin = int(dec.n_win.item())
    def reduce(t):  # tensor-parallel sum of the ranks' partial projections (fp32)
        if dec.tp_group is not None:
            import torch.distributed as dist

            dist.all_reduce(t, group=dec.tp_group)
        return t

    hq, hkv = dec.hq, dec.hkv
    for lw in dec.layers:
        h = rmsnorm(x, lw["n1"], s.eps).float()
        qkv = h @ lw["wqkv"].float()
        nq, nk = hq * s.head_dim, hkv * s.head_dim
        q = qkv[:, :nq].view(1, hq, s.head_dim)
        kk = qkv[:, nq:nq + nk].view(1, hkv, s.head_dim)
        v = qkv[:, nq + nk:].view(1, hkv, s.head_dim)
        cos, sin = dec.cos.index_select(0, pos), dec.sin.index_select(0, pos)
        q = apply_rope(q, cos, sin).to(torch.bfloat16).float()
        kk = apply_rope(kk, cos, sin).to(torch.bfloat16).float()
        v = v.to(torch.bfloat16).float()
        rows = dec.n + nwin
        K = torch.cat([lw["K"][0, :, :rows].float(), kk.transpose(0, 1)], dim=1)  # [Hkv, rows+1, d]
        V = torch.cat([lw["V"][0, :, :rows].float(), v.transpose(0, 1)], dim=1)
        G = hq // hkv
        Kq = K.repeat_interleave(G, 0)
        Vq = V.repeat_interleave(G, 0)
        sc = torch.einsum("hd,hnd->hn", q[0], Kq) / math.sqrt(s.head_dim)
        attn = torch.einsum("hn,hnd->hd", torch.softmax(sc, -1), Vq)
        x = x + reduce(attn.reshape(1, -1).to(torch.bfloat16).float() @ lw["wo"].float())
        h2 = rmsnorm(x, lw["n2"], s.eps).float()
        gu = h2 @ lw["wgu"].float()
        x = x + reduce((torch.nn.functional.silu(gu[:, :dec.ffn]) * gu[:, dec.ffn:]) @ lw["wd"].float())
    return rmsnorm(x, dec.norm_f, s.eps).float() @ dec.lm_head.float()
