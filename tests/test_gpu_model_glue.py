"""GPU: the fused decode-step kernels of csrc/model_glue.cu (tkv_model_*, the non-attention work
of TopkLlamaDecoder's CUDA step) against the plain PyTorch fp32 restatement of the same ops
(model.py rmsnorm / apply_rope / SwiGLU / argmax), through the C ABI."""

from __future__ import annotations

import pytest
import torch

pytestmark = pytest.mark.gpu


def _call(name, *args):
    from paper_2502_06766_b200 import _lib

    _lib.call(name, *args)


def _vp(t):
    from paper_2502_06766_b200.ops import _vp

    return _vp(t)


def _st(dev):
    from paper_2502_06766_b200.ops import _stream

    return _stream(dev)


@pytest.mark.parametrize("d,with_delta", [(4096, True), (4096, False), (256, True), (1000, True)])
def test_add_rmsnorm_matches_torch(cuda, d, with_delta):
    from paper_2502_06766_b200.model import rmsnorm

    g = torch.Generator(device=cuda).manual_seed(d)
    x = torch.randn((1, d), generator=g, device=cuda).to(torch.bfloat16)
    delta = torch.randn((1, d), generator=g, device=cuda).to(torch.bfloat16) if with_delta else None
    w = torch.rand(d, generator=g, device=cuda) + 0.5
    ref_x = x + delta if with_delta else x.clone()  # bf16 + bf16 -> bf16
    ref_h = rmsnorm(ref_x, w, 1e-5)
    h = torch.empty_like(x)
    _call("tkv_model_add_rmsnorm", _vp(x), _vp(delta), _vp(w), 1e-5, _vp(h), d, _st(cuda))
    torch.cuda.synchronize()
    assert torch.equal(x, ref_x)  # the residual stream: exact
    # h: same math, the mean-square reduction order differs -> at most 1 bf16 ulp
    err = (h.float() - ref_h.float()).abs()
    assert float((err / ref_h.float().abs().clamp_min(1e-3)).max()) <= 2 ** -7


def test_qkv_rope_append_matches_torch(cuda):
    from paper_2502_06766_b200.model import LLAMA3_8B, apply_rope, rope_tables

    hq, hkv, hd, rows = 8, 2, 128, 300
    n_ctx, n_win, pos = 200, 7, 207
    g = torch.Generator(device=cuda).manual_seed(3)
    qkv = torch.randn((1, (hq + 2 * hkv) * hd), generator=g, device=cuda).to(torch.bfloat16)
    cos, sin = rope_tables(LLAMA3_8B, rows, cuda)
    K = torch.randn((1, hkv, rows, hd), generator=g, device=cuda).to(torch.bfloat16)
    V = torch.randn((1, hkv, rows, hd), generator=g, device=cuda).to(torch.bfloat16)
    K0, V0 = K.clone(), V.clone()
    q_out = torch.empty((1, hq, hd), dtype=torch.bfloat16, device=cuda)
    pos_t = torch.tensor([pos], dtype=torch.int64, device=cuda)
    nc = torch.tensor([n_ctx], dtype=torch.int32, device=cuda)
    nw = torch.tensor([n_win], dtype=torch.int32, device=cuda)
    _call("tkv_model_qkv_rope_append", _vp(qkv), _vp(cos), _vp(sin), _vp(pos_t), _vp(q_out), _vp(K), _vp(V),
          _vp(nc), _vp(nw), rows, hq, hkv, hd, _st(cuda))
    torch.cuda.synchronize()
    f = qkv.float()
    c, s = cos[pos:pos + 1], sin[pos:pos + 1]
    ref_q = apply_rope(f[:, :hq * hd].view(1, hq, hd), c, s).to(torch.bfloat16)
    ref_k = apply_rope(f[:, hq * hd:(hq + hkv) * hd].view(1, hkv, hd), c, s).to(torch.bfloat16)
    ref_v = qkv[:, (hq + hkv) * hd:].view(1, hkv, hd)
    assert torch.equal(q_out, ref_q)
    row = n_ctx + n_win
    assert torch.equal(K[0, :, row], ref_k[0]) and torch.equal(V[0, :, row], ref_v[0])
    # every other row untouched, the window counter not advanced
    K[0, :, row], V[0, :, row] = K0[0, :, row], V0[0, :, row]
    assert torch.equal(K, K0) and torch.equal(V, V0)
    assert int(nw.item()) == n_win


def test_silu_mul_matches_torch(cuda):
    ffn = 14336
    g = torch.Generator(device=cuda).manual_seed(5)
    gu = (torch.randn((1, 2 * ffn), generator=g, device=cuda) * 3).to(torch.bfloat16)
    out = torch.empty((1, ffn), dtype=torch.bfloat16, device=cuda)
    _call("tkv_model_silu_mul", _vp(gu), _vp(out), ffn, _st(cuda))
    torch.cuda.synchronize()
    ref = (torch.nn.functional.silu(gu[:, :ffn].float()) * gu[:, ffn:].float()).to(torch.bfloat16)
    err = (out.float() - ref.float()).abs()
    assert float((err / ref.float().abs().clamp_min(1e-2)).max()) <= 2 ** -7


@pytest.mark.parametrize("n", [128256, 512, 1])
def test_logits_argmax_first_max_and_copy(cuda, n):
    g = torch.Generator(device=cuda).manual_seed(n)
    lg = torch.randn((1, n), generator=g, device=cuda).to(torch.bfloat16)
    if n > 10:  # a tie at the maximum: the lower index wins (torch.argmax's first occurrence)
        m = lg.max()
        lg[0, n // 3] = m
        lg[0, n // 2] = m
    out = torch.empty((1, n), dtype=torch.float32, device=cuda)
    tok = torch.full((1,), -1, dtype=torch.int64, device=cuda)
    scratch = torch.zeros(2, dtype=torch.int64, device=cuda)
    for _ in range(3):  # the scratch words reset themselves: repeated calls agree
        _call("tkv_model_logits_argmax", _vp(lg), n, _vp(out), _vp(tok), _vp(scratch), _st(cuda))
        torch.cuda.synchronize()
        assert int(tok.item()) == int(lg.float().argmax().item())
        assert torch.equal(out, lg.float())
        assert int(scratch.abs().sum().item()) == 0
