"""GPU parity of ttt_qkv_rope_split (RoPE'd q and the step's K / V slots from a fused projection
output) against the fp64 oracle (oracle/rope.py). Tolerance: the outputs are bf16 roundings of fp32
arithmetic on exact bf16 inputs with fp64-built angles -> |gpu - ref| <= 2^-8 |ref| + 1e-6."""
import numpy as np
import pytest
import torch

import paper_2603_18567_b200 as ttt
from oracle import rope as OR

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("B,L,Hq,Hkv,D,use_pos", [(1, 5, 2, 1, 16, False), (2, 2048, 32, 8, 128, False),
                                                  (1, 16384, 4, 2, 128, False), (2, 300, 8, 2, 64, True)])
def test_qkv_rope_split_vs_oracle(B, L, Hq, Hkv, D, use_pos):
    g = torch.Generator().manual_seed(L + D)
    qkv = torch.randn(B, L, Hq + 2 * Hkv, D, generator=g).to(torch.bfloat16)
    pos = torch.randint(0, 40000, (B, L), generator=g, dtype=torch.int32) if use_pos else None
    d = ttt.rope_desc(B, L, Hq, Hkv, D, 500000.0)
    dev = qkv.cuda()
    q = torch.empty(B, L, Hq, D, dtype=torch.bfloat16, device="cuda")
    k = torch.empty(B, L, Hkv, D, dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    ws = torch.empty(ttt.ttt_rope_workspace_size(d, use_pos), dtype=torch.uint8, device="cuda")
    ttt.ttt_qkv_rope_split(d, dev, q, k, v, ws, positions=None if pos is None else pos.cuda())
    torch.cuda.synchronize()
    qr, kr, vr = OR.qkv_rope_split(qkv.double().numpy(), Hq, Hkv, 500000.0,
                                   positions=None if pos is None else pos.numpy()[:, :])
    for name, got, want in (("q", q, qr), ("k", k, kr)):
        got = got.double().cpu().numpy()
        err = np.abs(got - want)
        assert (err <= 2.0 ** -8 * np.abs(want) + 1e-6).all(), f"{name}: max_abs={err.max():.3e}"
    assert torch.equal(v.cpu(), qkv[:, :, Hq + Hkv:])   # V is copied bit for bit


def _torch_rope(x, pos, base):
    """float64 torch mirror of oracle.rope.rope_rotate (autograd reference)."""
    D = x.shape[-1]
    half = D // 2
    inv = base ** (-torch.arange(half, dtype=torch.float64) * 2.0 / D)
    th = pos.to(torch.float64)[..., None] * inv
    c, s = th.cos()[..., None, :], th.sin()[..., None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)


def test_qkv_rope_join_bwd_and_autograd():
    """The backward kernel is the adjoint: dqkv matches torch float64 autograd of the rotation."""
    from paper_2603_18567_b200.autograd import qkv_rope_split
    B, L, Hq, Hkv, D = 2, 96, 8, 2, 128
    g = torch.Generator().manual_seed(3)
    qkv = torch.randn(B, L, Hq + 2 * Hkv, D, generator=g).to(torch.bfloat16)
    wq, wk, wv = (torch.randn(B, L, h, D, generator=g).to(torch.bfloat16) for h in (Hq, Hkv, Hkv))
    x = qkv.cuda().requires_grad_(True)
    q, k, v = qkv_rope_split(x, Hq, Hkv, 500000.0)
    ((q.float() * wq.cuda().float()).sum() + (k.float() * wk.cuda().float()).sum()
     + (v.float() * wv.cuda().float()).sum()).backward()
    xr = qkv.double().requires_grad_(True)
    pos = torch.arange(L)
    qr = _torch_rope(xr[:, :, :Hq], pos, 500000.0)
    kr = _torch_rope(xr[:, :, Hq:Hq + Hkv], pos, 500000.0)
    ((qr * wq.double()).sum() + (kr * wk.double()).sum() + (xr[:, :, Hq + Hkv:] * wv.double()).sum()).backward()
    got, want = x.grad.double().cpu(), xr.grad
    assert ((got - want).abs() <= 2.0 ** -8 * want.abs() + 1e-6).all(), (got - want).abs().max().item()
    np.testing.assert_allclose(q.detach().double().cpu().numpy(), qr.detach().numpy(), rtol=2.0 ** -8, atol=1e-6)
