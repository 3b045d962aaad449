"""GPU: the minimal EAGLE-3-style draft TTT unroll (paper_2603_18567_b200/draft.py: library GEMMs +
our RoPE split, TTT attention and Alg. 3 loss kernels) against the same computation in float64 torch
on the CPU, whose attention is dense softmax under the oracle's explicit Alg. 2 mask and whose loss
is torch's soft-label cross-entropy (both pinned in tests/test_oracle_*). bf16 end to end, so the
comparison is on the loss and on parameter-gradient norms: relative Frobenius error <= 5e-2."""
import numpy as np
import pytest
import torch

import oracle
from paper_2603_18567_b200.draft import DraftTTT

pytestmark = pytest.mark.gpu


def _rope64(x, base):
    D = x.shape[-1]
    half = D // 2
    L = x.shape[1]
    inv = base ** (-torch.arange(half, dtype=torch.float64) * 2.0 / D)
    th = torch.arange(L, dtype=torch.float64)[:, None] * inv
    c, s = th.cos()[None, :, None, :], th.sin()[None, :, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)


def _reference(m, lmh, targets, mask, lens):
    P = {n: p.detach().double().cpu().requires_grad_(True) for n, p in m.named_parameters()}
    B, L, _ = lmh.shape
    Hq, Hkv, D = m.Hq, m.Hkv, m.D
    x = lmh.double() @ P["fc"].t()
    ks, vs, total = [], [], 0.0
    for j, p in enumerate(targets):
        qkv = (x @ P["w_qkv"].t()).view(B, L, Hq + 2 * Hkv, D)
        q, k, v = _rope64(qkv[:, :, :Hq], m.base), _rope64(qkv[:, :, Hq:Hq + Hkv], m.base), qkv[:, :, Hq + Hkv:]
        if j == 0:
            k0, v0 = k, v
        else:
            ks.append(k)
            vs.append(v)
        K = torch.cat([k0] + ks, dim=1).repeat_interleave(Hq // Hkv, dim=2).transpose(1, 2)
        V = torch.cat([v0] + vs, dim=1).repeat_interleave(Hq // Hkv, dim=2).transpose(1, 2)
        outs = []
        for b in range(B):
            msk = torch.from_numpy(oracle.mask_dense(L, int(lens[b]), j))
            outs.append(torch.nn.functional.scaled_dot_product_attention(q[b:b + 1].transpose(1, 2), K[b:b + 1],
                                                                         V[b:b + 1], attn_mask=msk))
        o = torch.cat(outs).transpose(1, 2).reshape(B, L, Hq * D)
        x = o @ P["w_o"].t() + x
        logits = (x @ P["lm_head"].t()).reshape(B * L, -1)
        sel = mask.bool()
        total = total + torch.nn.functional.cross_entropy(logits[sel], p.double()[sel], reduction="mean")
    total.backward()
    return total.item(), {n: t.grad for n, t in P.items()}


def test_draft_ttt_unroll_matches_float64_reference(cuda_ok):
    torch.manual_seed(0)
    B, L, d, Hq, Hkv, D, V, S = 2, 256, 256, 4, 2, 64, 512, 3
    m = DraftTTT(d, Hq, Hkv, D, V, device="cuda", seed=1)
    g = torch.Generator().manual_seed(2)
    lmh = (torch.randn(B, L, 3 * d, generator=g)).to(torch.bfloat16)
    targets = [torch.softmax(torch.randn(B * L, V, generator=g) * 2, dim=-1).to(torch.bfloat16) for _ in range(S)]
    mask = (torch.rand(B * L, generator=g) > 0.2).to(torch.uint8)
    lens = [L, 200]
    loss = m(lmh.cuda(), [t.cuda() for t in targets], mask.cuda(), seq_lens=lens)
    loss.backward()
    ref_loss, ref_grads = _reference(m, lmh, targets, mask, lens)
    assert abs(loss.item() - ref_loss) <= 2e-2 * abs(ref_loss), (loss.item(), ref_loss)
    for n, p in m.named_parameters():
        got, want = p.grad.double().cpu(), ref_grads[n]
        rel = ((got - want).norm() / want.norm()).item()
        assert rel <= 5e-2, f"{n}: relative grad error {rel:.3e}"
