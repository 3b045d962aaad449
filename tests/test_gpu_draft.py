"""GPU: the EAGLE-3-style draft decoder layer unrolled over TTT steps (paper_2603_18567_b200/draft.py:
RMSNorms, library GEMMs, SwiGLU MLP, and our RoPE split, TTT attention and Alg. 3 loss kernels)
against the same computation in float64 torch on the CPU, whose attention is dense softmax under the
oracle's explicit Alg. 2 mask and whose loss is torch's soft-label cross-entropy (both pinned in
tests/test_oracle_*).

Element by element: the loss within 2e-2 relative, every parameter gradient within
atol = 3e-2 * max|ref| (of that tensor) + rtol 1e-1 * |ref|. Derivation of the bound: the GPU run
keeps every activation in bf16 (unit roundoff u = 2^-9 ~ 2e-3) across ~12 chained ops per step and 3
steps (fc, norm, qkv, RoPE, attention, o_proj, norm, gate/up/down, norm, LM head, loss), each adding
an O(u) relative perturbation with random sign, so per-element gradient errors of ~sqrt(36) u ~ 1.2e-2
of the tensor's scale; 3e-2 leaves 2.5 sigma of headroom. The data-parallel exchange of these
gradients (dp.exchange_grads) is checked at world size 1 here and at 2 (gloo) in test_dp_gloo.py."""
import numpy as np
import pytest
import torch

import oracle
from paper_2603_18567_b200.dp import GradBuckets, exchange_grads
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


def _rms64(x, w, eps=1e-6):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w


def _reference(m, lmh, targets, mask, lens):
    P = {n: p.detach().double().cpu().requires_grad_(True) for n, p in m.named_parameters()}
    B, L, _ = lmh.shape
    Hq, Hkv, D = m.Hq, m.Hkv, m.D
    x = lmh.double() @ P["fc"].t()
    ks, vs, total = [], [], 0.0
    for j, p in enumerate(targets):
        a = _rms64(x, P["g_attn"])
        qkv = (a @ P["w_qkv"].t()).view(B, L, Hq + 2 * Hkv, D)
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
        h = o @ P["w_o"].t() + x
        mm = _rms64(h, P["g_mlp"])
        x = h + (torch.nn.functional.silu(mm @ P["w_gate"].t()) * (mm @ P["w_up"].t())) @ P["w_down"].t()
        logits = (_rms64(x, P["g_out"]) @ P["lm_head"].t()).reshape(B * L, -1)
        sel = mask.bool()
        total = total + torch.nn.functional.cross_entropy(logits[sel], p.double()[sel], reduction="mean")
    total.backward()
    return total.item(), {n: t.grad for n, t in P.items()}


def test_draft_ttt_unroll_matches_float64_reference(cuda_ok):
    torch.manual_seed(0)
    B, L, d, Hq, Hkv, D, V, S = 2, 256, 256, 4, 2, 64, 512, 3
    m = DraftTTT(d, Hq, Hkv, D, V, intermediate=512, device="cuda", seed=1)
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
        got, want = p.grad.double().cpu().numpy(), ref_grads[n].numpy()
        atol = 3e-2 * np.abs(want).max()
        err = np.abs(got - want)
        bad = err > atol + 1e-1 * np.abs(want)
        assert not bad.any(), (f"{n}: {int(bad.sum())}/{bad.size} elements out of bound, max_abs {err.max():.3e} "
                               f"(atol {atol:.3e})")
    # the exchange the data-parallel optimizer step runs on these real gradients (world size 1: identity)
    before = m.flat_grads().clone()
    exchange_grads(m, GradBuckets(m.num_grad_elements(), 7, dtype=torch.bfloat16, device="cuda"))
    assert torch.equal(m.flat_grads(), before)
