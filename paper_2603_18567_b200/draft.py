"""An EAGLE-3-style draft decoder layer unrolled over TTT steps around the kernels (SURVEY.md §8(f)
NEXT #2).

Per TTT step j (§2.4; the draft layer trained with TTT, PAPER.md:277-285, 331;
SPEC.md:327-330, 470: "one decoder layer using ttt_attention_step; returns next-step features (fed
back at the next TTT step)"):

    x_0      = fc([low | mid | high])                     fused target hidden states, 3d -> d
    a_j      = rmsnorm(x_j) * g_attn
    q_j, k_j, v_j = qkv_rope_split(a_j W_qkv)              RoPE at positions 0..L-1 every step
    o_j      = TTT attention of step j over K_0 = k_0, K_i = k_i (i = 1..j)    (Alg. 1 / Alg. 2)
    h_j      = o_j W_o + x_j
    x_{j+1}  = h_j + W_down (silu(m_j W_gate) * (m_j W_up)),  m_j = rmsnorm(h_j) * g_mlp   (SwiGLU MLP)
    loss_j   = soft_label_loss((rmsnorm(x_{j+1}) * g_out) W_lm, p_j)   masked soft-label loss, Alg. 3

The next step drafts from x_{j+1} (gradients flow through the chain, which is why the attention
backward runs per step in reverse order). The attention, the RoPE split and the loss are our kernels
(autograd.py); the projections and the MLP are plain library GEMMs (torch.matmul on bf16 -> cuBLAS)
and the RMSNorms are torch elementwise ops — row-local work outside the attention hot path.
`flat_grads()` / `set_flat_grads()` move the parameter gradients through one flat buffer, the form
the data-parallel exchange (dp.GradBuckets / dp.Zero2Buckets) reduces.
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import torch

from .autograd import qkv_rope_split, soft_label_loss, ttt_attention


def rmsnorm(x: torch.Tensor, weight: torch.Tensor, eps: float = 1e-6) -> torch.Tensor:
    """Llama RMSNorm in fp32 (x / sqrt(mean(x^2) + eps) * weight), returned in x's dtype."""
    xf = x.float()
    y = xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)
    return (y * weight.float()).to(x.dtype)


class DraftTTT(torch.nn.Module):
    def __init__(self, hidden: int, num_q_heads: int, num_kv_heads: int, head_dim: int, vocab: int,
                 intermediate: Optional[int] = None, rope_base: float = 500000.0, dtype=torch.bfloat16,
                 device="cuda", seed: int = 0):
        super().__init__()
        g = torch.Generator(device="cpu").manual_seed(seed)
        w = lambda o, i: torch.nn.Parameter(
            (torch.randn(o, i, generator=g) / i ** 0.5).to(dtype=dtype, device=device))
        nw = lambda n: torch.nn.Parameter((1.0 + 0.1 * torch.randn(n, generator=g)).to(dtype=dtype, device=device))
        inter = intermediate or 2 * hidden
        self.Hq, self.Hkv, self.D, self.base = num_q_heads, num_kv_heads, head_dim, rope_base
        self.fc = w(hidden, 3 * hidden)
        self.g_attn = nw(hidden)
        self.w_qkv = w((num_q_heads + 2 * num_kv_heads) * head_dim, hidden)
        self.w_o = w(hidden, num_q_heads * head_dim)
        self.g_mlp = nw(hidden)
        self.w_gate = w(inter, hidden)
        self.w_up = w(inter, hidden)
        self.w_down = w(hidden, inter)
        self.g_out = nw(hidden)
        self.lm_head = w(vocab, hidden)

    def step(self, x: torch.Tensor, j: int, kv: dict, seq_lens=None):
        """One TTT step: returns (next-step features x_{j+1}, logits [B L, V])."""
        B, L, d = x.shape
        a = rmsnorm(x, self.g_attn)
        qkv = (a @ self.w_qkv.t()).view(B, L, self.Hq + 2 * self.Hkv, self.D)
        q, k, v = qkv_rope_split(qkv, self.Hq, self.Hkv, self.base)
        if j == 0:
            kv["k0"], kv["v0"] = k, v
        else:
            kv["ks"].append(k)
            kv["vs"].append(v)
        o = ttt_attention(q, kv["k0"], kv["v0"], kv["ks"], kv["vs"], j, seq_lens=seq_lens)
        h = o.reshape(B, L, self.Hq * self.D) @ self.w_o.t() + x
        m = rmsnorm(h, self.g_mlp)
        x_next = h + (torch.nn.functional.silu(m @ self.w_gate.t()) * (m @ self.w_up.t())) @ self.w_down.t()
        logits = (rmsnorm(x_next, self.g_out) @ self.lm_head.t()).reshape(B * L, -1)
        return x_next, logits

    def forward(self, low_mid_high: torch.Tensor, targets: Sequence[torch.Tensor],
                loss_mask: Optional[torch.Tensor] = None, seq_lens: Optional[Sequence[int]] = None) -> torch.Tensor:
        """low_mid_high [B, L, 3d]; targets: per step p_j [B L, V] (target distributions);
        returns the summed loss over the S = len(targets) steps."""
        x = low_mid_high @ self.fc.t()
        kv = {"ks": [], "vs": []}
        total = 0.0
        for j, p in enumerate(targets):
            x, logits = self.step(x, j, kv, seq_lens)
            total = total + soft_label_loss(logits, p, loss_mask)
        return total

    # ---- the data-parallel exchange's view of the gradients ----
    def flat_grads(self, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """All parameter gradients concatenated in parameter order (into `out` when given)."""
        gs = [p.grad.reshape(-1) for p in self.parameters()]
        if out is None:
            return torch.cat(gs)
        torch.cat(gs, out=out[:sum(g.numel() for g in gs)])
        return out

    def set_flat_grads(self, flat: torch.Tensor) -> None:
        """Write an (exchanged, averaged) flat buffer back into the parameter gradients."""
        off = 0
        for p in self.parameters():
            n = p.numel()
            p.grad.copy_(flat[off:off + n].view_as(p.grad))
            off += n

    def num_grad_elements(self) -> int:
        return sum(p.numel() for p in self.parameters())
