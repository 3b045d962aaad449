"""A minimal EAGLE-3-style draft TTT unroll around the kernels (in part).

Per TTT step j (§2.4):
    x_0      = fc([low | mid | high])              fused target hidden states, 3d -> d  (cuBLAS GEMM)
    qkv_j    = x_j W_qkv                                                                  (cuBLAS GEMM)
    q_j, k_j, v_j = qkv_rope_split(qkv_j)          RoPE at positions 0..L-1 every step   (our kernel)
    o_j      = TTT attention of step j over K_0 = k_0, K_i = k_i (i = 1..j)              (our kernels)
    h_j      = o_j W_o + x_j ;  x_{j+1} = h_j      the next step drafts from this step's output
    loss_j   = soft_label_loss(h_j W_lm, p_j)      masked soft-label loss, Alg. 3 backward (our kernel)
The layer's norms and MLP are left out (they are row-local GEMM / elementwise work outside the
attention path); the projections are plain library GEMMs (torch.matmul on bf16 -> cuBLAS).
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import torch

from .autograd import qkv_rope_split, soft_label_loss, ttt_attention


class DraftTTT(torch.nn.Module):
    def __init__(self, hidden: int, num_q_heads: int, num_kv_heads: int, head_dim: int, vocab: int,
                 rope_base: float = 500000.0, dtype=torch.bfloat16, device="cuda", seed: int = 0):
        super().__init__()
        g = torch.Generator(device="cpu").manual_seed(seed)
        w = lambda o, i: torch.nn.Parameter(
            (torch.randn(o, i, generator=g) / i ** 0.5).to(dtype=dtype, device=device))
        self.Hq, self.Hkv, self.D, self.base = num_q_heads, num_kv_heads, head_dim, rope_base
        self.fc = w(hidden, 3 * hidden)
        self.w_qkv = w((num_q_heads + 2 * num_kv_heads) * head_dim, hidden)
        self.w_o = w(hidden, num_q_heads * head_dim)
        self.lm_head = w(vocab, hidden)

    def forward(self, low_mid_high: torch.Tensor, targets: Sequence[torch.Tensor],
                loss_mask: Optional[torch.Tensor] = None, seq_lens: Optional[Sequence[int]] = None) -> torch.Tensor:
        """low_mid_high [B, L, 3d]; targets: per step p_j [B L, V] (target distributions);
        returns the summed loss over the S = len(targets) steps."""
        B, L, _ = low_mid_high.shape
        x = low_mid_high @ self.fc.t()
        ks: List[torch.Tensor] = []
        vs: List[torch.Tensor] = []
        total = 0.0
        for j, p in enumerate(targets):
            qkv = (x @ self.w_qkv.t()).view(B, L, self.Hq + 2 * self.Hkv, self.D)
            q, k, v = qkv_rope_split(qkv, self.Hq, self.Hkv, self.base)
            if j == 0:
                k0, v0 = k, v
            else:
                ks.append(k)
                vs.append(v)
            o = ttt_attention(q, k0, v0, ks, vs, j, seq_lens=seq_lens)
            x = o.reshape(B, L, self.Hq * self.D) @ self.w_o.t() + x
            logits = (x @ self.lm_head.t()).reshape(B * L, -1)
            total = total + soft_label_loss(logits, p, loss_mask)
        return total
