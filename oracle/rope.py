"""TEST INFRASTRUCTURE — fp64 CPU oracle of the draft layer's rotary position embedding
on the TTT step's fresh projections ("q/k/v projections writing
straight into step-list slots, RoPE with repeated position ids"). NOT product code; only
tests/ may use it; it shares nothing with the CUDA path.

What it follows
  * draft and target share the positional convention and "a TTT step reuses
    position ids 0..T_pad-1" — every step rotates its q / k with the same positions as the
    base step (reading R23).
  * The paper names no RoPE variant; the Llama draft layers of EAGLE-3 use the rotate-half
    form (reading R24): for i < D/2, theta_i = pos * base^(-2 i / D),
        x'_i       = x_i cos theta_i - x_{i+D/2} sin theta_i
        x'_{i+D/2} = x_{i+D/2} cos theta_i + x_i sin theta_i.
  * Layout (reading R25): the fused projection output qkv [B, L, Hq + 2 Hkv, D] (q heads,
    then k heads, then v heads) is split into q [B, L, Hq, D] (rotated), the step's K slot
    [B, L, Hkv, D] (rotated) and V slot [B, L, Hkv, D] (copied).
Pinned by tests/test_oracle_rope.py (transformers' Llama apply_rotary_pos_emb in float64,
position 0 = identity, pairwise norms, relative-position invariance of q.k).
"""
from __future__ import annotations

import numpy as np


def rope_rotate(x, positions, base: float):
    """x [..., L, H, D] (L the position axis = x.shape[-3]); positions [L] (or broadcastable
    [..., L]). Returns the rotate-half RoPE of x in fp64."""
    x = np.asarray(x, np.float64)
    D = x.shape[-1]
    half = D // 2
    inv_freq = base ** (-np.arange(half, dtype=np.float64) * 2.0 / D)      # base^(-2i/D)
    theta = np.asarray(positions, np.float64)[..., None] * inv_freq          # [..., L, D/2]
    c = np.cos(theta)[..., None, :]                                          # [..., L, 1, D/2]
    s = np.sin(theta)[..., None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def qkv_rope_split(qkv, Hq: int, Hkv: int, base: float, positions=None):
    """qkv [B, L, Hq + 2 Hkv, D] -> (q, k, v) with q, k rotated at positions (default 0..L-1)."""
    qkv = np.asarray(qkv, np.float64)
    L = qkv.shape[1]
    pos = np.arange(L) if positions is None else np.asarray(positions)
    q = qkv[:, :, :Hq]
    k = qkv[:, :, Hq:Hq + Hkv]
    v = qkv[:, :, Hq + Hkv:Hq + 2 * Hkv]
    return rope_rotate(q, pos, base), rope_rotate(k, pos, base), v.copy()
