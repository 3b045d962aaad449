"""Pins of the RoPE oracle (oracle/rope.py) — never against the CUDA path. CPU only."""
import numpy as np
import pytest
import torch

from oracle import rope as OR


def test_matches_transformers_llama_rotary_float64():
    """Library routine: transformers' Llama rotate-half apply_rotary_pos_emb in float64."""
    lm = pytest.importorskip("transformers.models.llama.modeling_llama")
    rng = np.random.default_rng(0)
    B, L, H, D, base = 2, 37, 3, 64, 500000.0
    x = rng.standard_normal((B, L, H, D))
    pos = np.arange(L)
    inv_freq = 1.0 / (base ** (torch.arange(0, D, 2, dtype=torch.float64) / D))
    freqs = torch.tensor(pos, dtype=torch.float64)[:, None] * inv_freq[None, :]
    emb = torch.cat([freqs, freqs], dim=-1)
    cos, sin = emb.cos()[None], emb.sin()[None]                    # [1, L, D]
    xt = torch.tensor(x).transpose(1, 2)                            # [B, H, L, D]
    q_ref, k_ref = lm.apply_rotary_pos_emb(xt, xt, cos, sin)
    np.testing.assert_allclose(OR.rope_rotate(x, pos, base), q_ref.transpose(1, 2).numpy(), rtol=1e-12, atol=1e-12)


def test_identity_at_zero_norms_and_relative_positions():
    rng = np.random.default_rng(1)
    D, base = 128, 10000.0
    x = rng.standard_normal((1, 5, 2, D))
    np.testing.assert_array_equal(OR.rope_rotate(x, np.zeros(5), base), x)          # theta = 0
    y = OR.rope_rotate(x, np.arange(5) * 97, base)
    half = D // 2
    np.testing.assert_allclose(x[..., :half] ** 2 + x[..., half:] ** 2,
                               y[..., :half] ** 2 + y[..., half:] ** 2, rtol=1e-12)  # each pair rotates
    q = rng.standard_normal((1, 1, 1, D))
    k = rng.standard_normal((1, 1, 1, D))
    for m, n, s in ((5, 2, 11), (300, 1000, 4096), (0, 7, 123)):
        a = (OR.rope_rotate(q, [m], base) * OR.rope_rotate(k, [n], base)).sum()
        b = (OR.rope_rotate(q, [m + s], base) * OR.rope_rotate(k, [n + s], base)).sum()
        assert abs(a - b) < 1e-9 * max(1.0, abs(a))                                # depends on m - n only


def test_split_layout():
    rng = np.random.default_rng(2)
    B, L, Hq, Hkv, D = 2, 6, 4, 2, 16
    qkv = rng.standard_normal((B, L, Hq + 2 * Hkv, D))
    q, k, v = OR.qkv_rope_split(qkv, Hq, Hkv, 10000.0)
    np.testing.assert_array_equal(v, qkv[:, :, Hq + Hkv:])
    np.testing.assert_array_equal(q[:, 0], qkv[:, 0, :Hq])                          # position 0
    np.testing.assert_allclose(k, OR.rope_rotate(qkv[:, :, Hq:Hq + Hkv], np.arange(L), 10000.0))
