"""Pins for the oracle's packed-batch functions (oracle.fwd_packed / bwd_packed) — CPU only.

A packed batch is B sequences laid back to back, sequence b = rows [cu[b], cu[b+1]) with no
padding rows. Checked against things other than the slicing itself:
  * torch float64 causal scaled_dot_product_attention per sequence at j = 0 (library routine;
    Alg. 2 with no step keys is causal attention);
  * Alg. 1 literally on sampled rows, j = 2;
  * the padded form of the same sequences (padding rows carry dO = 0): Alg. 2's m_pad
     keeps padding keys out of every valid row, so the valid rows and the
    valid keys' gradients must be the packed result — a wrong offset, a transposed lse or a
    row / head mix-up in the packing fails here.
"""
import math

import numpy as np
import pytest
import torch

import oracle


def _packed_case(lens, Hq=4, Hkv=2, D=8, j=2, seed=0):
    rng = np.random.default_rng(seed)
    N = int(sum(lens))
    f = lambda *s: rng.standard_normal(s).astype(np.float32)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    return (f(N, Hq, D), f(N, Hkv, D), f(N, Hkv, D), [f(N, Hkv, D) for _ in range(j)],
            [f(N, Hkv, D) for _ in range(j)], f(N, Hq, D), cu)


def _pad(x, cu, L):
    B = len(cu) - 1
    out = np.zeros((B, L) + x.shape[1:], dtype=x.dtype)
    for b in range(B):
        out[b, :cu[b + 1] - cu[b]] = x[cu[b]:cu[b + 1]]
    return out


def test_packed_step0_is_causal_sdpa_per_sequence():
    lens = [5, 1, 9, 3]
    q, kb, vb, _, _, _, cu = _packed_case(lens, j=0, seed=1)
    c = 1.0 / math.sqrt(q.shape[2])
    out, lse = oracle.fwd_packed(q, kb, vb, [], [], cu)
    G = q.shape[1] // kb.shape[1]
    for b in range(len(lens)):
        r0, r1 = cu[b], cu[b + 1]
        tq = torch.tensor(q[r0:r1], dtype=torch.float64).transpose(0, 1)            # [Hq,T,D]
        tk = torch.tensor(kb[r0:r1], dtype=torch.float64).transpose(0, 1).repeat_interleave(G, 0)
        tv = torch.tensor(vb[r0:r1], dtype=torch.float64).transpose(0, 1).repeat_interleave(G, 0)
        ref = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, is_causal=True, scale=c)
        np.testing.assert_allclose(out[r0:r1], ref.transpose(0, 1).numpy(), rtol=1e-12, atol=1e-12)
        T = r1 - r0
        logits = (tq @ tk.transpose(1, 2)) * c + torch.triu(torch.full((T, T), -math.inf, dtype=torch.float64), 1)
        np.testing.assert_allclose(lse[:, r0:r1], torch.logsumexp(logits, -1).numpy(), rtol=1e-12, atol=1e-12)


def test_packed_matches_alg1_rows():
    lens = [4, 7, 2]
    q, kb, vb, ks, vs, _, cu = _packed_case(lens, j=2, seed=2)
    c = 1.0 / math.sqrt(q.shape[2])
    out, _ = oracle.fwd_packed(q, kb, vb, ks, vs, cu)
    G = q.shape[1] // kb.shape[1]
    for b in range(len(lens)):
        r0 = cu[b]
        for r in range(lens[b]):
            for h in (0, q.shape[1] - 1):
                g = h // G
                o = oracle.alg1_row(q[r0 + r, h], kb[r0:r0 + r + 1, g], vb[r0:r0 + r + 1, g],
                                    [k[r0 + r, g] for k in ks], [v[r0 + r, g] for v in vs], c)
                np.testing.assert_allclose(out[r0 + r, h], o, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("lens,j", [([3, 8, 1, 6], 2), ([12], 1), ([1, 1, 2], 3)])
def test_packed_equals_padded_valid_rows(lens, j):
    q, kb, vb, ks, vs, do, cu = _packed_case(lens, j=j, seed=3 + j)
    L = max(lens) + 3  # padding rows after every sequence
    P = lambda x: _pad(x, cu, L)
    out_p, lse_p = oracle.fwd_packed(q, kb, vb, ks, vs, cu)
    out_d, lse_d = oracle.fwd(P(q), P(kb), P(vb), [P(x) for x in ks], [P(x) for x in vs], seq_lens=lens)
    g_p = oracle.bwd_packed(q, kb, vb, ks, vs, do, cu)
    g_d = oracle.bwd(P(q), P(kb), P(vb), [P(x) for x in ks], [P(x) for x in vs], P(do), seq_lens=lens)
    for b, T in enumerate(lens):
        r0 = cu[b]
        np.testing.assert_allclose(out_p[r0:r0 + T], out_d[b, :T], rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(lse_p[:, r0:r0 + T], lse_d[b, :, :T], rtol=1e-12, atol=1e-13)
        for key in ("dq", "dk_base", "dv_base"):
            np.testing.assert_allclose(g_p[key][r0:r0 + T], g_d[key][b, :T], rtol=1e-11, atol=1e-12)
        for i in range(j):
            np.testing.assert_allclose(g_p["dk_steps"][i][r0:r0 + T], g_d["dk_steps"][i][b, :T], rtol=1e-11, atol=1e-12)
            np.testing.assert_allclose(g_p["dv_steps"][i][r0:r0 + T], g_d["dv_steps"][i][b, :T], rtol=1e-11, atol=1e-12)


def test_packed_rejects_empty_sequence():
    q, kb, vb, ks, vs, _, _ = _packed_case([3, 2], j=1)
    with pytest.raises(AssertionError):
        oracle.fwd_packed(q, kb, vb, ks, vs, [0, 3, 3, 5])
