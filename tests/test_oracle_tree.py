"""Pins of the tree-attention oracle (oracle/tree.py) against what the paper and
mathematics fix — never against the CUDA path. CPU only."""
import numpy as np
import pytest
import torch

from oracle import tree as OT


def _rand(rng, *shape):
    return rng.standard_normal(shape)


def test_ancestor_sets_and_invalid_parents():
    # 0 <- 1 <- 3 ; 0 <- 2 ; 4 hangs off the context tip
    anc = OT.ancestors_or_self([-1, 0, 0, 1, -1])
    assert anc == [{0}, {0, 1}, {0, 2}, {0, 1, 3}, {4}]
    for bad in ([0], [-1, 1], [-1, 3, 0], [-2]):
        with pytest.raises(ValueError):
            OT.ancestors_or_self(bad)


def test_mask_brute_force_random_trees():
    """Brute force: k allowed iff prefix, or reachable from t by following parents."""
    rng = np.random.default_rng(0)
    for _ in range(50):
        n = int(rng.integers(1, 20))
        parents = [-1] + [int(rng.integers(-1, t)) for t in range(1, n)]
        P = int(rng.integers(0, 7))
        m = OT.tree_mask(P, parents, P + n + 3)
        for t in range(n):
            walk, u = set(), t
            while u != -1:
                walk.add(u)
                u = parents[u]
            want = [True] * P + [(j in walk) for j in range(n)] + [False] * 3
            assert list(m[t]) == want
            assert m[t].sum() == P + len(walk)   # |allowed| = prefix + depth + 1


def test_chain_tree_is_causal_attention():
    """A chain (topk = 1) is ordinary causal attention over prefix + chain:
    torch SDPA with a lower-triangular (offset P) mask in float64."""
    rng = np.random.default_rng(1)
    B, n, Hq, Hkv, D, P = 2, 9, 4, 2, 16, 13
    q = _rand(rng, B, n, Hq, D)
    k = _rand(rng, B, P + n, Hkv, D)
    v = _rand(rng, B, P + n, Hkv, D)
    parents = [[-1] + list(range(n - 1))] * B
    out, lse = OT.tree_attention(q, k, v, [P] * B, parents)
    qt = torch.tensor(q).transpose(1, 2)
    kt = torch.tensor(k).repeat_interleave(Hq // Hkv, dim=2).transpose(1, 2)
    vt = torch.tensor(v).repeat_interleave(Hq // Hkv, dim=2).transpose(1, 2)
    causal = torch.ones(n, P + n, dtype=torch.bool).tril(diagonal=P)
    ref = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, attn_mask=causal)
    np.testing.assert_allclose(out, ref.transpose(1, 2).numpy(), rtol=1e-12, atol=1e-12)
    s = (qt @ kt.transpose(-1, -2)) / np.sqrt(D)
    ref_lse = torch.logsumexp(s.masked_fill(~causal, float("-inf")), dim=-1)
    np.testing.assert_allclose(lse, ref_lse.numpy(), rtol=1e-12, atol=1e-12)


def test_closed_forms_q_zero_and_single_key():
    """q = 0: out = mean of the allowed V rows, lse = ln |allowed| (|allowed| = P + depth + 1).
    Star tree with P = 0: every node sees only itself -> out = its own v, lse = c q.k."""
    rng = np.random.default_rng(2)
    B, n, Hq, Hkv, D, P = 1, 6, 2, 1, 8, 5
    parents = [[-1, 0, 0, 1, 3, -1]]
    k = _rand(rng, B, P + n, Hkv, D)
    v = _rand(rng, B, P + n, Hkv, D)
    out, lse = OT.tree_attention(np.zeros((B, n, Hq, D)), k, v, [P], parents)
    anc = OT.ancestors_or_self(parents[0])
    for t in range(n):
        rows = list(range(P)) + [P + u for u in sorted(anc[t])]
        np.testing.assert_allclose(out[0, t, 0], v[0, rows, 0].mean(0), rtol=1e-12)
        assert abs(lse[0, 0, t] - np.log(len(rows))) < 1e-12
    q = _rand(rng, B, n, Hq, D)
    out, lse = OT.tree_attention(q, k[:, P:], v[:, P:], [0], [[-1] * n])
    np.testing.assert_allclose(out[0, :, 0], v[0, P:, 0], rtol=1e-12)
    np.testing.assert_allclose(lse[0, 0], (q[0, :, 0] * k[0, P:, 0]).sum(-1) / np.sqrt(D), rtol=1e-12)


def test_masked_keys_inert_and_gqa():
    """Keys outside the mask (other branches, rows past P + n) do not change the output;
    GQA equals MHA with repeated K/V."""
    rng = np.random.default_rng(3)
    B, n, Hq, Hkv, D, P = 1, 5, 4, 2, 8, 4
    parents = [[-1, 0, 0, 1, 2]]
    q = _rand(rng, B, n, Hq, D)
    k = _rand(rng, B, P + n + 2, Hkv, D)
    v = _rand(rng, B, P + n + 2, Hkv, D)
    a, _ = OT.tree_attention(q, k, v, [P], parents)
    k2, v2 = k.copy(), v.copy()
    k2[:, P + n:] = 1e3
    v2[:, P + n:] = -7.0
    b, _ = OT.tree_attention(q, k2, v2, [P], parents)
    np.testing.assert_array_equal(a, b)
    c, _ = OT.tree_attention(q, np.repeat(k, 2, axis=2), np.repeat(v, 2, axis=2), [P], parents)
    np.testing.assert_allclose(a, c, rtol=1e-13, atol=1e-13)
