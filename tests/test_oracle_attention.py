"""Pins for the oracle's TTT attention forward/backward — CPU only.

The oracle (oracle/ttt_oracle.c) is checked against things other than itself:
  * torch.nn.functional.scaled_dot_product_attention in float64 on CPU (a
    library routine) with a mask built structurally (tril + identity blocks),
    forward and autograd backward;
  * Alg. 1 literally, per row;
  * closed forms: q = 0 -> mean of allowed V rows and lse = ln|A|; a single
    allowed key -> out = v, lse = c q.k;
  * central finite differences (fp64) for every input tensor;
  * exact identities of softmax attention gradients;
  * GQA == MHA with explicitly repeated K/V.
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle


def _rand(rng, shape, scale=1.0):
    return (rng.standard_normal(shape) * scale).astype(np.float32)


def _case(B=2, L=12, Hq=4, Hkv=2, D=8, j=2, lens=None, seed=0, qscale=1.0):
    rng = np.random.default_rng(seed)
    q = _rand(rng, (B, L, Hq, D), qscale)
    kb, vb = _rand(rng, (B, L, Hkv, D)), _rand(rng, (B, L, Hkv, D))
    ks = [_rand(rng, (B, L, Hkv, D)) for _ in range(j)]
    vs = [_rand(rng, (B, L, Hkv, D)) for _ in range(j)]
    do = _rand(rng, (B, L, Hq, D))
    if lens is None:
        lens = np.full(B, L, dtype=np.int32)
    return q, kb, vb, ks, vs, do, np.asarray(lens, dtype=np.int32)


def _structural_mask(L, T, j):
    base = np.tril(np.ones((L, L), dtype=bool))
    base[:, T:] = False
    blocks = [base]
    for _ in range(j):
        d = np.eye(L, dtype=bool)
        d[T:, :] = False
        blocks.append(d)
    return np.concatenate(blocks, axis=1)


def _sdpa(q, kb, vb, ks, vs, lens, scale, do=None):
    """torch SDPA float64 on CPU over KVcat with a structural boolean mask."""
    B, L, Hq, D = q.shape
    Hkv = kb.shape[2]
    G = Hq // Hkv
    kcat = np.concatenate([kb] + list(ks), axis=1)  # [B,(j+1)L,Hkv,D]
    vcat = np.concatenate([vb] + list(vs), axis=1)
    tq = torch.tensor(q, dtype=torch.float64).permute(0, 2, 1, 3).requires_grad_(True)
    tk = torch.tensor(kcat, dtype=torch.float64).permute(0, 2, 1, 3).requires_grad_(True)
    tv = torch.tensor(vcat, dtype=torch.float64).permute(0, 2, 1, 3).requires_grad_(True)
    # GQA by explicit repetition: q head h reads kv head h // G
    tk_r = tk.repeat_interleave(G, dim=1)
    tv_r = tv.repeat_interleave(G, dim=1)
    j = len(ks)
    m = torch.stack([torch.tensor(_structural_mask(L, int(lens[b]), j)) for b in range(B)])[:, None]
    out = F.scaled_dot_product_attention(tq, tk_r, tv_r, attn_mask=m, scale=scale)
    logits = (tq @ tk_r.transpose(-1, -2)) * scale
    lse = torch.logsumexp(logits.masked_fill(~m, -math.inf), dim=-1)
    res = {"out": out.permute(0, 2, 1, 3).detach().numpy(), "lse": lse.detach().numpy()}
    if do is not None:
        out.backward(torch.tensor(do, dtype=torch.float64).permute(0, 2, 1, 3))
        dk = tk.grad.permute(0, 2, 1, 3).numpy()
        dv = tv.grad.permute(0, 2, 1, 3).numpy()
        res["dq"] = tq.grad.permute(0, 2, 1, 3).numpy()
        res["dk_base"] = dk[:, :L]
        res["dv_base"] = dv[:, :L]
        res["dk_steps"] = [dk[:, (i + 1) * L:(i + 2) * L] for i in range(j)]
        res["dv_steps"] = [dv[:, (i + 1) * L:(i + 2) * L] for i in range(j)]
    return res


CASES = [
    dict(B=1, L=8, Hq=2, Hkv=2, D=4, j=0),
    dict(B=2, L=12, Hq=4, Hkv=2, D=8, j=2, lens=[12, 7]),
    dict(B=2, L=16, Hq=6, Hkv=2, D=16, j=5, lens=[3, 16]),
    dict(B=1, L=9, Hq=4, Hkv=1, D=8, j=8, lens=[1]),
]


@pytest.mark.parametrize("cfg", CASES)
def test_fwd_matches_torch_sdpa_fp64(cfg):
    q, kb, vb, ks, vs, do, lens = _case(**cfg)
    c = 1.0 / math.sqrt(q.shape[-1])
    out, lse = oracle.fwd(q, kb, vb, ks, vs, seq_lens=lens, nthreads=3)
    ref = _sdpa(q, kb, vb, ks, vs, lens, c)
    np.testing.assert_allclose(out, ref["out"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(lse, ref["lse"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("cfg", CASES)
def test_bwd_matches_torch_autograd_fp64(cfg):
    q, kb, vb, ks, vs, do, lens = _case(**cfg)
    c = 1.0 / math.sqrt(q.shape[-1])
    g = oracle.bwd(q, kb, vb, ks, vs, do, seq_lens=lens, nthreads=2)
    ref = _sdpa(q, kb, vb, ks, vs, lens, c, do=do)
    for key in ("dq", "dk_base", "dv_base"):
        np.testing.assert_allclose(g[key], ref[key], rtol=0, atol=1e-11, err_msg=key)
    for i in range(len(ks)):
        np.testing.assert_allclose(g["dk_steps"][i], ref["dk_steps"][i], rtol=0, atol=1e-11)
        np.testing.assert_allclose(g["dv_steps"][i], ref["dv_steps"][i], rtol=0, atol=1e-11)


def test_step0_is_textbook_causal_attention():
    """ttt_steps = 1 reduces to causal attention: SDPA(is_causal=True) and an
    independently coded lower-triangular loop."""
    q, kb, vb, ks, vs, do, lens = _case(B=2, L=10, Hq=2, Hkv=2, D=8, j=0, seed=3)
    c = 1.0 / math.sqrt(8)
    out, lse = oracle.fwd(q, kb, vb, [], [])
    tq = torch.tensor(q, dtype=torch.float64).permute(0, 2, 1, 3)
    tk = torch.tensor(kb, dtype=torch.float64).permute(0, 2, 1, 3)
    tv = torch.tensor(vb, dtype=torch.float64).permute(0, 2, 1, 3)
    ref = F.scaled_dot_product_attention(tq, tk, tv, is_causal=True, scale=c).permute(0, 2, 1, 3)
    np.testing.assert_allclose(out, ref.numpy(), atol=1e-12, rtol=0)
    # loop version
    B, L, H, D = q.shape
    for b in range(B):
        for h in range(H):
            for r in range(L):
                s = [c * float(np.dot(q[b, r, h].astype(np.float64), kb[b, k, h])) for k in range(r + 1)]
                mx = max(s)
                w = [math.exp(x - mx) for x in s]
                tot = sum(w)
                o = sum(w[k] / tot * vb[b, k, h].astype(np.float64) for k in range(r + 1))
                np.testing.assert_allclose(out[b, r, h], o, atol=1e-12)
                assert abs(lse[b, h, r] - (mx + math.log(tot))) < 1e-12


@pytest.mark.parametrize("cfg", CASES[1:])
def test_alg1_per_row_formulation(cfg):
    """Third formulation: Alg. 1 per row with T := r+1 prefix keys, t := T+j+1
    (reading R3): same output within 1e-12."""
    q, kb, vb, ks, vs, do, lens = _case(**cfg)
    c = 1.0 / math.sqrt(q.shape[-1])
    out, _ = oracle.fwd(q, kb, vb, ks, vs, seq_lens=lens)
    B, L, Hq, D = q.shape
    G = Hq // kb.shape[2]
    for b in range(B):
        T = int(lens[b])
        for h in range(Hq):
            g = h // G
            for r in range(L):
                if r < T:
                    o = oracle.alg1_row(q[b, r, h], kb[b, :r + 1, g], vb[b, :r + 1, g],
                                        [k[b, r, g] for k in ks], [v[b, r, g] for v in vs], c)
                else:  # padded row: all valid base keys, no step key (Alg. 2 verbatim)
                    o = oracle.alg1_row(q[b, r, h], kb[b, :T, g], vb[b, :T, g], [], [], c)
                np.testing.assert_allclose(out[b, r, h], o, atol=1e-12, rtol=0)


def test_zero_query_closed_form():
    """q = 0: all allowed logits equal -> out = mean of allowed V rows and
    lse = ln |A(r,j)| with |A| = r+1+j (r < T) else T."""
    B, L, Hq, Hkv, D, j = 2, 11, 4, 2, 8, 3
    _, kb, vb, ks, vs, _, _ = _case(B=B, L=L, Hq=Hq, Hkv=Hkv, D=D, j=j, seed=5)
    q = np.zeros((B, L, Hq, D), np.float32)
    lens = np.array([11, 6], np.int32)
    out, lse = oracle.fwd(q, kb, vb, ks, vs, seq_lens=lens)
    G = Hq // Hkv
    for b in range(B):
        T = int(lens[b])
        for h in range(Hq):
            g = h // G
            for r in range(L):
                if r < T:
                    rows = [vb[b, k, g] for k in range(r + 1)] + [v[b, r, g] for v in vs]
                    n = r + 1 + j
                else:
                    rows = [vb[b, k, g] for k in range(T)]
                    n = T
                np.testing.assert_allclose(out[b, r, h], np.mean(np.asarray(rows, np.float64), 0), atol=1e-12)
                assert abs(lse[b, h, r] - math.log(n)) < 1e-12


def test_single_allowed_key():
    """r = 0 at step 0 sees only key 0: out = v_0, lse = c q_0.k_0."""
    q, kb, vb, ks, vs, do, lens = _case(B=1, L=5, Hq=2, Hkv=1, D=8, j=0, seed=9)
    c = 1.0 / math.sqrt(8)
    out, lse = oracle.fwd(q, kb, vb, [], [])
    for h in range(2):
        np.testing.assert_allclose(out[0, 0, h], vb[0, 0, 0], atol=1e-15)
        assert abs(lse[0, h, 0] - c * np.dot(q[0, 0, h].astype(np.float64), kb[0, 0, 0])) < 1e-12
    # T = 1 and padded rows: every row sees exactly key 0 (+ its own step keys if r < 1)
    out, _ = oracle.fwd(q, kb, vb, [], [], seq_lens=[1])
    for r in range(5):
        np.testing.assert_allclose(out[0, r, 0], vb[0, 0, 0], atol=1e-15)


def test_convex_hull_and_masked_inertness():
    """out lies in the convex hull of allowed V; disallowed K/V
    are inert."""
    q, kb, vb, ks, vs, do, lens = _case(B=1, L=16, Hq=2, Hkv=1, D=8, j=3, lens=[10], seed=11, qscale=4.0)
    out, lse = oracle.fwd(q, kb, vb, ks, vs, seq_lens=lens)
    m = oracle.mask_dense(16, 10, 3)
    vcat = np.concatenate([vb] + vs, axis=1)[0, :, 0]  # [(j+1)L, D]
    for r in range(16):
        allowed = vcat[m[r]]
        assert np.all(out[0, r, 0] <= allowed.max(0) + 1e-12)
        assert np.all(out[0, r, 0] >= allowed.min(0) - 1e-12)
    # poison every disallowed key/value position (finite, large)
    kb2, vb2 = kb.copy(), vb.copy()
    ks2, vs2 = [k.copy() for k in ks], [v.copy() for v in vs]
    kb2[0, 10:] = 3e4; vb2[0, 10:] = -3e4
    for k2, v2 in zip(ks2, vs2):
        k2[0, 10:] = 3e4; v2[0, 10:] = 3e4
    out2, lse2 = oracle.fwd(q, kb2, vb2, ks2, vs2, seq_lens=lens)
    np.testing.assert_array_equal(out2, out)
    np.testing.assert_array_equal(lse2, lse)


def test_gqa_equals_mha_with_repeated_kv():
    q, kb, vb, ks, vs, do, lens = _case(B=1, L=10, Hq=6, Hkv=2, D=8, j=2, lens=[8], seed=13)
    G = 3
    rep = lambda a: np.repeat(a, G, axis=2)
    out_g, lse_g = oracle.fwd(q, kb, vb, ks, vs, seq_lens=lens)
    out_m, lse_m = oracle.fwd(q, rep(kb), rep(vb), [rep(k) for k in ks], [rep(v) for v in vs], seq_lens=lens)
    np.testing.assert_array_equal(out_g, out_m)
    np.testing.assert_array_equal(lse_g, lse_m)
    gg = oracle.bwd(q, kb, vb, ks, vs, do, seq_lens=lens)
    gm = oracle.bwd(q, rep(kb), rep(vb), [rep(k) for k in ks], [rep(v) for v in vs], do, seq_lens=lens)
    np.testing.assert_allclose(gg["dq"], gm["dq"], atol=1e-14)
    summ = lambda a: a.reshape(a.shape[0], a.shape[1], 2, G, a.shape[3]).sum(3)
    np.testing.assert_allclose(gg["dk_base"], summ(gm["dk_base"]), atol=1e-13)
    np.testing.assert_allclose(gg["dv_base"], summ(gm["dv_base"]), atol=1e-13)
    for i in range(2):
        np.testing.assert_allclose(gg["dk_steps"][i], summ(gm["dk_steps"][i]), atol=1e-13)
        np.testing.assert_allclose(gg["dv_steps"][i], summ(gm["dv_steps"][i]), atol=1e-13)


def test_finite_differences_all_inputs():
    """Central differences in fp64, every input tensor incl.
    the step lists. Loss = sum(out * W) so dL/dout = W."""
    B, L, Hq, Hkv, D, j = 1, 6, 2, 1, 4, 2
    q, kb, vb, ks, vs, W, lens = _case(B=B, L=L, Hq=Hq, Hkv=Hkv, D=D, j=j, lens=[5], seed=17)
    # FD needs float64 perturbations; the oracle takes fp32 inputs, so use
    # inputs exactly representable after perturbation: perturb in fp32 with h
    # and difference in fp64 (h = 2^-10 keeps x +- h exact in fp32 for |x| < 8).
    h = 2.0 ** -10
    g = oracle.bwd(q, kb, vb, ks, vs, W, seq_lens=lens)

    def loss(q_, kb_, vb_, ks_, vs_):
        out, _ = oracle.fwd(q_, kb_, vb_, ks_, vs_, seq_lens=lens)
        return float(np.sum(out * W.astype(np.float64)))

    def check(arr, grad, setter, n=6):
        rng = np.random.default_rng(1)
        idxs = [tuple(rng.integers(0, s) for s in arr.shape) for _ in range(n)]
        for idx in idxs:
            a_p, a_m = arr.copy(), arr.copy()
            a_p[idx] += np.float32(h); a_m[idx] -= np.float32(h)
            fd = (setter(a_p) - setter(a_m)) / (float(a_p[idx]) - float(a_m[idx]))
            # O(h^2) truncation: |f'''| h^2 / 6 is well under 1e-5 here
            assert abs(fd - grad[idx]) <= 1e-5 * max(1.0, abs(grad[idx])), (idx, fd, grad[idx])

    check(q, g["dq"], lambda a: loss(a, kb, vb, ks, vs))
    check(kb, g["dk_base"], lambda a: loss(q, a, vb, ks, vs))
    check(vb, g["dv_base"], lambda a: loss(q, kb, a, ks, vs))
    for i in range(j):
        check(ks[i], g["dk_steps"][i], lambda a, i=i: loss(q, kb, vb, ks[:i] + [a] + ks[i + 1:], vs))
        check(vs[i], g["dv_steps"][i], lambda a, i=i: loss(q, kb, vb, ks, vs[:i] + [a] + vs[i + 1:]))


@pytest.mark.parametrize("cfg", CASES[1:])
def test_exact_gradient_identities(cfg):
    """Per (b, kv group g), exact in exact arithmetic (≤1e-10 in fp64):
    (i)   sum over all keys of dK_g = 0  (shift invariance of each row's softmax)
    (ii)  sum over all keys of dV_g = sum_{h in g, r} dO_{h,r}   (rows of P sum to 1)
    (iii) sum_{h in g, r} q_{h,r} . dq_{h,r} = sum_k K_g[k] . dK_g[k] (bilinearity)."""
    q, kb, vb, ks, vs, do, lens = _case(**cfg)
    g = oracle.bwd(q, kb, vb, ks, vs, do, seq_lens=lens)
    B, L, Hq, D = q.shape
    Hkv = kb.shape[2]
    G = Hq // Hkv
    dk_all = np.concatenate([g["dk_base"]] + g["dk_steps"], axis=1)
    dv_all = np.concatenate([g["dv_base"]] + g["dv_steps"], axis=1)
    k_all = np.concatenate([kb] + ks, axis=1).astype(np.float64)
    for b in range(B):
        for kv in range(Hkv):
            hs = slice(kv * G, (kv + 1) * G)
            np.testing.assert_allclose(dk_all[b, :, kv].sum(0), 0.0, atol=1e-10)
            np.testing.assert_allclose(dv_all[b, :, kv].sum(0),
                                       do[b, :, hs].astype(np.float64).sum((0, 1)), atol=1e-10)
            lhs = float(np.sum(q[b, :, hs].astype(np.float64) * g["dq"][b, :, hs]))
            rhs = float(np.sum(k_all[b, :, kv] * dk_all[b, :, kv]))
            assert abs(lhs - rhs) < 1e-10


def test_row_subset_reduction():
    """Row selection (used for full-size parity): forward rows equal the full
    run; backward with dO zero off the selection equals the full gradient."""
    q, kb, vb, ks, vs, do, lens = _case(B=2, L=16, Hq=4, Hkv=2, D=8, j=3, lens=[16, 9], seed=21)
    rng = np.random.default_rng(0)
    sel = rng.random((2, 4, 16)) < 0.3
    out_full, lse_full = oracle.fwd(q, kb, vb, ks, vs, seq_lens=lens)
    out_s, lse_s = oracle.fwd(q, kb, vb, ks, vs, seq_lens=lens, row_sel=sel)
    selq = sel.transpose(0, 2, 1)  # [B,L,Hq]
    np.testing.assert_array_equal(out_s[selq], out_full[selq])
    np.testing.assert_array_equal(lse_s[sel], lse_full[sel])
    do_z = do * selq[..., None]
    g_full = oracle.bwd(q, kb, vb, ks, vs, do_z, seq_lens=lens)
    g_sub = oracle.bwd(q, kb, vb, ks, vs, do_z, seq_lens=lens, row_sel=sel)
    for key in ("dk_base", "dv_base"):
        np.testing.assert_allclose(g_sub[key], g_full[key], atol=1e-13)
    for i in range(3):
        np.testing.assert_allclose(g_sub["dk_steps"][i], g_full["dk_steps"][i], atol=1e-13)
    np.testing.assert_allclose(g_sub["dq"][selq], g_full["dq"][selq], atol=1e-13)


def test_degenerate_length_rejected():
    q, kb, vb, ks, vs, do, lens = _case(B=1, L=4, Hq=1, Hkv=1, D=4, j=1)
    with pytest.raises(ValueError):
        oracle.fwd(q, kb, vb, ks, vs, seq_lens=[0])


def test_thread_count_invariance():
    q, kb, vb, ks, vs, do, lens = _case(B=3, L=8, Hq=4, Hkv=2, D=8, j=2, lens=[8, 3, 5], seed=23)
    a = oracle.bwd(q, kb, vb, ks, vs, do, seq_lens=lens, nthreads=1)
    b = oracle.bwd(q, kb, vb, ks, vs, do, seq_lens=lens, nthreads=5)
    for key in ("dq", "dk_base", "dv_base"):
        np.testing.assert_array_equal(a[key], b[key])
