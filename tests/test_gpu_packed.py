"""GPU parity of PACKED batches (include/ttt_attn.h cu_seqlens): sequences
laid back to back with no padding rows, through the same tcgen05 / fp32-check kernels, against the
oracle's packed functions (oracle.fwd_packed / bwd_packed, pinned in tests/test_oracle_packed.py).

Length mixes cover T_b = 1, tile-aligned ends (128, 256), sequences whose last tile is partial and
straddles the next sequence's first rows (127, 129, 300), and several sequences inside one 128-row
span. Also: the packed forward equals the padded forward of the same sequences bit for bit (the
tiles hold the same rows), the backward's accumulate semantics and the whole-unroll call."""
import numpy as np
import pytest
import torch

import oracle
import paper_2603_18567_b200 as ttt
from paper_2603_18567_b200.inputs import make_packed_case, packed_lens
from tests.gpu_helpers import TOL_BF16, TOL_FP32, assert_close, assert_close_sum, np32

pytestmark = pytest.mark.gpu

MIXES = {
    "mixed": [1, 127, 128, 129, 300, 64, 5, 256],
    "short": [3, 1, 7, 2, 40, 1],
    "one": [777],
}


class Packed:
    def __init__(self, case, dev="cuda"):
        self.c = case
        to = lambda t: t.to(dev).contiguous()
        self.q = [to(x) for x in case.q]
        self.dout = [to(x) for x in case.dout]
        self.k, self.v = to(case.k_base), to(case.v_base)
        self.ks = [to(x) for x in case.k_steps]
        self.vs = [to(x) for x in case.v_steps]
        dt = ttt.TTT_FP32_CHECK if case.dtype == torch.float32 else ttt.TTT_BF16
        self.desc = ttt.packed_desc(case.cu, case.num_q_heads, case.num_kv_heads, case.head_dim, dtype=dt)
        self.dev = dev

    def fwd(self, j):
        c = self.c
        out = torch.empty_like(self.q[j])
        lse = torch.full((c.num_q_heads, c.rows), float("nan"), dtype=torch.float32, device=self.dev)
        self.lo = torch.empty_like(out) if c.dtype == torch.bfloat16 else None
        ttt.ttt_attn_fwd(self.desc, j, self.q[j], self.k, self.v, self.ks, self.vs, out, lse, out_lo=self.lo)
        return out, lse

    def grads(self, n, fill=0.0):
        c = self.c
        z = lambda: torch.full((c.rows, c.num_kv_heads, c.head_dim), fill, dtype=torch.float32, device=self.dev)
        return {"dk_base": z(), "dv_base": z(), "dk_steps": [z() for _ in range(n)], "dv_steps": [z() for _ in range(n)]}

    def bwd(self, j, out, lse, g, accumulate=False):
        dq = torch.empty_like(self.q[j])
        ws = torch.empty(max(ttt.ttt_attn_workspace_size(self.desc, j, True), 16), dtype=torch.uint8, device=self.dev)
        ws.fill_(0xFF)  # NaN bytes: every workspace value the kernels read must have been written
        ttt.ttt_attn_bwd(self.desc, j, self.q[j], self.k, self.v, self.ks, self.vs, out, lse, self.dout[j], dq,
                         g["dk_base"], g["dv_base"], g["dk_steps"], g["dv_steps"],
                         flags=ttt.TTT_ACCUMULATE_DKV if accumulate else 0, workspace=ws, out_lo=self.lo)
        return dq


def _oracle_in(c, j):
    return (np32(c.q[j]), np32(c.k_base), np32(c.v_base), [np32(x) for x in c.k_steps[:j]],
            [np32(x) for x in c.v_steps[:j]])


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32], ids=["bf16", "fp32check"])
@pytest.mark.parametrize("mix", list(MIXES), ids=list(MIXES))
@pytest.mark.parametrize("heads", [(8, 2, 128), (4, 4, 64), (16, 1, 128)], ids=["gqa4_d128", "mha_d64", "gqa16"])
def test_packed_fwd_bwd_vs_oracle(cuda_ok, dtype, mix, heads):
    Hq, Hkv, D = heads
    S = 3
    c = make_packed_case(MIXES[mix], Hq, Hkv, D, S, dtype=dtype, seed=11)
    pk = Packed(c)
    tol = TOL_FP32 if dtype == torch.float32 else TOL_BF16
    for j in reversed(range(S)):
        out, lse = pk.fwd(j)
        q, kb, vb, ks, vs = _oracle_in(c, j)
        o_out, o_lse = oracle.fwd_packed(q, kb, vb, ks, vs, c.cu)
        assert_close(f"{mix} out j={j}", np32(out), o_out, **tol)
        assert_close(f"{mix} lse j={j}", np32(lse), o_lse, **tol)
        g = pk.grads(S - 1, fill=123.0)  # overwrite mode: every element must be written
        dq = pk.bwd(j, out, lse, g)
        og = oracle.bwd_packed(q, kb, vb, ks, vs, np32(c.dout[j]), c.cu)
        assert_close(f"{mix} dq j={j}", np32(dq), og["dq"], **tol)
        assert_close(f"{mix} dk_base j={j}", np32(g["dk_base"]), og["dk_base"], **tol)
        assert_close(f"{mix} dv_base j={j}", np32(g["dv_base"]), og["dv_base"], **tol)
        for i in range(j):
            assert_close(f"{mix} dk_{i + 1} j={j}", np32(g["dk_steps"][i]), og["dk_steps"][i], **tol)
            assert_close(f"{mix} dv_{i + 1} j={j}", np32(g["dv_steps"][i]), og["dv_steps"][i], **tol)


def test_packed_fwd_bitwise_equals_padded(cuda_ok):
    """The packed tiles hold the same rows as the padded tiles of each sequence, so out / lse of the
    valid rows are bit-identical (masked keys contribute exact zeros either way)."""
    lens = [1, 127, 128, 129, 300, 64]
    Hq, Hkv, D, j = 8, 2, 128, 3
    c = make_packed_case(lens, Hq, Hkv, D, j + 1, seed=5)
    pk = Packed(c)
    out_p, lse_p = pk.fwd(j)
    L = 384
    B = len(lens)

    def pad(x):
        y = torch.zeros((B, L) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        for b in range(B):
            y[b, :lens[b]] = x[c.cu[b]:c.cu[b + 1]]
        return y
    q, k, v = pad(pk.q[j]), pad(pk.k), pad(pk.v)
    ks, vs = [pad(x) for x in pk.ks], [pad(x) for x in pk.vs]
    d = ttt.desc_for(q, k, seq_lens=lens)
    out_d = torch.empty_like(q)
    lse_d = torch.empty((B, Hq, L), dtype=torch.float32, device="cuda")
    lo_d = torch.empty_like(q)
    ttt.ttt_attn_fwd(d, j, q, k, v, ks, vs, out_d, lse_d, out_lo=lo_d)
    for b in range(B):
        r0, T = int(c.cu[b]), lens[b]
        assert torch.equal(out_p[r0:r0 + T], out_d[b, :T]), f"seq {b}: out differs"
        assert torch.equal(lse_p[:, r0:r0 + T], lse_d[b, :, :T]), f"seq {b}: lse differs"
        assert torch.equal(pk.lo[r0:r0 + T], lo_d[b, :T]), f"seq {b}: out_lo differs"


def test_packed_accumulate_and_unroll(cuda_ok):
    """S reverse-order calls with TTT_ACCUMULATE_DKV after the first == the oracle's sums; the
    whole-unroll call gives the same dq bit for bit and the same accumulators up to fp32 order."""
    lens = [200, 1, 129, 333]
    Hq, Hkv, D, S = 8, 2, 128, 4
    c = make_packed_case(lens, Hq, Hkv, D, S, seed=7)
    pk = Packed(c)
    fw = {j: pk.fwd(j) + (pk.lo,) for j in range(S)}
    acc = pk.grads(S - 1)
    dqs, parts = {}, {"dk_base": [], "dv_base": []}
    for j in reversed(range(S)):
        out, lse, lo = fw[j]
        pk.lo = lo
        dqs[j] = pk.bwd(j, out, lse, acc, accumulate=(j != S - 1))
        og = oracle.bwd_packed(*_oracle_in(c, j), np32(c.dout[j]), c.cu)
        parts["dk_base"].append(og["dk_base"])
        parts["dv_base"].append(og["dv_base"])
    assert_close_sum("packed dk_base acc", np32(acc["dk_base"]), parts["dk_base"], **TOL_BF16)
    assert_close_sum("packed dv_base acc", np32(acc["dv_base"]), parts["dv_base"], **TOL_BF16)
    u = pk.grads(S - 1)
    dq_u = [torch.empty_like(pk.q[j]) for j in range(S)]
    ws = torch.empty(ttt.ttt_attn_bwd_unroll_workspace_size(pk.desc, S), dtype=torch.uint8, device="cuda")
    ttt.ttt_attn_bwd_unroll(pk.desc, pk.q, pk.k, pk.v, pk.ks, pk.vs, [fw[j][0] for j in range(S)],
                            [fw[j][1] for j in range(S)], pk.dout, dq_u, u["dk_base"], u["dv_base"],
                            u["dk_steps"], u["dv_steps"], workspace=ws, out_lo=[fw[j][2] for j in range(S)])
    for j in range(S):
        assert torch.equal(dq_u[j], dqs[j]), f"unroll dq[{j}] differs from the per-call dq"
    for key in ("dk_base", "dv_base"):
        np.testing.assert_allclose(np32(u[key]), np32(acc[key]), rtol=1e-5, atol=1e-5)
    for i in range(S - 1):
        np.testing.assert_allclose(np32(u["dk_steps"][i]), np32(acc["dk_steps"][i]), rtol=1e-5, atol=1e-5)


def test_packed_llama_heads_sampled_rows(cuda_ok):
    """Llama-3.1-8B draft heads (32 / 8, D = 128) over 16 sequences with the paper's length mix
    (T_b ~ U[512, 2048], ~20k rows), step j = 6: out / lse of every row of four sequences vs the
    oracle (the oracle runs those sequences alone — packing makes them independent problems)."""
    lens = packed_lens(16, 2048, seed=3)
    Hq, Hkv, D, j = 32, 8, 128, 6
    c = make_packed_case(lens, Hq, Hkv, D, j + 1, seed=3)
    pk = Packed(c)
    out, lse = pk.fwd(j)
    for b in (0, 5, 9, 15):
        r0, r1 = int(c.cu[b]), int(c.cu[b + 1])
        sl = lambda x: np32(x[r0:r1])
        o_out, o_lse = oracle.fwd_packed(sl(c.q[j]), sl(c.k_base), sl(c.v_base), [sl(x) for x in c.k_steps[:j]],
                                         [sl(x) for x in c.v_steps[:j]], [0, r1 - r0])
        assert_close(f"seq {b} out", np32(out[r0:r1]), o_out, **TOL_BF16)
        assert_close(f"seq {b} lse", np32(lse[:, r0:r1]), o_lse, **TOL_BF16)
    assert not torch.isnan(lse).any(), "every lse row of every sequence must be written"


def test_packed_autograd(cuda_ok):
    """autograd.ttt_attention(..., cu_seqlens=...) over a packed batch: loss = sum(out * w) and its
    gradients w.r.t. q and every K / V against the packed oracle's backward with dO = w."""
    from paper_2603_18567_b200.autograd import ttt_attention
    lens = [70, 1, 200]
    Hq, Hkv, D, j = 4, 2, 64, 2
    c = make_packed_case(lens, Hq, Hkv, D, j + 1, seed=9)
    leaf = lambda t: t.cuda().clone().requires_grad_(True)
    q, k, v = leaf(c.q[j]), leaf(c.k_base), leaf(c.v_base)
    ks, vs = [leaf(x) for x in c.k_steps], [leaf(x) for x in c.v_steps]
    w = c.dout[j].cuda()
    out = ttt_attention(q, k, v, ks, vs, j, cu_seqlens=c.cu)
    (out.float() * w.float()).sum().backward()
    og = oracle.bwd_packed(*_oracle_in(c, j), np32(c.dout[j]), c.cu)
    o_out, _ = oracle.fwd_packed(*_oracle_in(c, j), c.cu)
    assert_close("autograd packed out", np32(out), o_out, **TOL_BF16)
    assert_close("autograd packed dq", np32(q.grad), og["dq"], **TOL_BF16)
    assert_close("autograd packed dk", np32(k.grad), og["dk_base"], **TOL_BF16)
    assert_close("autograd packed dv", np32(v.grad), og["dv_base"], **TOL_BF16)
    for i in range(j):
        assert_close(f"autograd packed dk_{i + 1}", np32(ks[i].grad), og["dk_steps"][i], **TOL_BF16)
        assert_close(f"autograd packed dv_{i + 1}", np32(vs[i].grad), og["dv_steps"][i], **TOL_BF16)
