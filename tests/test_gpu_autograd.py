"""GPU: the torch.autograd wrappers (paper_2603_18567_b200/autograd.py) against the fp64
oracle — an unroll of S TTT steps sharing K_0 / V_0 / the step lists, where autograd sums
the per-step contributions, and the soft-label loss whose backward is Alg. 3 in place."""
import numpy as np
import pytest
import torch

import oracle
from oracle import loss as OL
from paper_2603_18567_b200.autograd import soft_label_loss, ttt_attention, ttt_attention_unroll
from paper_2603_18567_b200.inputs import Shape, make_case, make_loss_case
from tests.gpu_helpers import TOL_BF16, assert_close, assert_close_sum, np32, oracle_inputs

pytestmark = pytest.mark.gpu


def test_autograd_ttt_unroll_bf16(cuda_ok):
    shape = Shape(1, 256, 8, 2, 128, 3)
    case = make_case(shape, dtype=torch.bfloat16, seed=7, lens="ragged")
    dev = lambda t: t.cuda().contiguous().requires_grad_(True)
    qs = [dev(x) for x in case.q]
    kb, vb = dev(case.k_base), dev(case.v_base)
    ks, vs = [dev(x) for x in case.k_steps], [dev(x) for x in case.v_steps]
    lens = [int(x) for x in case.seq_lens]
    S = shape.ttt_steps
    total = 0
    for j in range(S):
        out = ttt_attention(qs[j], kb, vb, ks, vs, j, seq_lens=lens)
        total = total + (out.float() * case.dout[j].cuda().float()).sum()   # dL/dout_j = dout_j
    total.backward()
    parts = {"k": [], "v": [], "ks": [[] for _ in range(S - 1)], "vs": [[] for _ in range(S - 1)]}
    for j in range(S):
        og = oracle.bwd(*oracle_inputs(case, j), np32(case.dout[j]), seq_lens=case.seq_lens)
        assert_close(f"autograd dq_{j}", np32(qs[j].grad), og["dq"], **TOL_BF16)
        parts["k"].append(og["dk_base"])
        parts["v"].append(og["dv_base"])
        for i in range(j):
            parts["ks"][i].append(og["dk_steps"][i])
            parts["vs"][i].append(og["dv_steps"][i])
    # autograd sums bf16 per-step gradients: each part's bound plus one bf16 rounding of the sum
    tol = dict(atol=TOL_BF16["atol"] * 1.5, rtol=TOL_BF16["rtol"] * 1.5)
    assert_close_sum("autograd dk_base", np32(kb.grad), parts["k"], **tol)
    assert_close_sum("autograd dv_base", np32(vb.grad), parts["v"], **tol)
    for i in range(S - 1):
        assert_close_sum(f"autograd dk_{i+1}", np32(ks[i].grad), parts["ks"][i], **tol)
        assert_close_sum(f"autograd dv_{i+1}", np32(vs[i].grad), parts["vs"][i], **tol)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_autograd_soft_label_loss_inplace(cuda_ok, dtype):
    case = make_loss_case(40, 3000, dtype, seed=9)
    z0 = case.z.cuda().requires_grad_(True)
    z = z0 * 1.0                         # non-leaf logits (as out of an lm head); Alg. 3 overwrites z
    ptr = z.data_ptr()
    loss = soft_label_loss(z, case.p.cuda(), case.mask.cuda())
    loss.backward(torch.tensor(0.5, device="cuda"))
    zf, pf, mk = case.z.double().numpy(), case.p.double().numpy(), case.mask.numpy().astype(bool)
    L = OL.loss_forward(zf, pf, mk)[0]
    assert abs(loss.item() - L) <= 1e-5 * abs(L) + 1e-5
    ref = OL.loss_backward(zf, pf, mk, g_scale=0.5)
    got = z0.grad.double().cpu().numpy()
    rtol = 1e-5 if dtype == torch.float32 else 2.0 ** -8
    pi = OL.softmax_rows(zf)
    g = OL.upstream_g(40, mk, 0.5)
    s = pf.sum(1) * g
    atol = 1e-5 * (pi * np.abs(s)[:, None] + pf * np.abs(g)[:, None]) + 2.0 ** -120
    err = np.abs(got - ref)
    assert (err <= rtol * np.abs(ref) + atol).all(), err.max()
    assert z.data_ptr() == ptr and torch.equal(z.detach(), z0.grad.to(dtype))  # the gradient lives in z's buffer


def test_autograd_unroll_matches_oracle_and_per_step(cuda_ok):
    """ttt_attention_unroll (one autograd node, backward = ttt_attn_bwd_unroll with fp32
    accumulation) vs the oracle summed over steps, and vs the per-step wrapper."""
    shape = Shape(1, 256, 8, 2, 128, 3)
    case = make_case(shape, dtype=torch.bfloat16, seed=8, lens="ragged")
    dev = lambda t: t.cuda().contiguous().requires_grad_(True)
    qs = [dev(x) for x in case.q]
    kb, vb = dev(case.k_base), dev(case.v_base)
    ks, vs = [dev(x) for x in case.k_steps], [dev(x) for x in case.v_steps]
    lens = [int(x) for x in case.seq_lens]
    S = shape.ttt_steps
    outs = ttt_attention_unroll(qs, kb, vb, ks, vs, seq_lens=lens)
    total = sum((outs[j].float() * case.dout[j].cuda().float()).sum() for j in range(S))
    total.backward()
    parts = {"k": [], "v": [], "ks": [[] for _ in range(S - 1)], "vs": [[] for _ in range(S - 1)]}
    for j in range(S):
        og = oracle.bwd(*oracle_inputs(case, j), np32(case.dout[j]), seq_lens=case.seq_lens)
        assert_close(f"unroll-autograd dq_{j}", np32(qs[j].grad), og["dq"], **TOL_BF16)
        parts["k"].append(og["dk_base"])
        parts["v"].append(og["dv_base"])
        for i in range(j):
            parts["ks"][i].append(og["dk_steps"][i])
            parts["vs"][i].append(og["dv_steps"][i])
    tol = dict(atol=TOL_BF16["atol"] * 1.5, rtol=TOL_BF16["rtol"] * 1.5)  # + one bf16 rounding of the sum
    assert_close_sum("unroll-autograd dk_base", np32(kb.grad), parts["k"], **tol)
    assert_close_sum("unroll-autograd dv_base", np32(vb.grad), parts["v"], **tol)
    for i in range(S - 1):
        assert_close_sum(f"unroll-autograd dk_{i+1}", np32(ks[i].grad), parts["ks"][i], **tol)
        assert_close_sum(f"unroll-autograd dv_{i+1}", np32(vs[i].grad), parts["vs"][i], **tol)
