"""GPU parity at long TTT unrolls: the paper varies the TTT length from 1 to 17
(Fig. "TTT length"), i.e. steps j = 0..16 with up to 16 diagonal
step keys per row. bf16 (tensor-core path, north_star 2e-2 / 1e-2) and the fp32
check path (1e-5), small L element by element, and the Llama-3.1-8B draft shape
at j = 16 on sampled rows (row-subset reduction)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2603_18567_b200.inputs import CONFIGS, Shape, make_case, sample_rows
from tests.gpu_helpers import TOL_BF16, TOL_FP32, DeviceCase, assert_close, np32, oracle_inputs

pytestmark = pytest.mark.gpu


def _check_step(name, dc, case, j, tol, grads_acc=None):
    out, lse = dc.fwd(j)
    g = dc.alloc_grads(case.shape.ttt_steps - 1)
    dq = dc.bwd(j, out, lse, g, accumulate=False)
    if grads_acc is not None:
        dc.bwd(j, out, lse, grads_acc, accumulate=True)
    torch.cuda.synchronize()
    o_out, o_lse = oracle.fwd(*oracle_inputs(case, j), seq_lens=case.seq_lens)
    assert_close(f"{name} out j={j}", np32(out), o_out, **tol)
    assert_close(f"{name} lse j={j}", np32(lse), o_lse, **tol)
    og = oracle.bwd(*oracle_inputs(case, j), np32(case.dout[j]), seq_lens=case.seq_lens)
    assert_close(f"{name} dq j={j}", np32(dq), og["dq"], **tol)
    assert_close(f"{name} dk_base j={j}", np32(g["dk_base"]), og["dk_base"], **tol)
    assert_close(f"{name} dv_base j={j}", np32(g["dv_base"]), og["dv_base"], **tol)
    for i in range(j):
        assert_close(f"{name} dk_{i + 1} j={j}", np32(g["dk_steps"][i]), og["dk_steps"][i], **tol)
        assert_close(f"{name} dv_{i + 1} j={j}", np32(g["dv_steps"][i]), og["dv_steps"][i], **tol)
    return g


@pytest.mark.parametrize("dtype,shape,tol", [
    (torch.bfloat16, Shape(1, 256, 8, 2, 128, 17), TOL_BF16),
    (torch.bfloat16, Shape(2, 384, 4, 4, 64, 17), TOL_BF16),
    (torch.float32, Shape(1, 128, 4, 2, 64, 17), TOL_FP32),
], ids=["bf16_g4_d128", "bf16_mha_d64", "fp32_check"])
def test_ttt_length_17_all_steps(cuda_ok, dtype, shape, tol):
    """Every step j = 16..0 of a 17-step unroll (reverse order, as training runs it): per-call
    outputs vs the oracle, and the accumulated dK / dV equal to the fp32 sum of the per-call
    (overwrite-mode) outputs — accumulation adds nothing but fp32 adds."""
    case = make_case(shape, dtype=dtype, seed=17, lens="ragged")
    dc = DeviceCase(case)
    acc = dc.alloc_grads(shape.ttt_steps - 1)
    total = dc.alloc_grads(shape.ttt_steps - 1)
    for j in reversed(range(shape.ttt_steps)):
        g = _check_step(f"S17 {dtype}", dc, case, j, tol, grads_acc=acc)
        total["dk_base"] += g["dk_base"]
        total["dv_base"] += g["dv_base"]
        for i in range(j):
            total["dk_steps"][i] += g["dk_steps"][i]
            total["dv_steps"][i] += g["dv_steps"][i]
    torch.cuda.synchronize()
    for key in ("dk_base", "dv_base"):
        torch.testing.assert_close(acc[key], total[key], rtol=1e-5, atol=1e-5)
    for i in range(shape.ttt_steps - 1):
        torch.testing.assert_close(acc["dk_steps"][i], total["dk_steps"][i], rtol=1e-5, atol=1e-5)
        torch.testing.assert_close(acc["dv_steps"][i], total["dv_steps"][i], rtol=1e-5, atol=1e-5)


@pytest.mark.slow
def test_ttt_length_17_llama_full_size_row_subset(cuda_ok):
    """Llama-3.1-8B draft shape (B = 8, L = 2048, 32 / 8 heads) at the last step of a 17-step
    unroll (j = 16: 16 diagonal keys per row), forward on sampled rows and backward with dO = 0
    off the sampled rows (every gradient is then exactly the sum over those rows)."""
    base = CONFIGS["llama8b"]
    shape = Shape(base.batch, base.seq_len, base.num_q_heads, base.num_kv_heads, base.head_dim, 17)
    case = make_case(shape, dtype=torch.bfloat16, seed=2, lens="full", steps=1)
    j = 16
    case.q = [case.q[0]] * shape.ttt_steps
    sel = sample_rows(shape, 4, seed=5)
    selq = sel.transpose(0, 2, 1)
    do = case.dout[0].clone()
    do[torch.from_numpy(~selq)] = 0
    case.dout = [do] * shape.ttt_steps
    dc = DeviceCase(case)
    out, lse = dc.fwd(j)
    g = dc.alloc_grads(j)
    dq = dc.bwd(j, out, lse, g, accumulate=False)
    torch.cuda.synchronize()
    o_out, o_lse = oracle.fwd(*oracle_inputs(case, j), seq_lens=case.seq_lens, row_sel=sel)
    assert_close("S17 llama out", np32(out)[selq], o_out[selq], **TOL_BF16)
    assert_close("S17 llama lse", np32(lse)[sel], o_lse[sel], **TOL_BF16)
    og = oracle.bwd(*oracle_inputs(case, j), np32(do), seq_lens=case.seq_lens, row_sel=sel)
    assert_close("S17 llama dq", np32(dq)[selq], og["dq"][selq], **TOL_BF16)
    assert_close("S17 llama dk_base", np32(g["dk_base"]), og["dk_base"], **TOL_BF16)
    assert_close("S17 llama dv_base", np32(g["dv_base"]), og["dv_base"], **TOL_BF16)
    for i in range(j):
        assert_close(f"S17 llama dk_{i + 1}", np32(g["dk_steps"][i]), og["dk_steps"][i], **TOL_BF16)
        assert_close(f"S17 llama dv_{i + 1}", np32(g["dv_steps"][i]), og["dv_steps"][i], **TOL_BF16)
    assert np.abs(np32(dq)[~selq]).max() == 0.0


@pytest.mark.parametrize("dtype,shape,tol", [
    (torch.bfloat16, Shape(1, 256, 8, 2, 128, 32), TOL_BF16),
    (torch.bfloat16, Shape(1, 256, 4, 4, 64, 32), TOL_BF16),
    (torch.float32, Shape(1, 128, 4, 2, 64, 32), TOL_FP32),
], ids=["bf16_g4_d128", "bf16_mha_d64", "fp32_check"])
def test_max_step_31(cuda_ok, dtype, shape, tol):
    """The ABI's largest step, j = TTT_MAX_STEPS - 1 = 31 (31 diagonal keys per row, every step-list
    slot of the parameter block and of the diagonal rings in use; an odd count, so the forward's
    diagonal warps end on a single-stage pass), plus j = 30, against the oracle with ragged lengths."""
    case = make_case(shape, dtype=dtype, seed=31, lens="ragged")
    dc = DeviceCase(case)
    for j in (31, 30):
        _check_step(f"S32 {dtype}", dc, case, j, tol)
