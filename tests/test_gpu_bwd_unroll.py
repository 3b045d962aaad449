"""GPU: ttt_attn_bwd_unroll (one call for the S backward calls of an unroll, include/ttt_attn.h)
equals the S ttt_attn_bwd calls j = S-1..0 it replaces — the step-list gradients bit for bit
(each row's contributions are added in the same order j = S-1..0 by one writer), dq and
dK_0 / dV_0 up to fp32 summation order (their tiles are reduce-added by several CTAs in a
run-dependent order, in either path) — and matches the fp64 oracle summed over steps."""
import numpy as np
import pytest
import torch

import oracle
import paper_2603_18567_b200 as ttt
from paper_2603_18567_b200.inputs import CONFIGS, Shape, make_case
from tests.gpu_helpers import TOL_BF16, DeviceCase, assert_close_sum, np32, oracle_inputs

pytestmark = pytest.mark.gpu


def _fwd_all(dc, S):
    outs, lses, los = [], [], []
    for j in range(S):
        o, l = dc.fwd(j)
        outs.append(o)
        lses.append(l)
        los.append(dc.out_lo)
    return outs, lses, los


def _run_both(dc, S, accumulate):
    outs, lses, los = _fwd_all(dc, S)
    s = dc.case.shape
    init = lambda: dc.alloc_grads(S - 1)
    a, b = init(), init()
    if accumulate:  # pre-existing accumulator contents must be added to, identically
        g = torch.Generator(device="cuda").manual_seed(3)
        for ta, tb in zip([a["dk_base"], a["dv_base"]] + a["dk_steps"] + a["dv_steps"],
                          [b["dk_base"], b["dv_base"]] + b["dk_steps"] + b["dv_steps"]):
            ta.copy_(torch.randn(ta.shape, device="cuda", generator=g))
            tb.copy_(ta)
    dq_a = []
    for j in reversed(range(S)):
        dc.out_lo = los[j]
        dq = dc.bwd(j, outs[j], lses[j], a, accumulate=(accumulate or j != S - 1))
        dq_a.insert(0, dq)
    dq_b = [torch.empty(s.q_shape, dtype=dc.dt, device="cuda") for _ in range(S)]
    ws = torch.empty(ttt.ttt_attn_bwd_unroll_workspace_size(dc.desc, S), dtype=torch.uint8, device="cuda")
    ttt.ttt_attn_bwd_unroll(dc.desc, dc.q[:S], dc.k, dc.v, dc.ks, dc.vs, outs, lses, dc.dout[:S], dq_b,
                            b["dk_base"], b["dv_base"], b["dk_steps"], b["dv_steps"],
                            flags=ttt.TTT_ACCUMULATE_DKV if accumulate else 0, workspace=ws,
                            out_lo=los if los[0] is not None else None)
    torch.cuda.synchronize()
    return dq_a, a, dq_b, b


def _assert_equivalent(name, S, dq_a, a, dq_b, b):
    for j in range(S):  # dq: the bf16 rounding of fp32 sums in run-dependent order (<= 1 ulp apart)
        torch.testing.assert_close(dq_b[j].float(), dq_a[j].float(), rtol=2.0 ** -7, atol=1e-5,
                                   msg=lambda m: f"{name} dq_{j}: {m}")
    for i in range(S - 1):
        assert torch.equal(a["dk_steps"][i], b["dk_steps"][i]), f"{name}: dk_{i+1} differs"
        assert torch.equal(a["dv_steps"][i], b["dv_steps"][i]), f"{name}: dv_{i+1} differs"
    for k in ("dk_base", "dv_base"):
        torch.testing.assert_close(b[k], a[k], rtol=1e-5, atol=1e-5, msg=lambda m: f"{name} {k}: {m}")


CASES = [
    ("tiny_ragged", CONFIGS["tiny"], "ragged"),
    ("L384_ragged", Shape(2, 384, 4, 2, 128, 4), "ragged"),
    ("gqa16", Shape(1, 512, 16, 1, 128, 3), "ragged"),
    ("d64_s5", Shape(1, 640, 8, 2, 64, 5), "ragged"),
    ("s1", Shape(1, 256, 4, 2, 128, 1), "full"),
    ("s8_max", Shape(1, 256, 4, 2, 128, 8), "ragged"),
]


@pytest.mark.parametrize("accumulate", [False, True])
@pytest.mark.parametrize("name,shape,lens", CASES, ids=[c[0] for c in CASES])
def test_bwd_unroll_equals_per_call(cuda_ok, name, shape, lens, accumulate):
    case = make_case(shape, dtype=torch.bfloat16, seed=2, lens=lens)
    dc = DeviceCase(case)
    _assert_equivalent(name, shape.ttt_steps, *_run_both(dc, shape.ttt_steps, accumulate))


def test_bwd_unroll_vs_oracle(cuda_ok):
    shape = Shape(2, 384, 8, 2, 128, 4)
    case = make_case(shape, dtype=torch.bfloat16, seed=4, lens="ragged")
    dc = DeviceCase(case)
    S = shape.ttt_steps
    dq_a, a, dq_b, b = _run_both(dc, S, False)
    parts = {"dk_base": [], "dv_base": [], "dk_steps": [[] for _ in range(S - 1)], "dv_steps": [[] for _ in range(S - 1)]}
    for j in range(S):
        og = oracle.bwd(*oracle_inputs(case, j), np32(case.dout[j]), seq_lens=case.seq_lens)
        assert_close_sum(f"unroll dq_{j}", np32(dq_b[j]), [og["dq"]], **TOL_BF16)
        parts["dk_base"].append(og["dk_base"])
        parts["dv_base"].append(og["dv_base"])
        for i in range(j):
            parts["dk_steps"][i].append(og["dk_steps"][i])
            parts["dv_steps"][i].append(og["dv_steps"][i])
    assert_close_sum("unroll dk_base", np32(b["dk_base"]), parts["dk_base"], **TOL_BF16)
    assert_close_sum("unroll dv_base", np32(b["dv_base"]), parts["dv_base"], **TOL_BF16)
    for i in range(S - 1):
        assert_close_sum(f"unroll dk_{i+1}", np32(b["dk_steps"][i]), parts["dk_steps"][i], **TOL_BF16)
        assert_close_sum(f"unroll dv_{i+1}", np32(b["dv_steps"][i]), parts["dv_steps"][i], **TOL_BF16)


@pytest.mark.slow
def test_bwd_unroll_full_size_llama_equals_per_call(cuda_ok):
    """bench.py's launch configuration (Llama-3.1-8B draft shape, 7 steps): bit-identical dq and
    step-list gradients to the per-call sequence (parity of that sequence is tested elsewhere)."""
    shape = CONFIGS["llama8b"]
    case = make_case(shape, dtype=torch.bfloat16, seed=0, lens="full")
    dc = DeviceCase(case)
    _assert_equivalent("llama8b", shape.ttt_steps, *_run_both(dc, shape.ttt_steps, False))


def test_bwd_unroll_fp32_check_mode(cuda_ok):
    """FP32_CHECK: ttt_attn_bwd_unroll runs the S per-call check kernels; vs the oracle at 1e-5."""
    from tests.gpu_helpers import TOL_FP32
    shape = Shape(1, 128, 4, 2, 64, 3)
    case = make_case(shape, dtype=torch.float32, seed=6, lens="ragged")
    dc = DeviceCase(case)
    S = shape.ttt_steps
    outs, lses = [], []
    for j in range(S):
        o, l = dc.fwd(j)
        outs.append(o)
        lses.append(l)
    g = dc.alloc_grads(S - 1)
    dqs = [torch.empty_like(dc.q[0]) for _ in range(S)]
    ws = torch.empty(ttt.ttt_attn_bwd_unroll_workspace_size(dc.desc, S), dtype=torch.uint8, device="cuda")
    ttt.ttt_attn_bwd_unroll(dc.desc, dc.q[:S], dc.k, dc.v, dc.ks, dc.vs, outs, lses, dc.dout[:S], dqs,
                            g["dk_base"], g["dv_base"], g["dk_steps"], g["dv_steps"], workspace=ws)
    torch.cuda.synchronize()
    parts = {"dk_base": [], "dv_base": []}
    for j in range(S):
        og = oracle.bwd(*oracle_inputs(case, j), np32(case.dout[j]), seq_lens=case.seq_lens)
        assert_close_sum(f"check dq_{j}", np32(dqs[j]), [og["dq"]], **TOL_FP32)
        parts["dk_base"].append(og["dk_base"])
        parts["dv_base"].append(og["dv_base"])
    assert_close_sum("check dk_base", np32(g["dk_base"]), parts["dk_base"], **TOL_FP32)
    assert_close_sum("check dv_base", np32(g["dv_base"]), parts["dv_base"], **TOL_FP32)


@pytest.mark.slow
def test_bwd_unroll_qwen_shape_equals_per_call(cuda_ok):
    """Qwen3-235B-A22B draft shape (64 q / 4 kv heads, G = 16: head-split CTAs, L = 4096)."""
    shape = CONFIGS["qwen235b"]
    case = make_case(shape, dtype=torch.bfloat16, seed=1, lens="full")
    dc = DeviceCase(case)
    _assert_equivalent("qwen235b", shape.ttt_steps, *_run_both(dc, shape.ttt_steps, False))
