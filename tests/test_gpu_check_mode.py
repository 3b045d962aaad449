"""GPU parity of the TTT_FP32_CHECK path (CUDA-core fp32) against the fp64
oracle at the north_star fp32 tolerance (1e-5), through the C-ABI."""
import numpy as np
import pytest
import torch

import oracle
from paper_2603_18567_b200.inputs import CONFIGS, Shape, make_case
from tests.gpu_helpers import TOL_FP32, DeviceCase, assert_close, assert_close_sum, np32, oracle_inputs

pytestmark = pytest.mark.gpu

SHAPES = [
    ("tiny", CONFIGS["tiny"], "full"),
    ("tiny_ragged", CONFIGS["tiny"], "ragged"),
    ("odd_L_gqa3_d128", Shape(2, 100, 6, 2, 128, 5), "ragged"),
]


@pytest.mark.parametrize("name,shape,lens", SHAPES, ids=[s[0] for s in SHAPES])
def test_check_mode_fwd_bwd_all_steps(cuda_ok, name, shape, lens):
    case = make_case(shape, dtype=torch.float32, seed=0, lens=lens)
    dc = DeviceCase(case)
    S = shape.ttt_steps
    acc = dc.alloc_grads(S - 1)
    want_acc = None
    for j in reversed(range(S)):  # reverse step order, as in an unroll's backward
        out, lse = dc.fwd(j)
        qn, kb, vb, ks, vs = oracle_inputs(case, j)
        o_out, o_lse = oracle.fwd(qn, kb, vb, ks, vs, seq_lens=case.seq_lens)
        assert_close(f"{name} out j={j}", np32(out), o_out, **TOL_FP32)
        assert_close(f"{name} lse j={j}", np32(lse), o_lse, **TOL_FP32)
        # overwrite mode for this step alone
        g = dc.alloc_grads(S - 1)
        for t in g["dk_steps"] + g["dv_steps"] + [g["dk_base"], g["dv_base"]]:
            t.fill_(123.0)  # must be overwritten
        dq = dc.bwd(j, out, lse, g, accumulate=False)
        og = oracle.bwd(qn, kb, vb, ks, vs, np32(case.dout[j]), seq_lens=case.seq_lens)
        assert_close(f"{name} dq j={j}", np32(dq), og["dq"], **TOL_FP32)
        assert_close(f"{name} dk_base j={j}", np32(g["dk_base"]), og["dk_base"], **TOL_FP32)
        assert_close(f"{name} dv_base j={j}", np32(g["dv_base"]), og["dv_base"], **TOL_FP32)
        for i in range(j):
            assert_close(f"{name} dk_{i+1} j={j}", np32(g["dk_steps"][i]), og["dk_steps"][i], **TOL_FP32)
            assert_close(f"{name} dv_{i+1} j={j}", np32(g["dv_steps"][i]), og["dv_steps"][i], **TOL_FP32)
        # accumulate mode across the unroll
        dc.bwd(j, out, lse, acc, accumulate=True)
        if want_acc is None:
            want_acc = {"dk_base": og["dk_base"].copy(), "dv_base": og["dv_base"].copy(),
                        "dk_steps": [np.zeros_like(og["dk_base"]) for _ in range(S - 1)],
                        "dv_steps": [np.zeros_like(og["dk_base"]) for _ in range(S - 1)]}
        else:
            want_acc["dk_base"] += og["dk_base"]
            want_acc["dv_base"] += og["dv_base"]
        for i in range(j):
            want_acc["dk_steps"][i] += og["dk_steps"][i]
            want_acc["dv_steps"][i] += og["dv_steps"][i]
    torch.cuda.synchronize()
    assert_close(f"{name} acc dk_base", np32(acc["dk_base"]), want_acc["dk_base"], **TOL_FP32)
    assert_close(f"{name} acc dv_base", np32(acc["dv_base"]), want_acc["dv_base"], **TOL_FP32)
    for i in range(S - 1):
        assert_close(f"{name} acc dk_{i+1}", np32(acc["dk_steps"][i]), want_acc["dk_steps"][i], **TOL_FP32)
        assert_close(f"{name} acc dv_{i+1}", np32(acc["dv_steps"][i]), want_acc["dv_steps"][i], **TOL_FP32)
