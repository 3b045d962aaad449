"""GPU parity of the tcgen05 bf16 forward (fwd_sm100.cu) against the fp64
oracle on the same bf16-rounded inputs, north_star tolerance 2e-2 / 1e-2."""
import numpy as np
import pytest
import torch

import oracle
from paper_2603_18567_b200.inputs import CONFIGS, Shape, make_case, sample_rows
from tests.gpu_helpers import TOL_BF16, DeviceCase, assert_close, np32, oracle_inputs

pytestmark = pytest.mark.gpu

SMALL = [
    ("tiny_bf16", CONFIGS["tiny"], "full", False),
    ("tiny_bf16_ragged", CONFIGS["tiny"], "ragged", False),
    ("L384_ragged_d128", Shape(2, 384, 4, 2, 128, 4), "ragged", False),
    ("gqa3_odd", Shape(1, 256, 6, 2, 128, 3), "ragged", False),
    ("mha_g1", Shape(1, 256, 2, 2, 128, 2), "full", False),
    ("peaked_q", Shape(2, 256, 4, 1, 128, 3), "ragged", True),
    ("d64_long", Shape(1, 640, 8, 2, 64, 5), "ragged", False),
]


@pytest.mark.parametrize("name,shape,lens,peaked", SMALL, ids=[s[0] for s in SMALL])
def test_fwd_bf16_small(cuda_ok, name, shape, lens, peaked):
    case = make_case(shape, dtype=torch.bfloat16, seed=0, lens=lens, peaked=peaked)
    dc = DeviceCase(case)
    for j in range(shape.ttt_steps):
        out, lse = dc.fwd(j)
        torch.cuda.synchronize()
        o_out, o_lse = oracle.fwd(*oracle_inputs(case, j), seq_lens=case.seq_lens)
        assert_close(f"{name} out j={j}", np32(out), o_out, **TOL_BF16)
        assert_close(f"{name} lse j={j}", np32(lse), o_lse, **TOL_BF16)


def test_fwd_bf16_deterministic(cuda_ok):
    shape = Shape(2, 512, 8, 2, 128, 3)
    case = make_case(shape, dtype=torch.bfloat16, seed=4)
    dc = DeviceCase(case)
    a, la = dc.fwd(2)
    b, lb = dc.fwd(2)
    torch.cuda.synchronize()
    assert torch.equal(a, b) and torch.equal(la, lb)


def test_fwd_bf16_masked_inputs_inert(cuda_ok):
    """Finite poison at disallowed K/V positions (keys >= T_b, step rows >= T_b)
    leaves out/lse bitwise identical (SURVEY.md §8c 'Masked inertness')."""
    shape = Shape(2, 384, 4, 2, 128, 3)
    case = make_case(shape, dtype=torch.bfloat16, seed=5, lens="ragged")
    dc = DeviceCase(case)
    out0, lse0 = dc.fwd(2)
    for b, T in enumerate(case.seq_lens):
        T = int(T)
        dc.k[b, T:] = 3e4
        dc.v[b, T:] = -3e4
        for t in dc.ks + dc.vs:
            t[b, T:] = 3e4
    out1, lse1 = dc.fwd(2)
    torch.cuda.synchronize()
    assert torch.equal(out0, out1) and torch.equal(lse0, lse1)


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["llama8b", "qwen235b", "longctx"])
def test_fwd_bf16_full_size_sampled_rows(cuda_ok, cfg):
    """Full BASELINE.json shape, the launch configuration bench.py times;
    oracle on sampled rows (rows are independent in the forward)."""
    shape = CONFIGS[cfg]
    case = make_case(shape, dtype=torch.bfloat16, seed=0, lens="full", steps=1)
    # the last TTT step (the paper measures the final step) uses q_0's bits here
    j = shape.ttt_steps - 1
    case.q = [case.q[0]] * shape.ttt_steps
    dc = DeviceCase(case)
    out, lse = dc.fwd(j)
    torch.cuda.synchronize()
    sel = sample_rows(shape, 6, seed=0)
    o_out, o_lse = oracle.fwd(*oracle_inputs(case, j), seq_lens=case.seq_lens, row_sel=sel)
    selq = sel.transpose(0, 2, 1)
    assert_close(f"{cfg} out", np32(out)[selq], o_out[selq], **TOL_BF16)
    assert_close(f"{cfg} lse", np32(lse)[sel], o_lse[sel], **TOL_BF16)
