"""GPU parity of the tcgen05 bf16 backward (bwd_sm100.cu) against the fp64
oracle on the same bf16-rounded inputs, north_star tolerance 2e-2 / 1e-2.

The GPU backward consumes the GPU forward's (out, lse), as in training.
Full-size configs use the row-subset reduction: dO is zero
except on sampled rows, so every gradient is exactly the sum over those rows,
which the oracle computes in O(rows * KV * D)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2603_18567_b200.inputs import CONFIGS, Shape, make_case, sample_rows
from tests.gpu_helpers import TOL_BF16, DeviceCase, assert_close, assert_close_sum, np32, oracle_inputs

pytestmark = pytest.mark.gpu

SMALL = [
    ("tiny_bf16", CONFIGS["tiny"], "full"),
    ("tiny_bf16_ragged", CONFIGS["tiny"], "ragged"),
    ("L384_ragged_d128", Shape(2, 384, 4, 2, 128, 4), "ragged"),
    ("gqa3_odd", Shape(1, 256, 6, 2, 128, 3), "ragged"),
    ("mha_g1", Shape(1, 256, 2, 2, 128, 2), "full"),
    ("d64_long", Shape(1, 640, 8, 2, 64, 5), "ragged"),
    ("gqa16_headsplit", Shape(1, 512, 16, 1, 128, 3), "ragged"),
]


def _check_grads(name, dq, g, og, j, mask_q=None):
    if mask_q is None:
        assert_close(f"{name} dq j={j}", np32(dq), og["dq"], **TOL_BF16)
    else:
        assert_close(f"{name} dq j={j} (sampled)", np32(dq)[mask_q], og["dq"][mask_q], **TOL_BF16)
    assert_close(f"{name} dk_base j={j}", np32(g["dk_base"]), og["dk_base"], **TOL_BF16)
    assert_close(f"{name} dv_base j={j}", np32(g["dv_base"]), og["dv_base"], **TOL_BF16)
    for i in range(j):
        assert_close(f"{name} dk_{i+1} j={j}", np32(g["dk_steps"][i]), og["dk_steps"][i], **TOL_BF16)
        assert_close(f"{name} dv_{i+1} j={j}", np32(g["dv_steps"][i]), og["dv_steps"][i], **TOL_BF16)


@pytest.mark.parametrize("name,shape,lens", SMALL, ids=[s[0] for s in SMALL])
def test_bwd_bf16_small(cuda_ok, name, shape, lens):
    case = make_case(shape, dtype=torch.bfloat16, seed=1, lens=lens)
    dc = DeviceCase(case)
    S = shape.ttt_steps
    acc = dc.alloc_grads(S - 1)
    parts = {"dk_base": [], "dv_base": [], "dk_steps": [[] for _ in range(S - 1)],
             "dv_steps": [[] for _ in range(S - 1)]}
    total = dc.alloc_grads(S - 1)  # fp32 sum of the per-call (overwrite-mode) outputs
    for j in reversed(range(S)):
        out, lse = dc.fwd(j)
        g = dc.alloc_grads(S - 1)
        for t in g["dk_steps"] + g["dv_steps"] + [g["dk_base"], g["dv_base"]]:
            t.fill_(77.0)  # overwrite mode must not read these
        dq = dc.bwd(j, out, lse, g, accumulate=False)
        dc.bwd(j, out, lse, acc, accumulate=True)
        total["dk_base"] += g["dk_base"]
        total["dv_base"] += g["dv_base"]
        for i in range(j):
            total["dk_steps"][i] += g["dk_steps"][i]
            total["dv_steps"][i] += g["dv_steps"][i]
        torch.cuda.synchronize()
        og = oracle.bwd(*oracle_inputs(case, j), np32(case.dout[j]), seq_lens=case.seq_lens)
        _check_grads(name, dq, g, og, j)
        parts["dk_base"].append(og["dk_base"])
        parts["dv_base"].append(og["dv_base"])
        for i in range(j):
            parts["dk_steps"][i].append(og["dk_steps"][i])
            parts["dv_steps"][i].append(og["dv_steps"][i])
    # accumulate mode == the fp32 sum of the per-call outputs (each held to the plain bound above), so
    # reading R16's summed bound is exactly the triangle inequality over checked calls
    for key in ("dk_base", "dv_base"):
        torch.testing.assert_close(acc[key], total[key], rtol=1e-5, atol=1e-5)
    for i in range(S - 1):
        torch.testing.assert_close(acc["dk_steps"][i], total["dk_steps"][i], rtol=1e-5, atol=1e-5)
        torch.testing.assert_close(acc["dv_steps"][i], total["dv_steps"][i], rtol=1e-5, atol=1e-5)
    assert_close_sum(f"{name} acc dk_base", np32(acc["dk_base"]), parts["dk_base"], **TOL_BF16)
    assert_close_sum(f"{name} acc dv_base", np32(acc["dv_base"]), parts["dv_base"], **TOL_BF16)
    for i in range(S - 1):
        assert_close_sum(f"{name} acc dk_{i+1}", np32(acc["dk_steps"][i]), parts["dk_steps"][i], **TOL_BF16)
        assert_close_sum(f"{name} acc dv_{i+1}", np32(acc["dv_steps"][i]), parts["dv_steps"][i], **TOL_BF16)


def test_bwd_bf16_gradient_identities(cuda_ok):
    """Exact identities of the true gradient, on the GPU
    result, within bf16 tolerance: sum_k dK_g[k] = 0 and
    sum_k dV_g[k] = sum_{h in g, r} dO_{h,r}."""
    shape = Shape(2, 384, 8, 2, 128, 4)
    case = make_case(shape, dtype=torch.bfloat16, seed=3, lens="ragged")
    dc = DeviceCase(case)
    j = 3
    out, lse = dc.fwd(j)
    g = dc.alloc_grads(3)
    dc.bwd(j, out, lse, g, accumulate=False)
    torch.cuda.synchronize()
    dk_all = torch.cat([g["dk_base"]] + g["dk_steps"], dim=1).double().cpu()
    dv_all = torch.cat([g["dv_base"]] + g["dv_steps"], dim=1).double().cpu()
    do = case.dout[j].double()
    G = 4
    for b in range(2):
        for kv in range(2):
            s_dk = dk_all[b, :, kv].sum(0)
            s_dv = dv_all[b, :, kv].sum(0)
            want_dv = do[b, :, kv * G:(kv + 1) * G].sum((0, 1))
            assert s_dk.abs().max().item() < 0.5, s_dk.abs().max().item()
            assert (s_dv - want_dv).abs().max().item() < 0.5


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["llama8b", "qwen235b", "longctx"])
def test_bwd_bf16_full_size_row_subset(cuda_ok, cfg):
    shape = CONFIGS[cfg]
    case = make_case(shape, dtype=torch.bfloat16, seed=0, lens="full", steps=1)
    j = shape.ttt_steps - 1
    case.q = [case.q[0]] * shape.ttt_steps
    sel = sample_rows(shape, 4, seed=1)                # [B,Hq,L]
    selq = sel.transpose(0, 2, 1)                       # [B,L,Hq]
    do = case.dout[0].clone()
    do[torch.from_numpy(~selq)] = 0
    case.dout = [do] * shape.ttt_steps
    dc = DeviceCase(case)
    out, lse = dc.fwd(j)
    g = dc.alloc_grads(j)
    dq = dc.bwd(j, out, lse, g, accumulate=False)
    torch.cuda.synchronize()
    og = oracle.bwd(*oracle_inputs(case, j), np32(do), seq_lens=case.seq_lens, row_sel=sel)
    _check_grads(cfg, dq, g, og, j, mask_q=selq)
    # rows with dO = 0 have dS = 0 everywhere -> dq exactly 0
    assert np.abs(np32(dq)[~selq]).max() == 0.0


def test_bwd_bf16_shrinking_lengths_per_step(cuda_ok):
    """Variant of reading R6: step j passes T_b - j
    (labels of the last j positions do not exist) through the per-call seq_lens; one
    unroll in reverse order with accumulated dK/dV against the per-step oracle sums."""
    import paper_2603_18567_b200 as ttt
    shape = Shape(2, 384, 8, 2, 128, 4)
    case = make_case(shape, dtype=torch.bfloat16, seed=5, lens="ragged")
    dc = DeviceCase(case)
    S = shape.ttt_steps
    acc = dc.alloc_grads(S - 1)
    parts = {"dk_base": [], "dv_base": [], "dk_steps": [[] for _ in range(S - 1)],
             "dv_steps": [[] for _ in range(S - 1)]}
    for j in reversed(range(S)):
        lens_j = [max(1, int(t) - j) for t in case.seq_lens]
        dc.desc = ttt.desc_for(dc.q[0], dc.k, seq_lens=lens_j)
        out, lse = dc.fwd(j)
        dq = dc.bwd(j, out, lse, acc, accumulate=(j != S - 1))
        torch.cuda.synchronize()
        o_out, o_lse = oracle.fwd(*oracle_inputs(case, j), seq_lens=lens_j)
        assert_close(f"shrink out j={j}", np32(out), o_out, **TOL_BF16)
        assert_close(f"shrink lse j={j}", np32(lse), o_lse, **TOL_BF16)
        og = oracle.bwd(*oracle_inputs(case, j), np32(case.dout[j]), seq_lens=lens_j)
        assert_close(f"shrink dq j={j}", np32(dq), og["dq"], **TOL_BF16)
        parts["dk_base"].append(og["dk_base"])
        parts["dv_base"].append(og["dv_base"])
        for i in range(j):
            parts["dk_steps"][i].append(og["dk_steps"][i])
            parts["dv_steps"][i].append(og["dv_steps"][i])
    assert_close_sum("shrink acc dk_base", np32(acc["dk_base"]), parts["dk_base"], **TOL_BF16)
    assert_close_sum("shrink acc dv_base", np32(acc["dv_base"]), parts["dv_base"], **TOL_BF16)
    for i in range(S - 1):
        assert_close_sum(f"shrink acc dk_{i+1}", np32(acc["dk_steps"][i]), parts["dk_steps"][i], **TOL_BF16)
        assert_close_sum(f"shrink acc dv_{i+1}", np32(acc["dv_steps"][i]), parts["dv_steps"][i], **TOL_BF16)
