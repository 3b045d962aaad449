"""GPU: the head-parallel split of a long sequence (dp.seq_to_head) is
exact — the TTT attention of a block of Hkv/N kv heads (and their G q heads each), computed as a
problem of its own, equals those heads of the full problem: forward bit for bit; dK / dV (GQA sums
stay inside the block) and dq up to fp32 summation order (rows are grouped differently into
tensor-core tiles, and dq / dK_0 tiles are reduce-added by several CTAs)."""
import pytest
import torch

import paper_2603_18567_b200 as ttt
from paper_2603_18567_b200.inputs import Shape, make_case
from tests.gpu_helpers import DeviceCase

pytestmark = pytest.mark.gpu


def _unroll(dc, S, heads=None):
    """fwd all steps + bwd j = S-1..0 (accumulating) for a DeviceCase."""
    outs, lses, dqs = [], [], []
    g = dc.alloc_grads(S - 1)
    for j in range(S):
        o, l = dc.fwd(j)
        outs.append((o, l, dc.out_lo))
    for j in reversed(range(S)):
        o, l, lo = outs[j]
        dc.out_lo = lo
        dqs.insert(0, dc.bwd(j, o, l, g, accumulate=j != S - 1))
    torch.cuda.synchronize()
    return outs, dqs, g


@pytest.mark.parametrize("world", [2, 4])
def test_head_block_equals_full_problem(cuda_ok, world):
    shape = Shape(1, 1024, 16, 4, 128, 3)
    S = shape.ttt_steps
    case = make_case(shape, dtype=torch.bfloat16, seed=11, lens="full")
    full = DeviceCase(case)
    f_outs, f_dq, f_g = _unroll(full, S)
    Hq, Hkv = shape.num_q_heads // world, shape.num_kv_heads // world
    for r in range(world):
        part = DeviceCase(case)
        qs, ks = slice(r * Hq, (r + 1) * Hq), slice(r * Hkv, (r + 1) * Hkv)
        part.q = [t[:, :, qs].contiguous() for t in full.q]
        part.dout = [t[:, :, qs].contiguous() for t in full.dout]
        part.k, part.v = full.k[:, :, ks].contiguous(), full.v[:, :, ks].contiguous()
        part.ks = [t[:, :, ks].contiguous() for t in full.ks]
        part.vs = [t[:, :, ks].contiguous() for t in full.vs]
        part.case = type(case)(shape=Shape(1, 1024, Hq, Hkv, 128, S), dtype=case.dtype)
        part.desc = ttt.desc_for(part.q[0], part.k, seq_lens=part.lens)
        p_outs, p_dq, p_g = _unroll(part, S)
        for j in range(S):
            assert torch.equal(p_outs[j][0], f_outs[j][0][:, :, qs]), f"rank {r} out_{j}"
            assert torch.equal(p_outs[j][1], f_outs[j][1][:, qs]), f"rank {r} lse_{j}"
            torch.testing.assert_close(p_dq[j].float(), f_dq[j][:, :, qs].float(), rtol=2.0 ** -7, atol=1e-5)
        for i in range(S - 1):
            torch.testing.assert_close(p_g["dk_steps"][i], f_g["dk_steps"][i][:, :, ks], rtol=1e-5, atol=1e-6)
            torch.testing.assert_close(p_g["dv_steps"][i], f_g["dv_steps"][i][:, :, ks], rtol=1e-5, atol=1e-6)
        for k in ("dk_base", "dv_base"):
            torch.testing.assert_close(p_g[k], f_g[k][:, :, ks], rtol=1e-5, atol=1e-5)
