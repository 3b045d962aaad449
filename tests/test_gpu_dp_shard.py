"""Data-parallel sharding by sequence is exact ("attention outputs per rank must be
bit-identical to the 1-GPU run"). A rank of bench.py / dp.micro_batches runs a contiguous block of the
global batch through the same kernels; here the first and second halves of a ragged batch, computed as
separate calls (the two "ranks"), are compared with the same sequences inside the full-batch call.

Forward outputs (out, lse) must match bitwise: every CTA's work depends only on its own sequence. The
backward's dq partials are reduce-added into fp32 by several CTAs in hardware order, and dK / dV by
several head-subset CTAs when the grid is small, so the gradients are compared to fp32 rounding of that
order (and must still be identical in bf16 wherever both orders round the same way, checked loosely)."""
import pytest
import torch

import paper_2603_18567_b200 as ttt
from paper_2603_18567_b200.inputs import Shape, make_case

pytestmark = pytest.mark.gpu


def _run(q, k, v, ks, vs, dout, lens, j):
    desc = ttt.desc_for(q, k, seq_lens=lens)
    out = torch.empty_like(q)
    lo = torch.empty_like(q)
    lse = torch.empty(q.shape[0], q.shape[2], q.shape[1], device=q.device)
    ttt.ttt_attn_fwd(desc, j, q, k, v, ks, vs, out, lse, out_lo=lo)
    z = lambda: torch.zeros(k.shape, dtype=torch.float32, device=q.device)
    dk, dv = z(), z()
    dks, dvs = [z() for _ in range(j)], [z() for _ in range(j)]
    dq = torch.empty_like(q)
    ws = torch.empty(max(ttt.ttt_attn_workspace_size(desc, j, True), 16), dtype=torch.uint8, device=q.device)
    ttt.ttt_attn_bwd(desc, j, q, k, v, ks, vs, out, lse, dout, dq, dk, dv, dks, dvs, flags=0, workspace=ws,
                     out_lo=lo)
    torch.cuda.synchronize()
    return out, lse, dq, dk, dv, dks, dvs


@pytest.mark.parametrize("shape", [Shape(4, 384, 8, 2, 128, 4), Shape(4, 256, 4, 4, 64, 3)], ids=["gqa_d128", "mha_d64"])
def test_sequence_shards_equal_full_batch(cuda_ok, shape):
    case = make_case(shape, dtype=torch.bfloat16, seed=44, lens="ragged")
    dev = "cuda"
    j = shape.ttt_steps - 1
    q = case.q[j].to(dev)
    k, v = case.k_base.to(dev), case.v_base.to(dev)
    ks = [x.to(dev) for x in case.k_steps[:j]]
    vs = [x.to(dev) for x in case.v_steps[:j]]
    do = case.dout[j].to(dev)
    lens = [int(x) for x in case.seq_lens]
    full = _run(q, k, v, ks, vs, do, lens, j)
    B, h = shape.batch, shape.batch // 2
    for lo, hi in ((0, h), (h, B)):
        sl = lambda t: t[lo:hi].contiguous()
        part = _run(sl(q), sl(k), sl(v), [sl(x) for x in ks], [sl(x) for x in vs], sl(do), lens[lo:hi], j)
        out_f, lse_f, dq_f, dk_f, dv_f, dks_f, dvs_f = full
        out_p, lse_p, dq_p, dk_p, dv_p, dks_p, dvs_p = part
        assert torch.equal(out_p, out_f[lo:hi]), f"out of shard [{lo},{hi}) differs from the full batch"
        assert torch.equal(lse_p, lse_f[lo:hi]), f"lse of shard [{lo},{hi}) differs from the full batch"
        torch.testing.assert_close(dq_p.float(), dq_f[lo:hi].float(), rtol=1e-2, atol=2e-3)
        for name, a, b in [("dk", dk_p, dk_f), ("dv", dv_p, dv_f)] + \
                [(f"dk_{i + 1}", dks_p[i], dks_f[i]) for i in range(j)] + [(f"dv_{i + 1}", dvs_p[i], dvs_f[i]) for i in range(j)]:
            torch.testing.assert_close(a, b[lo:hi], rtol=1e-5, atol=1e-5, msg=lambda m: f"{name}: {m}")
