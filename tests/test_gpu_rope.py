"""GPU parity of ttt_qkv_rope_split (RoPE'd q and the step's K / V slots from a fused projection
output) against the fp64 oracle (oracle/rope.py). Tolerance: the outputs are bf16 roundings of fp32
arithmetic on exact bf16 inputs with fp64-built angles -> |gpu - ref| <= 2^-8 |ref| + 1e-6."""
import numpy as np
import pytest
import torch

import paper_2603_18567_b200 as ttt
from oracle import rope as OR

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("B,L,Hq,Hkv,D,use_pos", [(1, 5, 2, 1, 16, False), (2, 2048, 32, 8, 128, False),
                                                  (1, 16384, 4, 2, 128, False), (2, 300, 8, 2, 64, True)])
def test_qkv_rope_split_vs_oracle(B, L, Hq, Hkv, D, use_pos):
    g = torch.Generator().manual_seed(L + D)
    qkv = torch.randn(B, L, Hq + 2 * Hkv, D, generator=g).to(torch.bfloat16)
    pos = torch.randint(0, 40000, (B, L), generator=g, dtype=torch.int32) if use_pos else None
    d = ttt.rope_desc(B, L, Hq, Hkv, D, 500000.0)
    dev = qkv.cuda()
    q = torch.empty(B, L, Hq, D, dtype=torch.bfloat16, device="cuda")
    k = torch.empty(B, L, Hkv, D, dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    ws = torch.empty(ttt.ttt_rope_workspace_size(d, use_pos), dtype=torch.uint8, device="cuda")
    ttt.ttt_qkv_rope_split(d, dev, q, k, v, ws, positions=None if pos is None else pos.cuda())
    torch.cuda.synchronize()
    qr, kr, vr = OR.qkv_rope_split(qkv.double().numpy(), Hq, Hkv, 500000.0,
                                   positions=None if pos is None else pos.numpy()[:, :])
    for name, got, want in (("q", q, qr), ("k", k, kr)):
        got = got.double().cpu().numpy()
        err = np.abs(got - want)
        assert (err <= 2.0 ** -8 * np.abs(want) + 1e-6).all(), f"{name}: max_abs={err.max():.3e}"
    assert torch.equal(v.cpu(), qkv[:, :, Hq + Hkv:])   # V is copied bit for bit
