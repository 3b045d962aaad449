"""GPU parity of tree-attention verification (ttt_tree_attn_fwd, the tcgen05 forward pipeline in
tree mode) against the fp64 oracle (oracle/tree.py), north_star bf16 tolerance 2e-2 / 1e-2."""
import numpy as np
import pytest
import torch

import paper_2603_18567_b200 as ttt
from oracle import tree as OT
from paper_2603_18567_b200.inputs import make_tree_case

pytestmark = pytest.mark.gpu

TOL = dict(atol=2e-2, rtol=1e-2)

CASES = [  # (batch, n, prefix_lens, Hq, Hkv, D)
    (1, 1, [0], 2, 1, 128),             # a single node, no context
    (2, 7, [5, 130], 4, 2, 128),        # tree straddling a 128-key tile boundary
    (3, 33, [0, 127, 500], 8, 2, 64),   # empty prefix, tile-aligned edges, D = 64
    (2, 64, [1000, 2047], 32, 8, 128),  # TTT_MAX_TREE nodes, Llama-3.1-8B target heads
    (1, 64, [64], 5, 5, 128),           # odd head pairs (MHA, G = 1)
    (1, 50, [2040], 8, 2, 128),         # context split over 4 CTAs; tree keys straddle the last two tiles
    (2, 64, [4000, 700], 4, 2, 128),    # uneven contexts, splits by the shorter one
    (1, 64, [1000], 8, 2, 128),         # one tile per split: nodes 0-23 have no key in the last split
    (1, 48, [3000], 64, 4, 128),        # Qwen3-235B target heads (G = 16: four head quads per kv head)
]


def _run(c, extra_rows=0, ws_fill=None):
    B, n = c.q.shape[:2]
    Hq, Hkv, D = c.q.shape[2], c.k.shape[2], c.q.shape[3]
    fp32 = c.q.dtype == torch.float32
    d = ttt.tree_desc(B, n, c.k.shape[1], Hq, Hkv, D, c.prefix_lens,
                      dtype=ttt.TTT_FP32_CHECK if fp32 else ttt.TTT_BF16)
    dev = lambda t: t.cuda().contiguous()
    out = torch.empty(B, n, Hq, D, dtype=c.q.dtype, device="cuda")
    lse = torch.empty(B, Hq, n, dtype=torch.float32, device="cuda")
    ws = torch.empty(ttt.ttt_tree_attn_workspace_size(d), dtype=torch.uint8, device="cuda")
    if ws_fill is not None:
        ws.fill_(ws_fill)
    ttt.ttt_tree_attn_fwd(d, dev(c.q), dev(c.k), dev(c.v), dev(c.parents), out, lse, ws)
    torch.cuda.synchronize()
    return out.float().cpu().numpy(), lse.cpu().numpy()


@pytest.mark.parametrize("case", CASES, ids=[f"B{c[0]}n{c[1]}P{c[2][-1]}H{c[3]}x{c[4]}D{c[5]}" for c in CASES])
def test_tree_attention_vs_oracle(case):
    B, n, P, Hq, Hkv, D = case
    c = make_tree_case(B, n, P, Hq, Hkv, D, seed=n + D, kv_len=max(P) + n + 9)
    out, lse = _run(c)
    f = lambda t: t.float().numpy()
    o_out, o_lse = OT.tree_attention(f(c.q), f(c.k), f(c.v), P, c.parents.numpy())
    for name, got, want in (("out", out, o_out), ("lse", lse, o_lse)):
        err = np.abs(got - want)
        bad = err > TOL["atol"] + TOL["rtol"] * np.abs(want)
        assert not bad.any() and not np.isnan(got).any(), f"{name}: max_abs={err.max():.3e} bad={int(bad.sum())}"


def test_tree_chain_and_deterministic():
    """A chain tree (topk = 1) over a prefix is causal attention; repeated calls are bit-identical."""
    c = make_tree_case(2, 40, [300, 77], 8, 2, 128, seed=5)
    c.parents[:] = torch.arange(-1, 39, dtype=torch.int32)
    a = _run(c)
    b = _run(c)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    f = lambda t: t.float().numpy()
    o_out, _ = OT.tree_attention(f(c.q), f(c.k), f(c.v), c.prefix_lens, c.parents.numpy())
    assert np.abs(a[0] - o_out).max() <= 2e-2 + 1e-2 * np.abs(o_out).max()


@pytest.mark.parametrize("case", CASES[:4] + CASES[6:7], ids=lambda c: f"fp32_B{c[0]}n{c[1]}")
def test_tree_attention_fp32_check_mode(case):
    """TTT_FP32_CHECK: the CUDA-core fp32 path against the oracle at the north_star 1e-5."""
    B, n, P, Hq, Hkv, D = case
    c = make_tree_case(B, n, P, Hq, Hkv, D, dtype=torch.float32, seed=n + 1, kv_len=max(P) + n + 3)
    out, lse = _run(c)
    o_out, o_lse = OT.tree_attention(c.q.numpy(), c.k.numpy(), c.v.numpy(), P, c.parents.numpy())
    np.testing.assert_allclose(out, o_out, rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(lse, o_lse, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("case", [CASES[3], CASES[5]], ids=["split4", "one_tile_per_split"])
def test_tree_workspace_poison(case):
    """compute-sanitizer initcheck flags ttt_tree_combine_kernel's reads of the per-split partials
    (written by TMA stores, which initcheck does not track). Proof that every element the combine
    reads was written by this call: a workspace pre-filled with NaN (0xFF bytes) gives the same,
    finite result as a zero-filled one."""
    B, n, P, Hq, Hkv, D = case
    c = make_tree_case(B, n, P, Hq, Hkv, D, seed=3, kv_len=max(P) + n)
    a = _run(c, ws_fill=0)
    b = _run(c, ws_fill=255)
    assert not np.isnan(b[0]).any() and not np.isnan(b[1]).any()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
