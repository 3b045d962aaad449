"""GPU parity of the loss kernels (include/ttt_loss.h) against the fp64 oracle
(oracle/loss.py), element by element, through the C-ABI binding.

Tolerances ("loss"): the kernel computes in fp32 from the exact
stored inputs; the gradient leaves in the storage dtype.
  grad: |gpu - ref| <= rtol |ref| + 1e-5 (pi_v |s| + p_v |g|) + 2^-120
        rtol = 2^-8 for bf16 (twice the RNE half-ulp 2^-9 of the stored value),
        1e-5 for fp32 (north_star check-mode tolerance); the 1e-5 term bounds the
        fp32 error of pi = exp(z - lse) and of the two products of Alg. 3; 2^-120 is the
        fp32 / bf16 normal range (smaller exact values, e.g. pi = 1e-115 at |z| ~ 100,
        flush to zero).
  lse, loss: 1e-5 relative + 1e-5 absolute (fp32 row sums, fp64 across rows).
Masked-out rows: gradient exactly 0. In place == out of place, bit for bit.
"""
import numpy as np
import pytest
import torch

import paper_2603_18567_b200 as ttt
from oracle import loss as OL
from paper_2603_18567_b200.inputs import LOSS_CONFIGS, make_loss_case

pytestmark = pytest.mark.gpu

DT = {"bf16": torch.bfloat16, "fp32": torch.float32}
RTOL = {"bf16": 2.0 ** -8, "fp32": 1e-5}


def _run(case, mode="fused", g_scale=1.0, flags=ttt.TTT_LOSS_MEAN, use_g_rows=False, out_of_place=False):
    dev = torch.device("cuda")
    z = case.z.to(dev)
    p = case.p.to(dev)
    mask = case.mask.to(dev)
    g_rows = case.g_rows.to(dev) if use_g_rows else None
    d = ttt.loss_desc_for(z)
    ws = torch.empty(ttt.ttt_loss_workspace_size(d), dtype=torch.uint8, device=dev)
    stats = torch.full((2,), float("nan"), dtype=torch.float64, device=dev)
    lse = torch.full((z.shape[0],), float("nan"), dtype=torch.float32, device=dev)
    grad = torch.empty_like(z) if out_of_place else None
    if mode == "fused":
        ttt.ttt_loss_fwd_bwd_inplace(d, z, p, mask, stats, ws, g_scale=g_scale, flags=flags, g_rows=g_rows,
                                     grad=grad, lse=lse)
    else:
        ttt.ttt_loss_fwd(d, z, p, mask, stats, ws, lse=lse)
        ttt.ttt_loss_bwd_inplace(d, z, p, mask, ws, g_scale=g_scale, flags=flags, g_rows=g_rows, grad=grad)
    torch.cuda.synchronize()
    g = grad if out_of_place else z
    return g.cpu(), lse.cpu().numpy().astype(np.float64), stats.cpu().numpy()


def _check_grad(name, got, zf, pf, mask, g_rows, g_scale, mean, dt, rows=None):
    """got [n, V] GPU gradient rows; zf/pf fp64 inputs of the same rows."""
    ref = OL.alg3_backward(zf, pf, _g(mask, g_rows, g_scale, mean, rows))
    g = _g(mask, g_rows, g_scale, mean, rows)
    pi = OL.softmax_rows(zf)
    s = (pf * g[:, None]).sum(1)
    atol = 1e-5 * (pi * np.abs(s)[:, None] + pf * np.abs(g)[:, None]) + 2.0 ** -120
    got = got.double().numpy()
    err = np.abs(got - ref)
    bad = err > RTOL[dt] * np.abs(ref) + atol
    assert not bad.any(), f"{name}: max_abs={err.max():.3e} violations={int(bad.sum())}/{bad.size}"
    return ref


def _g(mask, g_rows, g_scale, mean, rows):
    g = OL.upstream_g(len(mask), mask.astype(bool), g_scale, g_rows, mean)
    return g if rows is None else g[rows]


# shapes: element path (odd vocab), one CTA per row (NV = 1 / 4 / 8), clusters of 2-8 CTAs
SMALL = [(1, 2), (3, 3), (7, 5), (64, 1000), (33, 2048), (9, 32000), (5, 16383), (3, 32767), (4, 65536),
         (2, 131072)]


@pytest.mark.parametrize("dt", ["bf16", "fp32"])
@pytest.mark.parametrize("rows,vocab", SMALL, ids=[f"{r}x{v}" for r, v in SMALL])
def test_loss_small(dt, rows, vocab):
    case = make_loss_case(rows, vocab, DT[dt], seed=rows + vocab)
    zf, pf = case.z.double().numpy(), case.p.double().numpy()
    mask = case.mask.numpy()
    grad, lse, stats = _run(case, use_g_rows=True, g_scale=0.75)
    L, _, lse_ref, n = OL.loss_forward(zf, pf, mask.astype(bool))
    assert stats[1] == n
    assert abs(stats[0] - L) <= 1e-5 * abs(L) + 1e-5, (stats[0], L)
    np.testing.assert_allclose(lse, lse_ref, rtol=1e-5, atol=1e-5)
    _check_grad("grad", grad, zf, pf, mask, case.g_rows.double().numpy(), 0.75, True, dt)
    assert torch.all(grad[torch.from_numpy(mask == 0)] == 0)          # masked-out rows: exactly zero
    rs = grad.double().sum(1).numpy()                                   # SPEC.md:282 conservation
    assert np.all(np.abs(rs) <= RTOL[dt] * np.abs(grad.double()).sum(1).numpy() + 1e-12)


@pytest.mark.parametrize("dt", ["bf16", "fp32"])
def test_loss_inplace_equals_out_of_place_and_separate_calls(dt):
    """in-place == out-of-place bit for bit; fused pass == fwd then bwd."""
    case = make_loss_case(48, 4096, DT[dt], seed=11)
    a, lse_a, st_a = _run(case, mode="fused")
    b, lse_b, st_b = _run(case, mode="fused", out_of_place=True)
    c, lse_c, st_c = _run(case, mode="separate")
    assert torch.equal(a, b) and torch.equal(a, c)
    assert np.array_equal(lse_a, lse_c) and np.array_equal(st_a, st_c) and np.array_equal(st_a, st_b)
    a2, _, st2 = _run(case, mode="fused")                               # deterministic
    assert torch.equal(a, a2) and np.array_equal(st_a, st2)


def test_loss_not_mean_and_empty_mask():
    case = make_loss_case(16, 1000, torch.bfloat16, seed=3, mask_mode="all")
    grad, _, stats = _run(case, flags=0, g_scale=2.0)
    zf, pf = case.z.double().numpy(), case.p.double().numpy()
    _check_grad("grad_sum", grad, zf, pf, case.mask.numpy(), None, 2.0, False, "bf16")
    case.mask.zero_()                                                   # SPEC.md:257 empty batch
    grad, _, stats = _run(case)
    assert np.isnan(stats[0]) and stats[1] == 0
    assert torch.all(grad == 0)


def test_loss_extreme_logits():
    """Large-magnitude logits (max subtraction) and one-hot targets (SPEC.md:259, 266 shapes)."""
    case = make_loss_case(8, 512, torch.float32, seed=4, z_scale=40.0, mask_mode="all")
    case.p.zero_()
    case.p[torch.arange(8), torch.arange(8) * 17] = 1.0
    grad, lse, stats = _run(case)
    zf, pf = case.z.double().numpy(), case.p.double().numpy()
    L, _, lse_ref, _ = OL.loss_forward(zf, pf)
    assert abs(stats[0] - L) <= 1e-5 * abs(L) + 1e-5
    np.testing.assert_allclose(lse, lse_ref, rtol=1e-5, atol=1e-5)
    _check_grad("grad", grad, zf, pf, case.mask.numpy(), None, 1.0, True, "fp32")


@pytest.mark.slow
def test_loss_full_size_llama_sampled_rows():
    """BASELINE workload rows (B L = 16384, draft vocab 32000, bf16) in bench.py's launch
    configuration; loss over all rows (oracle in row chunks), gradient on 96 sampled rows."""
    rows, vocab = LOSS_CONFIGS["llama8b"]
    case = make_loss_case(rows, vocab, torch.bfloat16, seed=0)
    zf_all = case.z
    grad, lse, stats = _run(case, use_g_rows=True)
    mask = case.mask.numpy().astype(bool)
    total, n = 0.0, int(mask.sum())
    lse_ref = np.empty(rows)
    for r0 in range(0, rows, 1024):
        zc = zf_all[r0:r0 + 1024].double().numpy()
        pc = case.p[r0:r0 + 1024].double().numpy()
        rl = OL.row_losses(zc, pc)
        lse_ref[r0:r0 + 1024] = OL.lse_rows(zc)
        for i in range(len(rl)):
            if mask[r0 + i]:
                total += rl[i]
    assert stats[1] == n
    assert abs(stats[0] - total / n) <= 1e-5 * abs(total / n) + 1e-5
    np.testing.assert_allclose(lse, lse_ref, rtol=1e-5, atol=1e-5)
    sel = np.sort(np.random.default_rng(9).choice(rows, 96, replace=False))
    sel = np.concatenate([sel, [0, rows - 1]])
    _check_grad("grad_rows", grad[sel], case.z[sel].double().numpy(), case.p[sel].double().numpy(),
                case.mask.numpy(), case.g_rows.double().numpy(), 1.0, True, "bf16", rows=sel)
    assert torch.all(grad[torch.from_numpy(~mask)] == 0)
