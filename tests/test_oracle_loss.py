"""Pins of the fp64 loss oracle (oracle/loss.py) against what the paper, SPEC.md
and mathematics fix — never against the CUDA path. CPU only.

Alg. 3: s <- sum(p g); pi <- softmax(z); z <- -(p g - pi s).
"""
import os

import numpy as np
import pytest
import torch

from oracle import loss as OL

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "loss_examples.txt")


def _rows(s):
    return np.array([[float(x) for x in r.split(",")] for r in s.split(";")])


def _golden():
    out = []
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        kind, z, p, mask, g, exp, tol, cite = line.split()
        out.append((kind, _rows(z), _rows(p), np.array([m == "1" for m in mask.split(",")]),
                    None if g == "-" else float(g), [float(x) for x in exp.split(",")], float(tol), cite))
    return out


@pytest.mark.parametrize("case", _golden(), ids=lambda c: c[-1])
def test_spec_worked_examples(case):
    kind, z, p, mask, g, exp, tol, _ = case
    if kind == "loss":
        L, rl, _, n = OL.loss_forward(z, p, mask)
        assert abs(L - exp[0]) <= tol
        assert np.all(rl[~mask] == 0.0)                       # SPEC.md:255 unmasked rows contribute exactly 0
    else:
        grad = OL.alg3_backward(z, p, np.array([g]))
        np.testing.assert_allclose(grad[0], exp, atol=tol, rtol=0)


def _rand_case(rng, N, V, sigma=2.0, peaked_target=False):
    z = rng.standard_normal((N, V)) * sigma
    zt = z + rng.standard_normal((N, V)) * (0.3 if peaked_target else 1.0)
    p = np.exp(zt - zt.max(1, keepdims=True))
    p /= p.sum(1, keepdims=True)
    return z, p


def test_matches_torch_soft_label_cross_entropy_and_autograd():
    """Library routine: torch.nn.functional.cross_entropy with probability targets
    (mean over the masked rows) in float64 and its autograd gradient."""
    rng = np.random.default_rng(0)
    N, V = 37, 50
    z, p = _rand_case(rng, N, V)
    mask = rng.random(N) < 0.7
    L, rl, lse, n = OL.loss_forward(z, p, mask)
    zt = torch.tensor(z[mask], dtype=torch.float64, requires_grad=True)
    ref = torch.nn.functional.cross_entropy(zt, torch.tensor(p[mask]), reduction="mean")
    assert abs(L - ref.item()) < 1e-12
    np.testing.assert_allclose(lse, torch.logsumexp(torch.tensor(z), 1).numpy(), rtol=1e-14, atol=1e-13)
    (ref * 1.7).backward()
    grad = OL.loss_backward(z, p, mask, g_scale=1.7)
    np.testing.assert_allclose(grad[mask], zt.grad.numpy(), rtol=1e-12, atol=1e-15)
    assert np.all(grad[~mask] == 0.0)                        # masked-out rows get zero gradient


def test_per_row_weights_match_autograd():
    rng = np.random.default_rng(5)
    N, V = 9, 13
    z, p = _rand_case(rng, N, V)
    w = rng.random(N) + 0.5
    zt = torch.tensor(z, requires_grad=True)
    per_row = -(torch.tensor(p) * torch.log_softmax(zt, 1)).sum(1)
    (per_row * torch.tensor(w)).sum().backward()
    grad = OL.loss_backward(z, p, None, g_scale=1.0, g_rows=w, mean=False)
    np.testing.assert_allclose(grad, zt.grad.numpy(), rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("V", [2, 3, 5, 8])
def test_finite_differences(V):
    """central finite differences of loss_forward (here fp64, h=1e-6)."""
    rng = np.random.default_rng(V)
    N = 4
    z, p = _rand_case(rng, N, V)
    mask = np.array([True, False, True, True])
    grad = OL.loss_backward(z, p, mask)
    h = 1e-6
    fd = np.zeros_like(z)
    for r in range(N):
        for v in range(V):
            zp = z.copy(); zp[r, v] += h
            zm = z.copy(); zm[r, v] -= h
            fd[r, v] = (OL.loss_forward(zp, p, mask)[0] - OL.loss_forward(zm, p, mask)[0]) / (2 * h)
    np.testing.assert_allclose(grad, fd, rtol=1e-6, atol=1e-9)


def test_gradient_rows_sum_to_zero_and_closed_form_one_hot():
    """s sum(pi) - g sum(p) = 0 per row; one-hot p, g = 1 gives pi - p."""
    rng = np.random.default_rng(3)
    z, p = _rand_case(rng, 16, 100)
    g = rng.random(16)
    grad = OL.alg3_backward(z, p, g)
    assert np.abs(grad.sum(1)).max() < 1e-15 * 100
    onehot = np.eye(100)[rng.integers(0, 100, 16)]
    np.testing.assert_allclose(OL.alg3_backward(z, onehot, np.ones(16)), OL.softmax_rows(z) - onehot,
                               atol=1e-16, rtol=1e-13)


def test_shift_invariance_and_empty_batch():
    """z and z + c give the same loss; zero masked rows is an error."""
    rng = np.random.default_rng(4)
    z, p = _rand_case(rng, 6, 20)
    a = OL.loss_forward(z, p)[0]
    b = OL.loss_forward(z + 123.25, p)[0]
    assert abs(a - b) < 1e-12
    np.testing.assert_allclose(OL.loss_backward(z, p), OL.loss_backward(z + 123.25, p), atol=1e-15)
    with pytest.raises(ValueError):
        OL.loss_forward(z, p, np.zeros(6, dtype=bool))


def test_loss_is_cross_entropy_identity():
    """Closed form: sum_v p log_softmax(z) = sum p z - lse sum p, and L >= entropy(p)
    (Gibbs' inequality), with equality iff p == softmax(z)."""
    rng = np.random.default_rng(6)
    z, p = _rand_case(rng, 8, 30)
    rl = OL.row_losses(z, p)
    np.testing.assert_allclose(rl, OL.lse_rows(z) * p.sum(1) - (p * z).sum(1), rtol=1e-12)
    ent = -(p * np.log(p)).sum(1)
    assert np.all(rl >= ent - 1e-12)
    pz = OL.softmax_rows(z)
    np.testing.assert_allclose(OL.row_losses(z, pz), -(pz * np.log(pz)).sum(1), rtol=1e-12)
