"""TEST INFRASTRUCTURE — fp64 CPU oracle of the masked soft-label log-softmax
loss and its in-place backward (Alg. 3). NOT product code.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` leg may import this module. It shares no code with the
CUDA path (``paper_2603_18567_b200/csrc/loss_sm100.cu``) and never imports it.

What it follows
  * PAPER.md:338-340 (§4.2.1 "Memory-Efficient Gradient Computation"): the
    backward of the masked softmax loss overwrites the logits tensor with the
    gradient w.r.t. the logits.
  * PAPER.md:342-354, Alg. 3 "In-place Backward for Log-Softmax Loss":
        Input: logits z, target p, upstream gradient g
        s  <- sum(p * g)
        pi <- softmax(z)
        z  <- -(p * g - pi * s)
  * SPEC.md:241-291 (the loss module written from the paper) for what the
    paper leaves open, taken as DESIGN.md readings R17-R20:
      - loss L = -sum_{masked rows} sum_v p log_softmax(z) / (number of masked
        rows);
      - s is a per-row sum;
      - g is the per-row upstream gradient of that row's term: for the mean
        loss, g_r = g_scale * w_r / n_masked on masked rows, 0 elsewhere
        (SPEC.md:264, 288);
      - pi is recomputed from z in the backward.

Every step is fp64 numpy on the exact input values; sums run in natural index
order per row. Pinned by tests/test_oracle_loss.py (SPEC worked examples in
tests/golden/loss_examples.txt, torch's soft-label cross-entropy and its
autograd gradient in float64, central finite differences, row-sum
conservation, shift invariance). Nothing here is "parity unpinned".
"""
from __future__ import annotations

import numpy as np


def _f64(a) -> np.ndarray:
    return np.asarray(a, dtype=np.float64)


def log_softmax_rows(z) -> np.ndarray:
    """log_softmax over the last axis: z - (m + ln sum exp(z - m))."""
    z = _f64(z)
    m = z.max(axis=-1, keepdims=True)
    return z - (m + np.log(np.exp(z - m).sum(axis=-1, keepdims=True)))


def lse_rows(z) -> np.ndarray:
    """Natural-log logsumexp of each row of z."""
    z = _f64(z)
    m = z.max(axis=-1)
    return m + np.log(np.exp(z - m[:, None]).sum(axis=-1))


def softmax_rows(z) -> np.ndarray:
    """pi = softmax(z) per row (Alg. 3 line 'pi <- softmax(z)')."""
    z = _f64(z)
    e = np.exp(z - z.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def row_losses(z, p) -> np.ndarray:
    """Per-row soft-label loss -sum_v p_v log_softmax(z)_v."""
    return -(_f64(p) * log_softmax_rows(z)).sum(axis=-1)


def loss_forward(z, p, mask=None):
    """Masked mean loss.

    z, p [N, V]; mask bool [N] (None = all rows). Returns
    (L, row_loss [N] fp64 with unmasked rows exactly 0, lse [N], n_masked).
    Raises ValueError on zero masked rows ("empty-batch error").
    """
    z = _f64(z)
    N = z.shape[0]
    msk = np.ones(N, dtype=bool) if mask is None else np.asarray(mask, dtype=bool)
    n = int(msk.sum())
    if n == 0:
        raise ValueError("empty batch: no masked row")
    rl = np.where(msk, row_losses(z, p), 0.0)
    total = 0.0
    for r in range(N):          # natural order, fp64 ("64-bit accumulation")
        total += rl[r]
    return total / n, rl, lse_rows(z), n


def upstream_g(N, mask=None, g_scale=1.0, g_rows=None, mean=True):
    """Per-row upstream gradient g_r of the (mean) loss: dL_total/d(row term r).

    g_r = g_scale * (g_rows[r] or 1) / (n_masked if mean else 1) on masked
    rows, 0 on the others (reading R19)."""
    msk = np.ones(N, dtype=bool) if mask is None else np.asarray(mask, dtype=bool)
    w = np.ones(N) if g_rows is None else _f64(g_rows)
    n = int(msk.sum())
    div = float(n) if mean else 1.0
    return np.where(msk, float(g_scale) * w / div, 0.0)


def alg3_backward(z, p, g) -> np.ndarray:
    """Alg. 3 literally, row by row.

    z, p [N, V]; g [N] per-row upstream gradient. Returns the array that Alg. 3
    leaves in z's buffer: -(p*g - pi*s) with s = sum(p*g) per row."""
    z = _f64(z)
    p = _f64(p)
    out = np.empty_like(z)
    for r in range(z.shape[0]):
        pg = p[r] * g[r]
        s = pg.sum()                     # s <- sum(p * g)
        pi = softmax_rows(z[r:r + 1])[0]  # pi <- softmax(z)
        out[r] = -(pg - pi * s)          # z <- -(p * g - pi * s)
    return out


def loss_backward(z, p, mask=None, g_scale=1.0, g_rows=None, mean=True) -> np.ndarray:
    """Gradient of g_scale * L (L the masked mean loss) w.r.t. z via Alg. 3."""
    g = upstream_g(np.asarray(z).shape[0], mask, g_scale, g_rows, mean)
    return alg3_backward(z, p, g)
