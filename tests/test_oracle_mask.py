"""Pins for the oracle's Alg. 2 mask — CPU only.

Each check is against something other than the oracle's own formula:
SPEC.md worked examples (tests/golden/), an independent block-structural
construction (tril + identity blocks), count identities, monotonicity.
"""
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _lines(name):
    with open(os.path.join(GOLDEN, name), encoding="utf-8") as f:
        for ln in f:
            ln = ln.strip()
            if ln and not ln.startswith("#"):
                yield ln.split()


def _render_row(row, L):
    """SPEC.md:157 render: █ allowed, · disallowed, │ at each L boundary."""
    out = []
    for k, a in enumerate(row):
        if k and k % L == 0:
            out.append("│")
        out.append("█" if a else "·")
    return "".join(out)


@pytest.mark.parametrize("fields", list(_lines("mask_examples.txt")), ids=lambda f: "-".join(f[:5]))
def test_spec_worked_examples(fields):
    kind, L, T, j, q = fields[0], *map(int, fields[1:5])
    payload = fields[5]
    row = oracle.mask_dense(L, T, j)[q]
    if kind == "allowed":
        want = sorted(int(x) for x in payload.split(","))
        assert [k for k in range(len(row)) if row[k]] == want
        assert all(oracle.mask(L, T, q, k) == (k in want) for k in range(len(row)))
    elif kind == "dense":
        assert "".join("1" if a else "0" for a in row) == payload
    elif kind == "render":
        assert _render_row(row, L) == payload
    else:
        raise AssertionError(kind)


def _block_classes(m, B):
    nq, nk = m.shape[0] // B, m.shape[1] // B
    full, part = {}, {}
    for i in range(nq):
        full[i], part[i] = [], []
        for kb in range(nk):
            blk = m[i * B:(i + 1) * B, kb * B:(kb + 1) * B]
            if blk.all():
                full[i].append(kb)
            elif blk.any():
                part[i].append(kb)
    return full, part


@pytest.mark.parametrize("fields", list(_lines("block_classes.txt")), ids=lambda f: "-".join(f[:6]))
def test_spec_block_classes(fields):
    kind = fields[0]
    L, T, j, B = map(int, fields[1:5])
    m = oracle.mask_dense(L, T, j)
    full, part = _block_classes(m, B)
    if kind == "classes":
        rb = int(fields[5])
        want_full = [] if fields[6] == "-" else [int(x) for x in fields[6].split(",")]
        want_part = [] if fields[7] == "-" else [int(x) for x in fields[7].split(",")]
        assert full[rb] == want_full and part[rb] == want_part
    else:  # every suffix key-block is partial, never full (pure diagonal)
        for rb in full:
            assert all(kb < L // B for kb in full[rb])
            assert all(kb in part[rb] for kb in range(L // B, (j + 1) * L // B))


def _structural_mask(L, T, j):
    """Independent construction: base block = lower triangle with key column
    cut at T; each step block i = identity restricted to rows r < T
    (the diagonal entries k = r + i*L of SURVEY.md §8 'Allowed set')."""
    base = np.tril(np.ones((L, L), dtype=bool))
    base[:, T:] = False
    blocks = [base]
    for _ in range(j):
        d = np.eye(L, dtype=bool)
        d[T:, :] = False
        blocks.append(d)
    return np.concatenate(blocks, axis=1)


def test_matches_structural_construction_200_draws():
    """200 random parameter draws, bit-exact."""
    rng = np.random.default_rng(7)
    for _ in range(200):
        L = int(rng.integers(1, 65))
        T = int(rng.integers(1, L + 1))
        j = int(rng.integers(0, 9))
        assert np.array_equal(oracle.mask_dense(L, T, j), _structural_mask(L, T, j)), (L, T, j)


@pytest.mark.parametrize("L,T,j", [(16, 16, 0), (16, 9, 3), (33, 1, 5), (64, 40, 8)])
def test_allowed_count_identity(L, T, j):
    """|A(r,j)| = r+1+j for r < T, else T."""
    m = oracle.mask_dense(L, T, j)
    for r in range(L):
        prefix = int(m[r, :L].sum())
        suffix = int(m[r, L:].sum())
        if r < T:
            assert (prefix, suffix) == (r + 1, j)
        else:
            assert (prefix, suffix) == (T, 0)


def test_step0_full_length_is_lower_triangular():
    """step 0 with T = Q_LEN is the plain causal mask."""
    for L in (1, 2, 5, 32):
        assert np.array_equal(oracle.mask_dense(L, L, 0), np.tril(np.ones((L, L), dtype=bool)))


def test_monotone_in_T():
    """increasing T never removes an allowed cell."""
    L, j = 24, 3
    prev = oracle.mask_dense(L, 1, j)
    for T in range(2, L + 1):
        cur = oracle.mask_dense(L, T, j)
        assert not (prev & ~cur).any()
        prev = cur
