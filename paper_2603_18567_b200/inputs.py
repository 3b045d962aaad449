"""Seeded synthetic inputs shared by tests/, bench.py and the oracle checks.

This module holds NO arithmetic of the method: it only draws random numbers
and rounds them to the storage dtype, so the oracle and the CUDA path see the
identical bits. Recipe (SURVEY.md §8d "Value distributions"):

  * q, k, v, dO ~ N(0, 1) drawn in fp32 by ``numpy.random.default_rng(seed)``
    then rounded to bf16 (round-to-nearest-even) for the BF16 path, kept fp32
    for the FP32_CHECK path. With c = 1/sqrt(D) the logits are ~N(0, 1).
  * "peaked" variant: q scaled by 4 before rounding (stresses max-subtraction).
  * sequence lengths T_b ~ U[L/4, L] (padded conversations),
    or T_b = L ("full") for throughput runs.
  * seeds: inputs ``seed``, dO ``seed + 1``, lengths ``seed + 2``.
  * one unroll of S TTT steps has S-1 step lists K_1..K_{S-1}, V_1..V_{S-1}
    (step j uses the first j, reading R1) and one q / dO per step
    (q_j depends on step j-1's output in EAGLE-3).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch


@dataclass(frozen=True)
class Shape:
    batch: int
    seq_len: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    ttt_steps: int

    @property
    def q_shape(self):
        return (self.batch, self.seq_len, self.num_q_heads, self.head_dim)

    @property
    def kv_shape(self):
        return (self.batch, self.seq_len, self.num_kv_heads, self.head_dim)


# BASELINE.json "configs" (index order kept).
CONFIGS = {
    "tiny": Shape(1, 128, 4, 2, 64, 3),
    "llama8b": Shape(8, 2048, 32, 8, 128, 7),
    "qwen235b": Shape(1, 4096, 64, 4, 128, 7),
    "longctx": Shape(1, 16384, 32, 8, 128, 7),
    "dp": Shape(8, 4096, 32, 8, 128, 7),  # one micro-batch of the global-batch-64 DP sweep
}


def _normal(rng: np.random.Generator, shape, scale=1.0) -> np.ndarray:
    x = rng.standard_normal(size=shape, dtype=np.float32)
    if scale != 1.0:
        x *= np.float32(scale)
    return x


def to_storage(x: np.ndarray, dtype: torch.dtype) -> torch.Tensor:
    """fp32 numpy -> torch CPU tensor of the storage dtype (bf16 rounding is RNE)."""
    return torch.from_numpy(np.ascontiguousarray(x)).to(dtype)


def seq_lens(shape: Shape, seed: int, mode: str = "ragged") -> np.ndarray:
    """T_b per sequence: 'full' -> L; 'ragged' -> U[L/4, L] (seed + 2)."""
    if mode == "full":
        return np.full(shape.batch, shape.seq_len, dtype=np.int32)
    rng = np.random.default_rng(seed + 2)
    lo = max(1, shape.seq_len // 4)
    return rng.integers(lo, shape.seq_len + 1, size=shape.batch, dtype=np.int32)


@dataclass
class Case:
    """Host-side (CPU torch) tensors of one TTT unroll."""
    shape: Shape
    dtype: torch.dtype
    q: list = field(default_factory=list)        # per step j: [B,L,Hq,D]
    dout: list = field(default_factory=list)     # per step j: [B,L,Hq,D]
    k_base: torch.Tensor = None                  # [B,L,Hkv,D]
    v_base: torch.Tensor = None
    k_steps: list = field(default_factory=list)  # S-1 of [B,L,Hkv,D]
    v_steps: list = field(default_factory=list)
    seq_lens: np.ndarray = None                  # int32[B]


def make_case(shape: Shape, dtype: torch.dtype = torch.bfloat16, seed: int = 0,
              lens: str = "ragged", peaked: bool = False, steps=None) -> Case:
    """Draw one unroll's inputs. ``steps`` limits how many per-step q/dO are drawn."""
    S = shape.ttt_steps if steps is None else steps
    rng = np.random.default_rng(seed)
    c = Case(shape=shape, dtype=dtype)
    c.k_base = to_storage(_normal(rng, shape.kv_shape), dtype)
    c.v_base = to_storage(_normal(rng, shape.kv_shape), dtype)
    for _ in range(max(shape.ttt_steps - 1, 0)):
        c.k_steps.append(to_storage(_normal(rng, shape.kv_shape), dtype))
        c.v_steps.append(to_storage(_normal(rng, shape.kv_shape), dtype))
    qscale = 4.0 if peaked else 1.0
    for _ in range(S):
        c.q.append(to_storage(_normal(rng, shape.q_shape, qscale), dtype))
    rng_do = np.random.default_rng(seed + 1)
    for _ in range(S):
        c.dout.append(to_storage(_normal(rng_do, shape.q_shape), dtype))
    c.seq_lens = seq_lens(shape, seed, lens)
    return c


@dataclass
class PackedCase:
    """Host tensors of one unroll over a PACKED batch (sequence b = rows [cu[b], cu[b+1]),
    include/ttt_attn.h cu_seqlens): q / dout per step [N,Hq,D], k / v lists [N,Hkv,D]."""
    cu: np.ndarray
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    ttt_steps: int
    dtype: torch.dtype
    q: list = field(default_factory=list)
    dout: list = field(default_factory=list)
    k_base: torch.Tensor = None
    v_base: torch.Tensor = None
    k_steps: list = field(default_factory=list)
    v_steps: list = field(default_factory=list)

    @property
    def rows(self) -> int:
        return int(self.cu[-1])


def make_packed_case(lens, num_q_heads: int, num_kv_heads: int, head_dim: int, ttt_steps: int,
                     dtype: torch.dtype = torch.bfloat16, seed: int = 0) -> PackedCase:
    """Same recipe as make_case (N(0,1) draws rounded to the storage dtype), packed rows."""
    lens = np.asarray(lens, dtype=np.int64)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    N = int(cu[-1])
    rng = np.random.default_rng(seed)
    c = PackedCase(cu, num_q_heads, num_kv_heads, head_dim, ttt_steps, dtype)
    kv, qs = (N, num_kv_heads, head_dim), (N, num_q_heads, head_dim)
    c.k_base = to_storage(_normal(rng, kv), dtype)
    c.v_base = to_storage(_normal(rng, kv), dtype)
    for _ in range(max(ttt_steps - 1, 0)):
        c.k_steps.append(to_storage(_normal(rng, kv), dtype))
        c.v_steps.append(to_storage(_normal(rng, kv), dtype))
    for _ in range(ttt_steps):
        c.q.append(to_storage(_normal(rng, qs), dtype))
    rng_do = np.random.default_rng(seed + 1)
    for _ in range(ttt_steps):
        c.dout.append(to_storage(_normal(rng_do, qs), dtype))
    return c


def packed_lens(n: int, max_len: int, seed: int) -> np.ndarray:
    """Lengths of a packed batch: T_b ~ U[max_len/4, max_len] (the padded recipe's mix, seed + 2)."""
    rng = np.random.default_rng(seed + 2)
    return rng.integers(max(1, max_len // 4), max_len + 1, size=n, dtype=np.int64)


def sample_rows(shape: Shape, n_per_head: int, seed: int) -> np.ndarray:
    """Boolean row selector [B, Hq, L] with n_per_head random rows per (b, h),
    always including rows 0 and L-1 (the ends of the causal range)."""
    rng = np.random.default_rng(seed + 3)
    sel = np.zeros((shape.batch, shape.num_q_heads, shape.seq_len), dtype=bool)
    for b in range(shape.batch):
        for h in range(shape.num_q_heads):
            idx = rng.choice(shape.seq_len, size=min(n_per_head, shape.seq_len), replace=False)
            sel[b, h, idx] = True
            sel[b, h, 0] = True
            sel[b, h, shape.seq_len - 1] = True
    return sel


# ---- loss inputs (recipe in DESIGN.md §4) ----

# Llama-3.1-8B EAGLE-3 draft: 32000-token draft vocabulary; one row per
# (sequence, position) of a TTT step: B * L = 8 * 2048 rows.
LOSS_CONFIGS = {
    "tiny": (128, 1000),
    "llama8b": (8 * 2048, 32000),
}


@dataclass
class LossCase:
    z: torch.Tensor       # [N, V] logits, storage dtype (CPU)
    p: torch.Tensor       # [N, V] target probabilities, storage dtype (CPU)
    mask: torch.Tensor    # [N] uint8 loss-position mask
    g_rows: torch.Tensor  # [N] fp32 per-row weights


def make_loss_case(rows: int, vocab: int, dtype: torch.dtype = torch.bfloat16, seed: int = 0,
                   z_scale: float = 3.0, mask_mode: str = "padded") -> LossCase:
    """Seeded loss inputs: draft logits z ~ N(0, z_scale^2); target rows p = lam e_k + (1 - lam) d
    with a random top token k, lam ~ U[0.3, 0.95] and a heavy tail d = u^8 / sum(u^8),
    u ~ U(0, 1) (one dominant token plus a long tail, like a language model's next-token
    distribution; stored after rounding, so rows sum to 1 only up to the storage rounding);
    mask: "all", or "padded" = the last U[0, rows/4) rows plus ~10% scattered rows false
    (padding and non-assistant positions); per-row weights g_rows ~ U[0.5, 1.5).
    Seeds: z `seed`, p `seed+1`, mask / weights `seed+2`. Drawn in row chunks (bounded memory)."""
    rz = np.random.default_rng(seed)
    rp = np.random.default_rng(seed + 1)
    z = torch.empty((rows, vocab), dtype=dtype)
    p = torch.empty((rows, vocab), dtype=dtype)
    chunk = max(1, (1 << 26) // vocab)
    for r0 in range(0, rows, chunk):
        n = min(chunk, rows - r0)
        z[r0:r0 + n] = to_storage(_normal(rz, (n, vocab), z_scale), dtype)
        lam = rp.uniform(0.3, 0.95, size=n).astype(np.float32)
        top = rp.integers(0, vocab, size=n)
        d = rp.random((n, vocab), dtype=np.float32) ** 8
        d *= ((1.0 - lam) / d.sum(axis=1, dtype=np.float64)).astype(np.float32)[:, None]
        d[np.arange(n), top] += lam
        p[r0:r0 + n] = to_storage(d, dtype)
    rm = np.random.default_rng(seed + 2)
    mask = np.ones(rows, dtype=np.uint8)
    if mask_mode == "padded":
        pad = int(rm.integers(0, max(rows // 4, 1)))
        mask[rows - pad:] = 0
        mask[rm.random(rows) < 0.1] = 0
        if mask.sum() == 0:
            mask[0] = 1
    g_rows = rm.uniform(0.5, 1.5, size=rows).astype(np.float32)
    return LossCase(z, p, torch.from_numpy(mask), torch.from_numpy(g_rows))


# ---- tree-attention verification inputs ----

@dataclass
class TreeCase:
    q: torch.Tensor        # [B, n, Hq, D]
    k: torch.Tensor        # [B, Lk, Hkv, D]: prefix rows then the tree's own rows
    v: torch.Tensor
    parents: torch.Tensor  # int32 [B, n], topological (parent < child), -1 = context tip
    prefix_lens: list


def make_tree_case(batch: int, n: int, prefix_lens, num_q_heads: int, num_kv_heads: int, head_dim: int,
                   dtype=torch.bfloat16, seed: int = 0, kv_len=None) -> TreeCase:
    """Seeded draft trees: node t's parent is uniform over {-1, 0, .., t-1} with -1 drawn at
    probability 1/8 (EAGLE-style wide-and-shallow trees hang most nodes off a few roots);
    q, k, v ~ N(0, 1) -> storage dtype; rows past P_b + n of the cache are noise (never attended).
    Seeds: tensors `seed`, parents `seed + 1`."""
    rng = np.random.default_rng(seed)
    Lk = kv_len or (max(prefix_lens) + n)
    q = to_storage(_normal(rng, (batch, n, num_q_heads, head_dim)), dtype)
    k = to_storage(_normal(rng, (batch, Lk, num_kv_heads, head_dim)), dtype)
    v = to_storage(_normal(rng, (batch, Lk, num_kv_heads, head_dim)), dtype)
    rp = np.random.default_rng(seed + 1)
    par = np.full((batch, n), -1, dtype=np.int32)
    for b in range(batch):
        for t in range(1, n):
            par[b, t] = -1 if rp.random() < 0.125 else int(rp.integers(0, t))
    return TreeCase(q, k, v, torch.from_numpy(par), [int(x) for x in prefix_lens])
