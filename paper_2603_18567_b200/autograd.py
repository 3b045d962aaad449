"""torch.autograd wrappers over the C-ABI (argument marshalling only; every step of
the computation runs in libtttattn.so's kernels). SURVEY.md §8(b) "Python side".

``ttt_attention(q, k_base, v_base, k_steps, v_steps, step)``
    TTT step ``j = step`` (Alg. 1/2): out [B, L, Hq, D].
    Backward calls ``ttt_attn_bwd`` for this step in overwrite mode; autograd itself sums
    the contributions of the S steps of an unroll into K_0 / V_0 / K_i / V_i (the kernel's
    TTT_ACCUMULATE_DKV path is the fused alternative bench.py times). Gradients of K/V come
    out of the kernel in fp32 and are returned in the inputs' dtype.

``ttt_attention_unroll(qs, k_base, v_base, k_steps, v_steps)``
    All S steps of one unroll as one autograd node: forward = S ttt_attn_fwd calls, backward =
    one ttt_attn_bwd_unroll call whose fp32 dK / dV accumulators sum the steps' contributions
    before a single cast to the inputs' dtype (the per-step wrapper lets autograd add S bf16
    gradients instead).

``qkv_rope_split(qkv, num_q_heads, num_kv_heads, rope_base)``
    The fused q/k/v projection output -> RoPE'd q and the step's K / V (ttt_qkv_rope_split);
    backward = ttt_qkv_rope_join_bwd (the rotation's adjoint).

``soft_label_loss(z, p, mask)``
    Masked soft-label log-softmax loss (reading R17) whose backward is Alg. 3
     IN PLACE: the logits buffer z is overwritten with dL/dz and handed
    to autograd as the gradient, so no [N, V] gradient buffer is allocated. z must not be
    read again after backward (its storage then holds the gradient) — the paper's trick.
"""
from __future__ import annotations

from typing import Optional, Sequence

import torch

from . import _lib as L


class _TTTAttention(torch.autograd.Function):
    @staticmethod
    def forward(ctx, step: int, seq_lens, scale: float, q, k_base, v_base, *kv_steps):
        j = int(step)
        c = lambda t: t.contiguous()  # the C-ABI takes raw row-major pointers (views are copied here)
        q, k_base, v_base = c(q), c(k_base), c(v_base)
        k_steps, v_steps = [c(t) for t in kv_steps[:j]], [c(t) for t in kv_steps[j:2 * j]]
        if isinstance(seq_lens, tuple):  # ("packed", cu_seqlens): q [N, Hq, D], K / V [N, Hkv, D]
            N, Hq, D = q.shape
            dt = L.TTT_FP32_CHECK if q.dtype == torch.float32 else L.TTT_BF16
            desc = L.packed_desc(seq_lens[1], Hq, k_base.shape[1], D, dtype=dt, softmax_scale=scale)
            lse_shape = (Hq, N)
        else:
            desc = L.desc_for(q, k_base, seq_lens=seq_lens, softmax_scale=scale)
            B, Lq, Hq, D = q.shape
            lse_shape = (B, Hq, Lq)
        out = torch.empty_like(q)
        out_lo = torch.empty_like(q) if q.dtype == torch.bfloat16 else None
        lse = torch.empty(lse_shape, dtype=torch.float32, device=q.device)
        L.ttt_attn_fwd(desc, j, q, k_base, v_base, k_steps, v_steps, out, lse, out_lo=out_lo)
        ctx.j, ctx.desc = j, desc
        ctx.save_for_backward(q, k_base, v_base, out, lse, *([out_lo] if out_lo is not None else []),
                              *k_steps, *v_steps)
        ctx.has_lo = out_lo is not None
        return out

    @staticmethod
    def backward(ctx, dout):
        j, desc = ctx.j, ctx.desc
        saved = ctx.saved_tensors
        q, k_base, v_base, out, lse = saved[:5]
        rest = saved[5:]
        out_lo = rest[0] if ctx.has_lo else None
        rest = rest[1:] if ctx.has_lo else rest
        k_steps, v_steps = list(rest[:j]), list(rest[j:2 * j])
        dout = dout.contiguous()
        dq = torch.empty_like(q)
        f32 = lambda t: torch.empty(t.shape, dtype=torch.float32, device=t.device)
        dk, dv = f32(k_base), f32(v_base)
        dks, dvs = [f32(t) for t in k_steps], [f32(t) for t in v_steps]
        ws = torch.empty(max(L.ttt_attn_workspace_size(desc, j, True), 16), dtype=torch.uint8, device=q.device)
        L.ttt_attn_bwd(desc, j, q, k_base, v_base, k_steps, v_steps, out, lse, dout, dq, dk, dv, dks, dvs,
                       flags=0, workspace=ws, out_lo=out_lo)
        cast = lambda g, like: g.to(like.dtype)
        grads = [cast(dk, k_base), cast(dv, v_base)] + [cast(g, t) for g, t in zip(dks, k_steps)] + \
                [cast(g, t) for g, t in zip(dvs, v_steps)]
        return (None, None, None, dq, *grads)


def ttt_attention(q: torch.Tensor, k_base: torch.Tensor, v_base: torch.Tensor,
                  k_steps: Sequence[torch.Tensor], v_steps: Sequence[torch.Tensor], step: int,
                  seq_lens: Optional[Sequence[int]] = None, softmax_scale: float = 0.0,
                  cu_seqlens: Optional[Sequence[int]] = None) -> torch.Tensor:
    """Differentiable TTT attention of step ``step`` (uses k_steps[:step], v_steps[:step]).
    BSHD tensors, contiguous, on the GPU: q [B, L, Hq, D], K/V [B, L, Hkv, D]; or, with
    ``cu_seqlens`` (B + 1 host offsets), a packed batch: q [N, Hq, D], K/V [N, Hkv, D]."""
    j = int(step)
    ks, vs = list(k_steps[:j]), list(v_steps[:j])
    if len(ks) != j or len(vs) != j:
        raise ValueError(f"step {j} needs {j} step K/V tensors, got {len(ks)} / {len(vs)}")
    if cu_seqlens is not None:
        if seq_lens is not None:
            raise ValueError("pass seq_lens (padded) or cu_seqlens (packed), not both")
        lens = ("packed", tuple(int(x) for x in cu_seqlens))
    else:
        lens = None if seq_lens is None else [int(x) for x in seq_lens]
    return _TTTAttention.apply(j, lens, float(softmax_scale), q, k_base, v_base, *ks, *vs)


class _TTTAttentionUnroll(torch.autograd.Function):
    @staticmethod
    def forward(ctx, S: int, seq_lens, scale: float, k_base, v_base, *rest):
        c = lambda t: t.contiguous()
        k_base, v_base = c(k_base), c(v_base)
        qs = [c(t) for t in rest[:S]]
        ks, vs = [c(t) for t in rest[S:2 * S - 1]], [c(t) for t in rest[2 * S - 1:3 * S - 2]]
        desc = L.desc_for(qs[0], k_base, seq_lens=seq_lens, softmax_scale=scale)
        B, Lq, Hq, D = qs[0].shape
        outs, los, lses = [], [], []
        for j in range(S):
            out = torch.empty_like(qs[j])
            lo = torch.empty_like(qs[j]) if qs[j].dtype == torch.bfloat16 else None
            lse = torch.empty((B, Hq, Lq), dtype=torch.float32, device=qs[j].device)
            L.ttt_attn_fwd(desc, j, qs[j], k_base, v_base, ks, vs, out, lse, out_lo=lo)
            outs.append(out)
            los.append(lo)
            lses.append(lse)
        ctx.S, ctx.desc, ctx.has_lo = S, desc, los[0] is not None
        ctx.save_for_backward(k_base, v_base, *qs, *ks, *vs, *outs, *lses, *(los if ctx.has_lo else []))
        return tuple(outs)

    @staticmethod
    def backward(ctx, *douts):
        S, desc = ctx.S, ctx.desc
        t = ctx.saved_tensors
        k_base, v_base = t[0], t[1]
        o = 2
        qs = list(t[o:o + S]); o += S
        ks = list(t[o:o + S - 1]); o += S - 1
        vs = list(t[o:o + S - 1]); o += S - 1
        outs = list(t[o:o + S]); o += S
        lses = list(t[o:o + S]); o += S
        los = list(t[o:o + S]) if ctx.has_lo else None
        douts = [d.contiguous() if d is not None else torch.zeros_like(outs[j]) for j, d in enumerate(douts)]
        dqs = [torch.empty_like(q) for q in qs]
        f32 = lambda x: torch.empty(x.shape, dtype=torch.float32, device=x.device)
        dk, dv = f32(k_base), f32(v_base)
        dks, dvs = [f32(x) for x in ks], [f32(x) for x in vs]
        ws = torch.empty(max(L.ttt_attn_bwd_unroll_workspace_size(desc, S), 16), dtype=torch.uint8,
                         device=k_base.device)
        L.ttt_attn_bwd_unroll(desc, qs, k_base, v_base, ks, vs, outs, lses, douts, dqs, dk, dv, dks, dvs,
                              flags=0, workspace=ws, out_lo=los)
        cast = lambda g, like: g.to(like.dtype)
        return (None, None, None, cast(dk, k_base), cast(dv, v_base), *dqs,
                *[cast(g, x) for g, x in zip(dks, ks)], *[cast(g, x) for g, x in zip(dvs, vs)])


def ttt_attention_unroll(qs: Sequence[torch.Tensor], k_base: torch.Tensor, v_base: torch.Tensor,
                         k_steps: Sequence[torch.Tensor], v_steps: Sequence[torch.Tensor],
                         seq_lens: Optional[Sequence[int]] = None, softmax_scale: float = 0.0):
    """Differentiable TTT unroll: returns [out_0, ..., out_{S-1}] for S = len(qs) steps
    (step j uses k_steps[:j], v_steps[:j]); backward is one ttt_attn_bwd_unroll call."""
    S = len(qs)
    if S < 1 or S > L.TTT_MAX_UNROLL:
        raise ValueError(f"1 <= steps <= {L.TTT_MAX_UNROLL}")
    ks, vs = list(k_steps[:S - 1]), list(v_steps[:S - 1])
    if len(ks) != S - 1 or len(vs) != S - 1:
        raise ValueError(f"{S} steps need {S - 1} step K/V tensors")
    lens = None if seq_lens is None else [int(x) for x in seq_lens]
    return list(_TTTAttentionUnroll.apply(S, lens, float(softmax_scale), k_base, v_base, *qs, *ks, *vs))


class _QkvRopeSplit(torch.autograd.Function):
    @staticmethod
    def forward(ctx, qkv, Hq: int, Hkv: int, base: float, positions):
        qkv = qkv.contiguous()
        B, Lr, H, D = qkv.shape
        d = L.rope_desc(B, Lr, Hq, Hkv, D, base)
        ws = torch.empty(max(L.ttt_rope_workspace_size(d, positions is not None), 16), dtype=torch.uint8,
                         device=qkv.device)
        q = torch.empty(B, Lr, Hq, D, dtype=qkv.dtype, device=qkv.device)
        k = torch.empty(B, Lr, Hkv, D, dtype=qkv.dtype, device=qkv.device)
        v = torch.empty_like(k)
        L.ttt_qkv_rope_split(d, qkv, q, k, v, ws, positions=positions)
        ctx.d, ctx.ws, ctx.positions, ctx.shape = d, ws, positions, qkv.shape
        return q, k, v

    @staticmethod
    def backward(ctx, dq, dk, dv):
        z = lambda g, like_shape: g.contiguous() if g is not None else torch.zeros(
            like_shape, dtype=torch.bfloat16, device=ctx.ws.device)
        B, Lr, H, D = ctx.shape
        dq = z(dq, (B, Lr, ctx.d.num_q_heads, D))
        dk = z(dk, (B, Lr, ctx.d.num_kv_heads, D))
        dv = z(dv, (B, Lr, ctx.d.num_kv_heads, D))
        dqkv = torch.empty(ctx.shape, dtype=dq.dtype, device=dq.device)
        L.ttt_qkv_rope_join_bwd(ctx.d, dq, dk, dv, dqkv, ctx.ws, positions=ctx.positions)
        return dqkv, None, None, None, None


def qkv_rope_split(qkv: torch.Tensor, num_q_heads: int, num_kv_heads: int, rope_base: float = 500000.0,
                   positions: Optional[torch.Tensor] = None):
    """qkv bf16 [B, L, Hq + 2 Hkv, D] -> (q, k, v): q and k RoPE'd at positions 0..L-1 (or the given
    int32 [B, L] positions), v copied; differentiable (backward = the rotation's adjoint)."""
    return _QkvRopeSplit.apply(qkv, int(num_q_heads), int(num_kv_heads), float(rope_base), positions)


class _SoftLabelLoss(torch.autograd.Function):
    @staticmethod
    def forward(ctx, z, p, mask, g_rows):
        if not z.is_contiguous():
            raise ValueError("soft_label_loss: z must be contiguous (its buffer is overwritten in place by "
                             "the backward; a copy would defeat Alg. 3)")
        p, mask = p.contiguous(), mask.contiguous()
        g_rows = None if g_rows is None else g_rows.contiguous()
        desc = L.loss_desc_for(z)
        ws = torch.empty(L.ttt_loss_workspace_size(desc), dtype=torch.uint8, device=z.device)
        stats = torch.empty(2, dtype=torch.float64, device=z.device)
        L.ttt_loss_fwd(desc, z, p, mask, stats, ws)
        ctx.desc, ctx.ws, ctx.done = desc, ws, False
        ctx.save_for_backward(z, p, mask, g_rows)
        return stats[0].to(torch.float32)

    @staticmethod
    def backward(ctx, g):
        if ctx.done:
            raise RuntimeError("soft_label_loss: backward ran already; z now holds dL/dz (Alg. 3 in place), "
                               "so a second backward (retain_graph=True) cannot recompute it")
        z, p, mask, g_rows = ctx.saved_tensors
        ws = ctx.ws
        # Alg. 3 in place: z <- dL/dz. The upstream scalar g enters as g_scale; it is read on the
        # host (one sync) because the C-ABI takes g_scale by value.
        L.ttt_loss_bwd_inplace(ctx.desc, z, p, mask, ws, g_scale=float(g), flags=L.TTT_LOSS_MEAN,
                               g_rows=g_rows)
        ctx.done = True
        # z's storage now holds the gradient: bump its version counter so any other autograd node
        # that saved z (e.g. a z-loss on the same logits) fails loudly instead of reading dL/dz
        torch.autograd.graph.increment_version(z)
        return z, None, None, None


def soft_label_loss(z: torch.Tensor, p: torch.Tensor, mask: Optional[torch.Tensor] = None,
                    g_rows: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Masked mean soft-label loss over rows of z [N, V] (bf16 or fp32) against target
    probabilities p [N, V]; mask uint8 [N] (None = all rows), g_rows optional fp32 [N] row
    weights. Backward overwrites z with dL/dz (Alg. 3, in place) and returns it as z's grad."""
    if mask is None:
        mask = torch.ones(z.shape[0], dtype=torch.uint8, device=z.device)
    return _SoftLabelLoss.apply(z, p, mask.to(torch.uint8), g_rows)
