"""Shared helpers for the -m gpu parity tests: run the CUDA path through the
C-ABI binding, run the oracle on the same bits, compare with allclose
semantics |gpu - oracle| <= atol + rtol * |oracle|."""
from __future__ import annotations

import os

import numpy as np
import torch

import oracle
import paper_2603_18567_b200 as ttt

TOL_BF16 = dict(atol=2e-2, rtol=1e-2)   # north_star (BASELINE.json)
TOL_FP32 = dict(atol=1e-5, rtol=1e-5)   # north_star fp32 check mode


def np32(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy()


def report(name, got, want, atol, rtol):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    err = np.abs(got - want)
    bad = err > atol + rtol * np.abs(want)
    msg = (f"{name}: max_abs={err.max():.3e} max_rel={(err / (np.abs(want) + 1e-30)).max():.3e} "
           f"violations={int(bad.sum())}/{bad.size}")
    return bad.any(), msg


def assert_close_sum(name, got, parts, atol, rtol):
    """Accumulated result vs a sum of per-call oracle contributions: each call is
    allowed atol + rtol*|part|, so the sum is held to the sum of those bounds
    (triangle inequality; reading R16)."""
    got = np.asarray(got, np.float64)
    want = np.sum(parts, axis=0)
    bound = sum(atol + rtol * np.abs(np.asarray(x, np.float64)) for x in parts)
    assert not np.isnan(got).any(), f"{name}: NaN in GPU result"
    err = np.abs(got - want)
    bad = err > bound
    assert not bad.any(), f"{name}: max_abs={err.max():.3e} violations={int(bad.sum())}/{bad.size} (n={len(parts)})"


def assert_close(name, got, want, atol, rtol, mask=None):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    if mask is not None:
        got, want = got[mask], want[mask]
    assert not np.isnan(got).any(), f"{name}: NaN in GPU result"
    failed, msg = report(name, got, want, atol, rtol)
    assert not failed, msg
    return msg


class DeviceCase:
    """Device copies of a Case plus output buffers for every step."""

    def __init__(self, case, dev="cuda"):
        self.case = case
        s = case.shape
        self.dt = case.dtype
        to = lambda t: t.to(dev).contiguous()
        self.q = [to(x) for x in case.q]
        self.dout = [to(x) for x in case.dout]
        self.k = to(case.k_base)
        self.v = to(case.v_base)
        self.ks = [to(x) for x in case.k_steps]
        self.vs = [to(x) for x in case.v_steps]
        self.lens = [int(x) for x in case.seq_lens]
        self.desc = ttt.desc_for(self.q[0], self.k, seq_lens=self.lens)
        self.gdt = torch.float32  # dk/dv accumulators are fp32 in both modes
        self.dev = dev

    def fwd(self, j, stream=None):
        s = self.case.shape
        out = torch.empty(s.q_shape, dtype=self.dt, device=self.dev)
        lse = torch.empty((s.batch, s.num_q_heads, s.seq_len), dtype=torch.float32, device=self.dev)
        # TTT_TEST_NO_OUTLO=1: run without the O - bf16(O) residual (Delta from the bf16 out alone)
        use_lo = self.dt == torch.bfloat16 and os.environ.get("TTT_TEST_NO_OUTLO", "0") != "1"
        self.out_lo = torch.empty_like(out) if use_lo else None
        ttt.ttt_attn_fwd(self.desc, j, self.q[j], self.k, self.v, self.ks, self.vs, out, lse,
                         out_lo=self.out_lo, stream=stream)
        return out, lse

    def alloc_grads(self, nsteps):
        s = self.case.shape
        z = lambda: torch.zeros(s.kv_shape, dtype=self.gdt, device=self.dev)
        return {"dk_base": z(), "dv_base": z(), "dk_steps": [z() for _ in range(nsteps)],
                "dv_steps": [z() for _ in range(nsteps)]}

    def bwd(self, j, out, lse, grads, accumulate, dout=None):
        s = self.case.shape
        dq = torch.empty(s.q_shape, dtype=self.dt, device=self.dev)
        wsb = ttt.ttt_attn_workspace_size(self.desc, j, True)
        ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device=self.dev)
        ttt.ttt_attn_bwd(self.desc, j, self.q[j], self.k, self.v, self.ks, self.vs, out, lse,
                         self.dout[j] if dout is None else dout, dq, grads["dk_base"], grads["dv_base"],
                         grads["dk_steps"], grads["dv_steps"],
                         flags=ttt.TTT_ACCUMULATE_DKV if accumulate else 0, workspace=ws,
                         out_lo=getattr(self, "out_lo", None))
        return dq


def oracle_inputs(case, j):
    return (np32(case.q[j]), np32(case.k_base), np32(case.v_base),
            [np32(x) for x in case.k_steps[:j]], [np32(x) for x in case.v_steps[:j]])
