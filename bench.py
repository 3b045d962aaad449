#!/usr/bin/env python
"""bench.py — TTT unrolled attention fwd+bwd on B200 (the driver's bench contract).

One bench "step" = one optimizer step of the EAGLE-3 draft layer's TTT attention:
the rank's micro-batches, each one TTT unroll (7 forward calls j = 0..6, then 7
backward calls j = 6..0, the first overwriting, the rest accumulating dK/dV), all
through the C-ABI (libtttattn.so), then ONE draft-gradient exchange.

  N = 1 (default --config llama8b): BASELINE.json configs[1], the Llama-3.1-8B draft
        shape B=8, L=2048, 32 q / 8 kv heads, head_dim 128, ttt_steps 7, bf16 — one
        micro-batch per step.
  N > 1 (default --config dp): BASELINE.json configs[4], the DP scaling sweep — global
        batch 64 x L=4096 per optimizer step, 64/N sequences per rank as micro-batches
        of 8 (strong scaling), the draft-layer gradient bucket all-reduced over NCCL once
        per optimizer step after the last micro-batch's backward (the draft's parameters
        are shared by every TTT step and micro-batch, so their gradients are final only
        then). The N = 1 point of this sweep is reported beside the headline as
        next_rows.dp_sweep_n1.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0. See DESIGN.md §6 for every field.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_18567_b200.inputs import CONFIGS, Shape  # noqa: E402

METRIC = "TTT attn fwd+bwd tokens/sec (Llama-3.1-8B EAGLE-3 draft shape, ttt_steps=7)"
UNIT = "tokens/s"
# EAGLE-3 draft layer of Llama-3.1-8B: fc 3d->d, q/k/v/o, MLP 14336, norms, 32000 head
DRAFT_PARAMS = 424_700_000
LOSS_ROWS, LOSS_VOCAB = 8 * 2048, 32000  # one TTT step's rows of the Llama draft, 32000-token draft vocab


def alg_pairs(s: Shape, seq_lens=None):
    """Allowed (q, k) pairs of one unroll, all b and q-heads:
    per (b, h, step j): T(T+1)/2 + (L-T)T + j*T."""
    L = s.seq_len
    lens = [L] * s.batch if seq_lens is None else list(seq_lens)
    base = sum(T * (T + 1) // 2 + (L - T) * T for T in lens)
    diag = sum(lens)
    per_step = [s.num_q_heads * (base + j * diag) for j in range(s.ttt_steps)]
    base_only = s.num_q_heads * base
    return per_step, base_only


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi sampling of SM clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- oracle legs
def oracle_sample(shape: Shape, target_s: float, seed: int = 0):
    """Time the fp64 CPU oracle (oracle/, test infrastructure) on a bounded
    sample of the workload: sequence 0, all query heads, `n` evenly spaced
    query rows per head, all ttt_steps forward + backward. The oracle's cost
    per row is uniform (it is dense over all (j+1)L keys), so the sample
    scales: tokens-equivalent = n rows of one sequence with all heads."""
    import oracle
    rng = np.random.default_rng(seed)
    L, Hq, Hkv, D, S = shape.seq_len, shape.num_q_heads, shape.num_kv_heads, shape.head_dim, shape.ttt_steps
    bf = lambda a: torch.from_numpy(a).to(torch.bfloat16).float().numpy()
    q = [bf(rng.standard_normal((1, L, Hq, D), dtype=np.float32)) for _ in range(S)]
    do = [bf(rng.standard_normal((1, L, Hq, D), dtype=np.float32)) for _ in range(S)]
    kb = bf(rng.standard_normal((1, L, Hkv, D), dtype=np.float32))
    vb = bf(rng.standard_normal((1, L, Hkv, D), dtype=np.float32))
    ks = [bf(rng.standard_normal((1, L, Hkv, D), dtype=np.float32)) for _ in range(S - 1)]
    vs = [bf(rng.standard_normal((1, L, Hkv, D), dtype=np.float32)) for _ in range(S - 1)]
    threads = oracle.default_threads()

    def run(n_rows):
        sel = np.zeros((1, Hq, L), dtype=bool)
        sel[:, :, np.linspace(0, L - 1, n_rows).astype(int)] = True
        t0 = time.perf_counter()
        for j in range(S):
            oracle.fwd(q[j], kb, vb, ks[:j], vs[:j], row_sel=sel, nthreads=threads)
        for j in reversed(range(S)):
            oracle.bwd(q[j], kb, vb, ks[:j], vs[:j], do[j], row_sel=sel, nthreads=threads)
        return time.perf_counter() - t0

    t1 = run(1)  # calibration: one row per head
    n = int(max(1, min(L, target_s / max(t1, 1e-6))))
    return n, threads, run


def run_reference(args, shape: Shape, rank: int, world: int):
    """--impl reference: the oracle as it stands, timed on this box's host cores."""
    if rank != 0:
        return
    n, threads, run = oracle_sample(shape, target_s=2.0)
    for _ in range(args.warmup):
        run(n)
    times = [run(n) for _ in range(args.steps)]
    sec = sum(times) / len(times)
    value = n / sec
    sample = (f"sequence 0 of {shape.batch}, all {shape.num_q_heads} q heads, {n} of {shape.seq_len} rows, "
              f"all {shape.ttt_steps} TTT steps fwd+bwd (dense fp64 oracle); tokens-equivalent = {n} per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "strong" if args.config == "dp" else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(shape, world, args.config),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def global_batch_of(cfg: str, shape: Shape, world: int) -> int:
    """Sequences per optimizer step, all ranks: configs[4] fixes 64 (strong scaling); the other
    configs run one micro-batch per rank (weak scaling)."""
    return 64 if cfg == "dp" else shape.batch * world


def workload_config(shape: Shape, world: int, cfg: str = "llama8b"):
    gb = global_batch_of(cfg, shape, world)
    names = {"llama8b": "llama3.1-8b-eagle3-draft TTT attention unroll (fwd j=0..6 + bwd j=6..0)",
             "dp": "DP sweep (BASELINE configs[4]): llama3.1-8b-eagle3-draft TTT attention, global batch 64 x "
                   "L=4096 per optimizer step, micro-batches of 8, one NCCL grad all-reduce per step"}
    per_rank = gb // world
    return {"workload": names.get(cfg, f"{cfg} TTT attention unroll"), "config": cfg,
            "batch_per_gpu": per_rank, "micro_batch": shape.batch,
            "micro_batches_per_rank": -(-per_rank // shape.batch), "global_batch": gb,
            "seq_len": shape.seq_len, "num_q_heads": shape.num_q_heads, "num_kv_heads": shape.num_kv_heads,
            "head_dim": shape.head_dim, "ttt_steps": shape.ttt_steps, "seq_lens": "full (T_b = L)",
            "parallelism": f"dp{world}",
            "l2": "inputs larger than L2 (~5 GB touched per unroll vs 126 MB L2); no flush in the headline; "
                  "cold_l2 = the same unroll after a 512 MB L2 flush"}


# --------------------------------------------------------------------------- our arm
class Unroll:
    """Device buffers of one per-GPU unroll + the C-ABI calls of one step."""

    def __init__(self, shape: Shape, seed: int, dev, bwd_unroll: bool = False, seq_lens=None, packed: bool = False):
        """seq_lens: T_b per sequence (padded layout [B][L] with those lengths, or with packed=True the
        packed layout: the sequences back to back, [sum T_b][H][D], include/ttt_attn.h cu_seqlens)."""
        import paper_2603_18567_b200 as ttt
        self.ttt = ttt
        self.s = s = shape
        S = s.ttt_steps
        if packed:
            cu = [0]
            for T in seq_lens:
                cu.append(cu[-1] + int(T))
            N = cu[-1]
            q_shape, kv_shape, lse_shape = (N, s.num_q_heads, s.head_dim), (N, s.num_kv_heads, s.head_dim), \
                (s.num_q_heads, N)
        else:
            q_shape, kv_shape, lse_shape = s.q_shape, s.kv_shape, (s.batch, s.num_q_heads, s.seq_len)
        g = torch.Generator(device=dev).manual_seed(seed)
        mk = lambda shp: torch.randn(shp, device=dev, generator=g, dtype=torch.float32).to(torch.bfloat16)
        self.q = [mk(q_shape) for _ in range(S)]
        self.do = [mk(q_shape) for _ in range(S)]
        self.k, self.v = mk(kv_shape), mk(kv_shape)
        self.ks = [mk(kv_shape) for _ in range(S - 1)]
        self.vs = [mk(kv_shape) for _ in range(S - 1)]
        self.out = [torch.empty(q_shape, dtype=torch.bfloat16, device=dev) for _ in range(S)]
        self.out_lo = [torch.empty(q_shape, dtype=torch.bfloat16, device=dev) for _ in range(S)]
        self.lse = [torch.empty(lse_shape, device=dev) for _ in range(S)]
        self.dq = [torch.empty(q_shape, dtype=torch.bfloat16, device=dev) for _ in range(S)]
        z = lambda: torch.zeros(kv_shape, dtype=torch.float32, device=dev)
        self.dk, self.dv = z(), z()
        self.dks = [z() for _ in range(S - 1)]
        self.dvs = [z() for _ in range(S - 1)]
        if packed:
            self.desc = ttt.packed_desc(cu, s.num_q_heads, s.num_kv_heads, s.head_dim)
        else:
            self.desc = ttt.make_desc(s.batch, s.seq_len, s.num_q_heads, s.num_kv_heads, s.head_dim,
                                      seq_lens=seq_lens)
        self.ws = torch.empty(ttt.ttt_attn_workspace_size(self.desc, S - 1, True), dtype=torch.uint8, device=dev)
        self.inputs = self.q + self.do + [self.k, self.v] + self.ks + self.vs
        # every result of the unroll (what a caller reads back): out_j, lse_j, dq_j, dK_0, dV_0, dK_i, dV_i
        self.outputs = self.out + self.lse + self.dq + [self.dk, self.dv] + self.dks + self.dvs
        self.bwd_unroll = bwd_unroll  # one ttt_attn_bwd_unroll call for the S backward calls
        if bwd_unroll:
            self.ws_unroll = torch.empty(ttt.ttt_attn_bwd_unroll_workspace_size(self.desc, S), dtype=torch.uint8,
                                         device=dev)

    def step(self, stream, marks=None):
        """One unroll. `marks` (optional): dict of CUDA events recorded around every call,
        marks[("fwd", j)] / marks[("bwd", j)] = (start, end), for per-step times."""
        t, s = self.ttt, self.s
        S = s.ttt_steps
        ev = lambda key: marks.setdefault(key, (torch.cuda.Event(enable_timing=True),
                                                torch.cuda.Event(enable_timing=True))) if marks is not None else None
        nvtx = torch.cuda.nvtx
        for j in range(S):
            e = ev(("fwd", j))
            nvtx.range_push(f"ttt fwd j={j}")
            if e:
                e[0].record(stream)
            t.ttt_attn_fwd(self.desc, j, self.q[j], self.k, self.v, self.ks, self.vs, self.out[j], self.lse[j],
                           out_lo=self.out_lo[j], stream=stream)
            if e:
                e[1].record(stream)
            nvtx.range_pop()
        if self.bwd_unroll:
            nvtx.range_push("ttt bwd unroll")
            t.ttt_attn_bwd_unroll(self.desc, self.q, self.k, self.v, self.ks, self.vs, self.out, self.lse, self.do,
                                  self.dq, self.dk, self.dv, self.dks, self.dvs, flags=0, workspace=self.ws_unroll,
                                  stream=stream, out_lo=self.out_lo)
            nvtx.range_pop()
            return
        for j in reversed(range(S)):
            e = ev(("bwd", j))
            nvtx.range_push(f"ttt bwd j={j}")
            if e:
                e[0].record(stream)
            t.ttt_attn_bwd(self.desc, j, self.q[j], self.k, self.v, self.ks, self.vs, self.out[j], self.lse[j],
                           self.do[j], self.dq[j], self.dk, self.dv, self.dks, self.dvs,
                           flags=0 if j == S - 1 else t.TTT_ACCUMULATE_DKV, workspace=self.ws, stream=stream,
                           out_lo=self.out_lo[j])
            if e:
                e[1].record(stream)
            nvtx.range_pop()


def pick_peak(peaks, clocks):
    """roofline peak matching the clock record of the timed region: the burst bf16 figure when the
    SMs ran near their max clock (>= 90%), the sustained (power-capped) one otherwise."""
    sm, mx = clocks.get("sm_mhz"), clocks.get("sm_max_mhz")
    if sm is not None and mx and sm >= 0.9 * mx:
        return peaks["bf16_tflops"], "burst"
    return peaks["bf16_tflops_sustained"], "sustained"


def run_ours(args, shape: Shape, rank: int, world: int, local_rank: int):
    import paper_2603_18567_b200 as ttt
    from paper_2603_18567_b200.dp import GradBuckets, OptimizerStep, Zero2Buckets, max_over_ranks
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
    cfg = args.config
    gb = global_batch_of(cfg, shape, world)
    stream = torch.cuda.current_stream(dev)
    S = shape.ttt_steps

    # draft-layer gradient bucket (synthetic stand-in of the draft's parameter gradients), bf16,
    # 7 buckets; exchanged once per optimizer step after the last micro-batch's backward (dp.OptimizerStep)
    Buckets = Zero2Buckets if args.zero2 else GradBuckets
    grads = Buckets(DRAFT_PARAMS if world > 1 else 1, 7, dtype=torch.bfloat16, device=dev)
    params = torch.zeros_like(grads.flat) if args.zero2 and world > 1 else None
    if world > 1:
        grads.flat.normal_()
    opt = OptimizerStep(grads, gb, shape.batch, world, rank, params)
    # micro-batch buffer sets (two alternate when a rank runs several micro-batches per step)
    sets = [Unroll(shape, seed=1234 + rank, dev=dev, bwd_unroll=args.bwd_unroll)]
    if len(opt.micro) > 1:
        sets.append(Unroll(shape, seed=5678 + rank, dev=dev, bwd_unroll=args.bwd_unroll))
    u = sets[0]

    def one_step():
        opt.run(lambda m, lo, hi: sets[m % len(sets)].step(stream))

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()

    # ---------------- timed region ----------------
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        e0.record(stream)
        torch.cuda.nvtx.range_push(f"timed region: {args.steps} steps")
        for _ in range(args.steps):
            one_step()
        torch.cuda.nvtx.range_pop()
        e1.record(stream)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        wall = time.perf_counter() - w0
    ms = max_over_ranks(e0.elapsed_time(e1), device=dev)
    ms_per_step = ms / args.steps
    tokens_per_step = gb * shape.seq_len
    value = tokens_per_step / (ms_per_step / 1e3)
    clocks = clk.summary()

    # ---------------- per-kernel attribution (separate pass, CUDA events on the launch stream) ----------
    prof_steps = 2
    ttt.ttt_attn_profile_begin()
    for _ in range(prof_steps):
        one_step()
    torch.cuda.synchronize()
    kern = ttt.ttt_attn_profile_end()
    launches_per_step = sum(n for _, n in kern.values()) // prof_steps
    # per-TTT-step call times (the paper measures the final step), separate pass
    # (the backward split per step through S ttt_attn_bwd calls: the unroll call has no per-step boundary)
    per_step = {"fwd_ms": [0.0] * S, "bwd_ms": [0.0] * S, "bwd_api": "ttt_attn_bwd per call"}
    reps = 3
    unroll_mode, u.bwd_unroll = u.bwd_unroll, False
    for _ in range(reps):
        marks = {}
        u.step(stream, marks=marks)
        torch.cuda.synchronize()
        for (kind, j), (a, b) in marks.items():
            per_step[f"{kind}_ms"][j] += a.elapsed_time(b) / reps
    u.bwd_unroll = unroll_mode
    # cold L2 (SURVEY.md §8d "report both warm and cold"): one unroll right after a 512 MB write
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    cold = []
    for _ in range(3):
        flush.zero_()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        u.step(stream)
        c1.record(stream)
        torch.cuda.synchronize()
        cold.append(c0.elapsed_time(c1))
    del flush
    warm_unroll_ms = ms_per_step / len(opt.micro) if world == 1 else None

    peaks = load_peaks()
    peak, peak_kind = pick_peak(peaks, clocks)
    per_step_pairs, base_pairs = alg_pairs(shape)
    D = shape.head_dim
    n_unrolls = gb // shape.batch  # unrolls (micro-batches) per optimizer step, all ranks
    flops_step = 12 * D * sum(per_step_pairs) * n_unrolls  # algorithmic: fwd 4D + bwd 8D per allowed pair
    tflops = flops_step / (ms_per_step / 1e3) / 1e12 / world  # per GPU
    # dominant kernel -> roofline
    dom = max(kern.items(), key=lambda kv: kv[1][0])
    dom_name, (dom_ms, dom_n) = dom
    per_launch_flops = {
        "ttt_bwd_sm100_kernel": 8 * D * base_pairs,   # dV, dP, dK, dQ over the base (causal) pairs
        "ttt_fwd_sm100_kernel": 4 * D * base_pairs,   # QK^T, PV over the base pairs
    }
    roof = None
    if dom_name in per_launch_flops:
        avg_ms = dom_ms / dom_n
        achieved = per_launch_flops[dom_name] / (avg_ms / 1e3) / 1e12
        roof = {"kernel": dom_name, "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak,
                "peak_kind": f"bf16 {peak_kind} ({peaks['source']}, MEASURED_PEAKS.json), chosen by the timed "
                             f"region's clock record",
                "frac_of_burst": achieved / peaks["bf16_tflops"],
                "frac_of_sustained": achieved / peaks["bf16_tflops_sustained"], "avg_launch_ms": avg_ms,
                "share_of_step": dom_ms / prof_steps / ms_per_step if world == 1 else None,
                "traffic": ncu_traffic(dom_name), "algorithmic_flops_per_launch": per_launch_flops[dom_name]}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if cfg == "dp" else "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (torch Philox N(0,1) -> bf16, random per rank)",
        "config": workload_config(shape, world, cfg),
        "tflops_per_gpu": tflops, "frac_of_bf16_peak": tflops / peak, "bf16_peak_kind": peak_kind,
        "frac_of_bf16_burst_peak": tflops / peaks["bf16_tflops"],
        "frac_of_bf16_sustained_peak": tflops / peaks["bf16_tflops_sustained"],
        "flops_convention": "algorithmic 12*D per allowed (q,k) pair (fwd 4D + bwd 8D; recompute excluded)",
        # the FlashAttention literature's convention, bwd = 2.5 x fwd (14 D per pair), for comparison
        "tflops_per_gpu_fa_convention": tflops * 14.0 / 12.0,
        "bwd_api": "ttt_attn_bwd_unroll (one call per unroll)" if u.bwd_unroll else "ttt_attn_bwd x S",
        "roofline": roof,
        "kernels_ms_per_step": {k: v[0] / prof_steps for k, v in kern.items()},
        "per_ttt_step_ms": per_step,
        "cold_l2": {"ms_per_unroll": statistics.median(cold), "warm_ms_per_unroll": warm_unroll_ms,
                    "flush": "512 MB device write before each unroll (not timed)"},
        "gpu_launches": launches_per_step * args.steps,
        "grad_allreduce_bytes_per_step": grads.nbytes if world > 1 else 0,
        "grad_exchange": ("zero2 reduce-scatter + param all-gather" if args.zero2 else "bucketed all-reduce (AVG)")
        + ", once per optimizer step after the last micro-batch's backward" if world > 1 else "none (1 GPU)",
        "wall_s_timed_region": wall,
        "clocks": clocks,
    }
    if not args.no_e2e:
        line["e2e"] = run_e2e(sets, opt, stream, args, shape, gb, dev)
    if not args.no_loss:
        line["next_rows"] = {"loss_inplace": run_loss(args, stream, peaks, world)}
        if world == 1:
            line["next_rows"]["longctx"] = run_longctx(args, stream, peaks)
            line["next_rows"]["packed"] = run_packed(args, stream, peaks)
            line["next_rows"]["qwen235b"] = run_config(
                "qwen235b", stream, peaks,
                "Qwen3-235B-A22B draft shape (BASELINE configs[2]): 1 x L=4096, 64/4 heads, D=128, ttt_steps=7, bf16")
            if cfg != "dp":
                del sets, u, opt
                torch.cuda.empty_cache()
                line["next_rows"]["dp_sweep_n1"] = run_dp_n1(args, stream, peaks)
        if world == 1:
            line["next_rows"]["draft_layer_step"] = run_draft(args, stream, peaks,
                                                              warm_unroll_ms if cfg == "llama8b" else None)
        line["next_rows"]["tree_verify"] = run_tree(args, stream, peaks)
        line["next_rows"]["qkv_rope"] = run_rope(args, stream, peaks)
    if rank == 0 and world == 1 and not args.no_cpu:
        n, threads, run = oracle_sample(shape, target_s=15.0)
        sec = run(n)
        line["cpu_baseline"] = {
            "value": n / sec, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": (f"sequence 0 of {shape.batch}, all {shape.num_q_heads} q heads, {n} of {shape.seq_len} rows, "
                       f"all {shape.ttt_steps} TTT steps fwd+bwd (dense fp64 oracle, {sec:.1f} s); "
                       f"tokens-equivalent = {n}")}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_dp_n1(args, stream, peaks):
    """The N = 1 point of the BASELINE configs[4] DP sweep (global batch 64 x L = 4096 per optimizer
    step = 8 micro-batches of 8 on one GPU), so the sweep's scaling can be read against it (the N > 1
    bench lines run this config by default)."""
    from paper_2603_18567_b200.dp import GradBuckets, OptimizerStep
    shape = CONFIGS["dp"]
    dev = stream.device
    sets = [Unroll(shape, seed=91, dev=dev), Unroll(shape, seed=92, dev=dev)]
    opt = OptimizerStep(GradBuckets(1, 7, device=dev), 64, shape.batch, 1, 0)
    one = lambda: opt.run(lambda m, lo, hi: sets[m % 2].step(stream))
    one()
    torch.cuda.synchronize()
    n = 2
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(n):
        one()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    per_step_pairs, _ = alg_pairs(shape)
    tflops = 12 * shape.head_dim * sum(per_step_pairs) * 8 / (ms / 1e3) / 1e12
    del sets
    torch.cuda.empty_cache()
    return {"workload": "BASELINE configs[4] at N=1: global batch 64 x L=4096 (8 micro-batches of 8), 32/8 heads, "
                        "D=128, ttt_steps=7, bf16", "ms_per_step": ms, "tokens_per_s": 64 * 4096 / (ms / 1e3),
            "steps": n, "tflops": tflops, "frac_of_bf16_burst_peak": tflops / peaks["bf16_tflops"],
            "frac_of_bf16_sustained_peak": tflops / peaks["bf16_tflops_sustained"]}


def run_loss(args, stream, peaks, world: int):
    """SURVEY.md §8(f) NEXT #1, measured beside the headline (not part of its step): the masked
    soft-label loss + Alg. 3 in-place backward (include/ttt_loss.h), one fused pass per TTT step,
    on one TTT step's rows of the Llama draft (B L = 16384 rows x 32000 vocab, bf16; z + p = 2.1 GB,
    larger than L2). The timed loop re-runs on the buffer the previous pass overwrote (the cost is
    data-independent: every element takes one exp2 either way)."""
    import paper_2603_18567_b200 as ttt
    rows, vocab = LOSS_ROWS, LOSS_VOCAB
    dev = torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator(device=dev).manual_seed(77)
    z = (torch.randn((rows, vocab), device=dev, generator=g) * 3).to(torch.bfloat16)
    p = torch.rand((rows, vocab), device=dev, generator=g) ** 8
    p = (p / p.sum(1, keepdim=True)).to(torch.bfloat16)
    mask = torch.ones(rows, dtype=torch.uint8, device=dev)
    stats = torch.empty(2, dtype=torch.float64, device=dev)
    lse = torch.empty(rows, dtype=torch.float32, device=dev)
    d = ttt.loss_desc_for(z)
    ws = torch.empty(ttt.ttt_loss_workspace_size(d), dtype=torch.uint8, device=dev)

    def one():
        ttt.ttt_loss_fwd_bwd_inplace(d, z, p, mask, stats, ws, lse=lse, stream=stream)

    for _ in range(max(args.warmup, 3)):
        one()
    torch.cuda.synchronize()
    n = max(args.steps, 10)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(n):
        one()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    ttt.ttt_attn_profile_begin()
    for _ in range(n):
        one()
    torch.cuda.synchronize()
    kern = ttt.ttt_attn_profile_end()
    k_ms, k_n = kern["ttt_loss_kernel"]
    avg = k_ms / k_n
    # algorithmic bytes per launch: read z, read p, write dL/dz over z (2 B each) + mask, lse, row loss
    alg_bytes = rows * vocab * 2 * 3 + rows * (1 + 4 + 4)
    achieved = alg_bytes / (avg / 1e3) / 1e9
    peak = peaks["hbm_gbs"]
    return {
        "workload": f"{rows} rows x {vocab} vocab, bf16, fused loss + in-place grad (TTT_LOSS_MEAN), one TTT step",
        "ms_per_call": ms, "rows_per_s": rows * world / (ms / 1e3), "unit": "rows/s",
        "launches_per_call": sum(c for _, c in kern.values()) // n,
        "roofline": {"kernel": "ttt_loss_kernel", "bound": "hbm", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "peak_kind": f"HBM ({peaks['source']})",
                     "avg_launch_ms": avg, "algorithmic_bytes_per_launch": alg_bytes,
                     "traffic": ncu_traffic("ttt_loss_ring_kernel") or ncu_traffic("ttt_loss_kernel")},
    }


def run_draft(args, stream, peaks, attn_unroll_ms=None):
    """SURVEY.md §8(f) NEXT #2, beside the headline: one training step (forward + backward, no optimizer
    update) of the EAGLE-3 draft layer unrolled over 7 TTT steps (draft.DraftTTT: fc 3d -> d, RMSNorms,
    the q/k/v projection with our RoPE / step-slot kernel, our TTT attention, o_proj, SwiGLU MLP 14336,
    LM head 32000 and our soft-label loss with the Alg. 3 in-place backward; projections on cuBLAS) at the
    Llama-3.1-8B draft shape B = 8, L = 2048 — how much of a draft-training step the attention is."""
    from paper_2603_18567_b200.draft import DraftTTT
    B, L, d, Hq, Hkv, D, V, I, S = 8, 2048, 4096, 32, 8, 128, 32000, 14336, 7
    dev = stream.device
    try:
        model = DraftTTT(d, Hq, Hkv, D, V, intermediate=I, device=dev, seed=3)
        g = torch.Generator(device=dev).manual_seed(21)
        lmh = (torch.randn(B, L, 3 * d, device=dev, generator=g) * 0.5).to(torch.bfloat16)
        targets = [torch.softmax(torch.randn(B * L, V, device=dev, generator=g), -1).to(torch.bfloat16)
                   for _ in range(S)]

        def one():
            for prm in model.parameters():
                prm.grad = None
            model(lmh, targets).backward()

        with torch.cuda.stream(stream):
            for _ in range(2):
                one()
            torch.cuda.synchronize()
            iters = 3
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(iters):
                one()
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / iters
        res = {"workload": f"EAGLE-3 draft layer (d={d}, {Hq}/{Hkv} heads x {D}, MLP {I}, vocab {V}), {S} TTT steps, "
                           f"B={B} x L={L}, forward + backward (no optimizer update)",
               "ms_per_step": ms, "tokens_per_s": B * L / (ms / 1e3)}
        if attn_unroll_ms:
            res["attention_unroll_ms"] = attn_unroll_ms
            res["attention_share"] = attn_unroll_ms / ms
            res["note"] = ("attention = the headline's 7-step unroll of the same shape (same calls); the rest is cuBLAS "
                           "projections / MLP / LM head, torch RMSNorms and our RoPE and loss kernels")
        del model, lmh, targets
        torch.cuda.empty_cache()
        return res
    except Exception as e:  # noqa: BLE001 - a side row; the headline stands without it
        return {"error": f"{type(e).__name__}: {str(e)[:300]}"}


def run_rope(args, stream, peaks):
    """SURVEY.md §8(f) NEXT #2 part, beside the headline: one TTT step's fused q/k/v projection
    output (B L = 16384 rows x (32 + 2 x 8) heads x 128, bf16) -> RoPE'd q and the step's K / V
    slots (ttt_qkv_rope_split), one HBM pass."""
    import paper_2603_18567_b200 as ttt
    B, L, Hq, Hkv, D = 8, 2048, 32, 8, 128
    dev = stream.device
    g = torch.Generator(device=dev).manual_seed(11)
    qkv = torch.randn(B, L, Hq + 2 * Hkv, D, device=dev, generator=g).to(torch.bfloat16)
    q = torch.empty(B, L, Hq, D, dtype=torch.bfloat16, device=dev)
    k = torch.empty(B, L, Hkv, D, dtype=torch.bfloat16, device=dev)
    v = torch.empty_like(k)
    d = ttt.rope_desc(B, L, Hq, Hkv, D, 500000.0)
    ws = torch.empty(ttt.ttt_rope_workspace_size(d), dtype=torch.uint8, device=dev)
    one = lambda: ttt.ttt_qkv_rope_split(d, qkv, q, k, v, ws, stream=stream)
    for _ in range(3):
        one()
    torch.cuda.synchronize()
    iters = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(iters):
        one()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    nbytes = 2 * 2 * qkv.numel()  # read qkv, write q / k / v
    return {"workload": f"{B} x {L} rows, {Hq}+2x{Hkv} heads x {D}, bf16, rotate-half RoPE (base 5e5) + K/V slots",
            "ms_per_call": ms,
            "roofline": {"bound": "hbm", "achieved": nbytes / (ms / 1e3) / 1e9, "peak": peaks["hbm_gbs"],
                         "unit": "GB/s", "frac": nbytes / (ms / 1e3) / 1e9 / peaks["hbm_gbs"],
                         "algorithmic_bytes_per_call": nbytes}}


def run_tree(args, stream, peaks):
    """SURVEY.md §8(f) NEXT #4, beside the headline: tree-attention verification (ttt_tree_attn_fwd)
    with the Llama-3.1-8B target's attention heads (32 q / 8 kv, D = 128): 8 sequences, 4096
    context tokens each, a 64-node draft tree per sequence (the inference-side use of EAGLE-3)."""
    import paper_2603_18567_b200 as ttt
    B, n, P, Hq, Hkv, D = 8, 64, 4096, 32, 8, 128
    dev = stream.device
    g = torch.Generator(device=dev).manual_seed(5)
    mk = lambda *shp: torch.randn(shp, device=dev, generator=g).to(torch.bfloat16)
    q, k, v = mk(B, n, Hq, D), mk(B, P + n, Hkv, D), mk(B, P + n, Hkv, D)
    par = torch.randint(0, 1 << 20, (B, n), device=dev, generator=g)
    parents = torch.where(torch.arange(n, device=dev) > 0, par % torch.arange(n, device=dev).clamp(min=1), -1)
    parents = parents.to(torch.int32).contiguous()
    out = torch.empty_like(q)
    lse = torch.empty(B, Hq, n, device=dev)
    d = ttt.tree_desc(B, n, P + n, Hq, Hkv, D, [P] * B)
    ws = torch.empty(ttt.ttt_tree_attn_workspace_size(d), dtype=torch.uint8, device=dev)
    one = lambda: ttt.ttt_tree_attn_fwd(d, q, k, v, parents, out, lse, ws, stream=stream)
    for _ in range(3):
        one()
    torch.cuda.synchronize()
    iters = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(iters):
        one()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    kv_bytes = 2 * B * (P + n) * Hkv * D * 2
    return {"workload": f"{B} seqs x {P} context + {n}-node draft tree, 32/8 heads, D=128, bf16 (target verify)",
            "ms_per_call": ms, "tree_tokens_per_s": B * n / (ms / 1e3),
            "roofline": {"bound": "hbm", "achieved": (kv_bytes + 2 * 2 * B * n * Hq * D) / (ms / 1e3) / 1e9,
                         "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "note": ("K/V cache read once; latency-bound: 8 seqs x 8 kv heads x 2 context splits = "
                                  "128 CTAs (4 heads x 64 tree rows each) walk ~17 kv tiles through the forward "
                                  "pipeline, then a combine pass merges the splits")}}


def run_config(name: str, stream, peaks, workload: str):
    """A BASELINE.json configuration beside the headline: one 7-step unroll (fwd + bwd) on one GPU."""
    shape = CONFIGS[name]
    u = Unroll(shape, seed=99, dev=stream.device)
    for _ in range(2):
        u.step(stream)
    torch.cuda.synchronize()
    n = 3
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(n):
        u.step(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    per_step_pairs, _ = alg_pairs(shape)
    tflops = 12 * shape.head_dim * sum(per_step_pairs) / (ms / 1e3) / 1e12
    del u
    torch.cuda.empty_cache()
    return {"workload": workload, "ms_per_step": ms, "tokens_per_s": shape.batch * shape.seq_len / (ms / 1e3),
            "steps": n, "tflops": tflops, "frac_of_bf16_peak": tflops / peaks["bf16_tflops_sustained"]}


def run_packed(args, stream, peaks):
    """the Llama-3.1-8B draft unroll over a PACKED batch (8 sequences with the
    paper's padded-conversation length mix T_b ~ U[L/4, L], L = 2048, back to back, cu_seqlens) beside
    the same sequences in the padded layout (B x L with seq_lens). Throughput counts valid tokens;
    the FLOP count is the allowed pairs of the valid rows only (a padded row r >= T_b is work the
    packed layout does not have)."""
    from paper_2603_18567_b200.inputs import packed_lens
    shape = CONFIGS["llama8b"]
    lens = [int(x) for x in packed_lens(shape.batch, shape.seq_len, seed=0)]
    valid = sum(lens)
    pairs = sum(shape.num_q_heads * sum(T * (T + 1) // 2 + j * T for T in lens) for j in range(shape.ttt_steps))
    res = {"workload": (f"Llama-3.1-8B draft heads, {shape.batch} sequences T_b ~ U[{shape.seq_len // 4}, "
                        f"{shape.seq_len}] ({valid} valid tokens), ttt_steps=7, fwd + bwd unroll"),
           "seq_lens": lens}
    for mode in ("packed", "padded"):
        u = Unroll(shape, seed=98, dev=stream.device, seq_lens=lens, packed=(mode == "packed"))
        for _ in range(2):
            u.step(stream)
        torch.cuda.synchronize()
        n = 3
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(n):
            u.step(stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        tflops = 12 * shape.head_dim * pairs / (ms / 1e3) / 1e12
        res[mode] = {"ms_per_step": ms, "valid_tokens_per_s": valid / (ms / 1e3), "tflops_valid": tflops,
                     "frac_of_bf16_peak": tflops / peaks["bf16_tflops_sustained"],
                     "input_bytes": sum(t.nbytes for t in u.inputs)}
        del u
        torch.cuda.empty_cache()
    return res


def run_longctx(args, stream, peaks):
    """BASELINE.json configs[3]: 1 x L = 16384, Llama-3.1-8B draft heads. Across GPUs this shape
    splits by kv-head block (dp.seq_to_head), each rank running this same
    kernel sequence on Hq/N, Hkv/N heads."""
    return run_config("longctx", stream, peaks,
                      "long-context: 1 x L=16384, 32/8 heads, D=128, ttt_steps=7, bf16, fwd+bwd unroll")


def run_head_parallel(args, shape: Shape, rank: int, world: int, local_rank: int):
    """--head-parallel: one long sequence split over N GPUs by kv-head
    block. Every rank starts from sequence shards [L/N, H, D] of q_j / dO_j / K / V (as
    sequence-parallel projections produce them), one NCCL all-to-all per tensor turns them into head
    shards [L, H/N, D] (dp.seq_to_head), the rank runs the whole unroll on Hq/N, Hkv/N heads with no
    communication inside the attention, and out_j, dq_j, dK, dV go back to sequence shards
    (dp.head_to_seq). Strong scaling: the total work is fixed. (The exchange is gloo-tested and the
    head-block result is checked equal to the full problem on one GPU, tests/test_gpu_head_parallel.py.)"""
    import torch.distributed as dist

    from paper_2603_18567_b200.dp import head_to_seq, max_over_ranks, seq_to_head
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    B, L, Hq, Hkv, D, S = shape.batch, shape.seq_len, shape.num_q_heads, shape.num_kv_heads, shape.head_dim, shape.ttt_steps
    if B != 1 or Hkv % world or L % world:
        raise SystemExit("--head-parallel needs batch 1 and Hkv, L divisible by the GPU count")
    local = Shape(1, L, Hq // world, Hkv // world, D, S)
    u = Unroll(local, seed=1234 + rank, dev=dev)
    stream = torch.cuda.current_stream(dev)
    g = torch.Generator(device=dev).manual_seed(77 + rank)
    shard = lambda H: torch.randn((L // world, H, D), device=dev, generator=g).to(torch.bfloat16)
    q_sh, do_sh = [shard(Hq) for _ in range(S)], [shard(Hq) for _ in range(S)]
    kv_sh = [shard(Hkv) for _ in range(2 * S)]  # K_0, V_0, K_1.., V_1..

    def one_step():
        for j in range(S):
            u.q[j].view(L, Hq // world, D).copy_(seq_to_head(q_sh[j], world))
            u.do[j].view(L, Hq // world, D).copy_(seq_to_head(do_sh[j], world))
        kv = [u.k, u.v] + u.ks + u.vs
        for t, sh in zip(kv, kv_sh):
            t.view(L, Hkv // world, D).copy_(seq_to_head(sh, world))
        u.step(stream)
        outs = [head_to_seq(x.view(L, Hq // world, D), world) for x in u.out + u.dq]
        grads = [head_to_seq(x.view(L, Hkv // world, D), world) for x in [u.dk, u.dv] + u.dks + u.dvs]
        return outs, grads

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            one_step()
        e1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
    ms = max_over_ranks(e0.elapsed_time(e1), device=dev) / args.steps
    per_step_pairs, _ = alg_pairs(shape)
    tflops = 12 * D * sum(per_step_pairs) / (ms / 1e3) / 1e12
    peaks = load_peaks()
    line = {
        "metric": METRIC, "value": L / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (torch Philox N(0,1) -> bf16)",
        "config": {"workload": f"long-context head-parallel: 1 x L={L}, {Hq}/{Hkv} heads split over {world} GPUs, "
                               f"ttt_steps={S}, incl. the seq<->head all-to-alls", "global_batch": 1,
                   "seq_len": L, "parallelism": f"head-parallel{world}"},
        "tflops_per_gpu": tflops / world, "frac_of_bf16_peak": tflops / world / peaks["bf16_tflops_sustained"],
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_e2e(sets, opt, stream, args, shape: Shape, gb: int, dev):
    """Same metric through the public API with host buffers. Every micro-batch's inputs (q_j, dO_j,
    K_0, V_0, K_i, V_i) are copied H2D from pinned memory and EVERY result of its unroll (out_j,
    lse_j, dq_j, dK_0, dV_0, dK_i, dV_i) is read back D2H into pinned memory, copies inside the timed
    region. Buffers are double-buffered like a data loader's prefetch: micro-batch i+1's H2D runs on
    a copy stream while micro-batch i computes, and micro-batch i's D2H on a second copy stream while
    micro-batch i+1 computes (a buffer set is refilled only after its results were read back)."""
    import paper_2603_18567_b200  # noqa: F401
    if len(sets) == 1:
        sets = [sets[0], Unroll(shape, seed=4321, dev=dev, bwd_unroll=sets[0].bwd_unroll)]
    u = sets[0]
    host_in = [t.cpu().pin_memory() for t in u.inputs]
    host_out = [[torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in u.outputs] for _ in range(2)]
    h2d = sum(t.numel() * t.element_size() for t in host_in)
    d2h = sum(t.numel() * t.element_size() for t in host_out[0])
    per_step = len(opt.micro)
    n = max(3, min(args.steps, 6))
    cin, cout = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    ev = lambda: torch.cuda.Event()
    h2d_done, comp_done, d2h_done = [ev(), ev()], [ev(), ev()], [ev(), ev()]
    state = {"i": 0, "total": 0}

    def copy_in(k):
        with torch.cuda.stream(cin):
            cin.wait_event(comp_done[k])
            for d, h in zip(sets[k].inputs, host_in):
                d.copy_(h, non_blocking=True)
            h2d_done[k].record(cin)

    def micro(m, lo, hi):
        i = state["i"]
        k = i % 2
        if i + 1 < state["total"]:
            copy_in(1 - k)
        stream.wait_event(h2d_done[k])
        stream.wait_event(d2h_done[k])
        sets[k].step(stream)
        comp_done[k].record(stream)
        with torch.cuda.stream(cout):
            cout.wait_event(comp_done[k])
            for h, d in zip(host_out[k], sets[k].outputs):
                h.copy_(d, non_blocking=True)
            d2h_done[k].record(cout)
        state["i"] = i + 1

    def run(steps):
        state["i"], state["total"] = 0, steps * per_step
        for k in range(2):
            comp_done[k].record(stream)
            d2h_done[k].record(stream)
        copy_in(0)
        for _ in range(steps):
            opt.run(micro)

    run(2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    run(n)
    stream.wait_stream(cin)
    stream.wait_stream(cout)
    e1.record(stream)
    torch.cuda.synchronize()
    from paper_2603_18567_b200.dp import max_over_ranks
    ms = max_over_ranks(e0.elapsed_time(e1), device=dev) / n
    return {"value": gb * shape.seq_len / (ms / 1e3), "unit": UNIT, "ms_per_step": ms,
            "h2d_bytes_per_step": h2d * per_step, "d2h_bytes_per_step": d2h * per_step, "steps": n,
            "overlap": "double-buffered micro-batches: H2D of the next and D2H of the previous on two copy "
                       "streams under the current one's compute; D2H = every output of each unroll"}


def ncu_traffic(kernel: str):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")  # copy of the latest profiles/ncu_summary_rNN.json
    if not os.path.exists(p):
        return None
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(kernel, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="workload (default: llama8b = BASELINE configs[1] at N = 1, dp = configs[4] at N > 1)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-loss", action="store_true", help="skip the §8(f) loss-kernel measurement")
    ap.add_argument("--head-parallel", action="store_true",
                    help="split one long sequence (e.g. --config longctx) over the GPUs by kv-head block "
                         "(NCCL all-to-alls around the attention; strong scaling)")
    ap.add_argument("--zero2", action="store_true",
                    help="ZeRO-2 draft gradient exchange (reduce-scatter per backward call + parameter all-gather "
                         "after the step, PAPER.md:281) instead of the bucketed all-reduce")
    ap.add_argument("--bwd-unroll", action="store_true",
                    help="one ttt_attn_bwd_unroll call per unroll instead of S ttt_attn_bwd calls. Needs every "
                         "step's dO up front, which chained TTT training does not have (step j's output feeds "
                         "step j+1, so dO_j exists only after step j+1's backward): a what-if, not the headline")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # contract: W >= 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.config is None:
        args.config = "llama8b" if world == 1 or args.head_parallel else "dp"
    shape = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, shape, rank, world)
        return
    if world > 1 or args.head_parallel:
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if world == 1:  # single-rank head-parallel run (plumbing check): a 1-process NCCL group
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29511")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank), rank=rank, world_size=world)
    try:
        if args.head_parallel:
            run_head_parallel(args, shape, rank, world, local_rank)
        else:
            run_ours(args, shape, rank, world, local_rank)
    finally:
        if world > 1 or args.head_parallel:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
