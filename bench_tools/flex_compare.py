"""On-box context comparators for one TTT step (SURVEY.md §8(d) "optional on-box context comparators";
dev tool under bench_tools/, never part of the library or of bench.py's timed step).

The paper's kernel comparison (TTT length 7, the final step, vs "a native SDPA-based
implementation") reproduced on this B200 for the Llama-3.1-8B draft shape at j = 6:
  ours   ttt_attn_fwd + ttt_attn_bwd (this library, one call each, the bench's per-step form)
  flex   torch flex_attention (torch.compile) with the Alg. 2 mask_mod over [K_0; K_1..K_j] — the
         paper's own kernel design (FlexAttention compiled to Triton)
  sdpa   torch scaled_dot_product_attention with the materialised boolean L x (j+1)L mask — the
         paper's "native SDPA" baseline
fwd + bwd per call, CUDA events, median of reps. usage: python bench_tools/flex_compare.py [j] [reps] [L]
(L overrides the sequence length at the same tokens per call; the paper's figure is at L = 4096)
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2603_18567_b200 as ttt
from paper_2603_18567_b200.inputs import CONFIGS


def timeit(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    j = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    s = CONFIGS["llama8b"]
    B, L, Hq, Hkv, D = s.batch, s.seq_len, s.num_q_heads, s.num_kv_heads, s.head_dim
    if len(sys.argv) > 3:  # sequence length override (the paper's kernel figure is at L = 4096)
        L = int(sys.argv[3])
        B = max(1, B * s.seq_len // L)  # same tokens per call
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(0)
    mk = lambda *shp: torch.randn(shp, device=dev, generator=g, dtype=torch.float32).to(torch.bfloat16)
    q = mk(B, L, Hq, D)
    ks = [mk(B, L, Hkv, D) for _ in range(j + 1)]
    vs = [mk(B, L, Hkv, D) for _ in range(j + 1)]
    do = mk(B, L, Hq, D)
    res = {"workload": f"llama3.1-8b draft shape B={B} L={L} {Hq}/{Hkv} heads D={D}, TTT step j={j} "
                       "(final step of a 7-step unroll), fwd + bwd of one call", "reps": reps}

    # ---- ours (C-ABI through the binding) ----
    desc = ttt.make_desc(B, L, Hq, Hkv, D)
    out = torch.empty_like(q)
    olo = torch.empty_like(q)
    lse = torch.empty(B, Hq, L, device=dev)
    dq = torch.empty_like(q)
    z = lambda: torch.zeros(B, L, Hkv, D, device=dev)
    dk, dv = z(), z()
    dks, dvs = [z() for _ in range(j)], [z() for _ in range(j)]
    ws = torch.empty(ttt.ttt_attn_workspace_size(desc, j, True), dtype=torch.uint8, device=dev)

    def ours():
        ttt.ttt_attn_fwd(desc, j, q, ks[0], vs[0], ks[1:], vs[1:], out, lse, out_lo=olo)
        ttt.ttt_attn_bwd(desc, j, q, ks[0], vs[0], ks[1:], vs[1:], out, lse, do, dq, dk, dv, dks, dvs,
                         flags=0, workspace=ws, out_lo=olo)

    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    res["ours_ms"] = timeit(ours, reps)
    res["ours_extra_mem_gb"] = (torch.cuda.max_memory_allocated() - base) / 1e9  # beyond inputs + outputs + ws
    res["ours_workspace_gb"] = ws.numel() / 1e9  # caller-allocated workspace (delta, lse2, fp32 dq_acc)

    # ---- flex_attention with the Alg. 2 mask ----
    try:
        from torch.nn.attention.flex_attention import create_block_mask, flex_attention

        def mask_mod(b, h, qi, kv):
            causal = kv <= qi
            suffix = (kv >= L) & ((kv - qi) % L == 0)
            return causal | suffix

        bm = create_block_mask(mask_mod, None, None, L, (j + 1) * L, device=dev)
        qf = q.transpose(1, 2).contiguous().requires_grad_(True)
        kf = torch.cat(ks, 1).transpose(1, 2).contiguous().requires_grad_(True)
        vf = torch.cat(vs, 1).transpose(1, 2).contiguous().requires_grad_(True)
        dof = do.transpose(1, 2).contiguous()
        fa = torch.compile(flex_attention)

        def flex():
            o = fa(qf, kf, vf, block_mask=bm, enable_gqa=True)
            o.backward(dof)

        base = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        res["flex_ms"] = timeit(flex, reps)
        res["flex_extra_mem_gb"] = (torch.cuda.max_memory_allocated() - base) / 1e9
        # same results (spot check of the forward against ours)
        with torch.no_grad():
            o = fa(qf, kf, vf, block_mask=bm, enable_gqa=True).transpose(1, 2)
        res["flex_max_abs_diff_out"] = float((o.float() - out.float()).abs().max())
    except Exception as e:  # noqa: BLE001 - context only
        res["flex_error"] = f"{type(e).__name__}: {str(e)[:200]}"

    # ---- naive SDPA with the materialised mask (the paper's baseline) ----
    try:
        torch.cuda.empty_cache()
        qi = torch.arange(L, device=dev)[:, None]
        kv = torch.arange((j + 1) * L, device=dev)[None, :]
        mask = (kv <= qi) | ((kv >= L) & ((kv - qi) % L == 0))
        qs = q.transpose(1, 2).contiguous().requires_grad_(True)
        kr = torch.cat(ks, 1).transpose(1, 2).repeat_interleave(Hq // Hkv, 1).contiguous().requires_grad_(True)
        vr = torch.cat(vs, 1).transpose(1, 2).repeat_interleave(Hq // Hkv, 1).contiguous().requires_grad_(True)
        dos = do.transpose(1, 2).contiguous()

        def sdpa():
            o = torch.nn.functional.scaled_dot_product_attention(qs, kr, vr, attn_mask=mask)
            o.backward(dos)

        base = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        res["sdpa_ms"] = timeit(sdpa, max(3, reps // 2))
        res["sdpa_extra_mem_gb"] = (torch.cuda.max_memory_allocated() - base) / 1e9
    except Exception as e:  # noqa: BLE001
        res["sdpa_error"] = f"{type(e).__name__}: {str(e)[:200]}"

    for k in ("flex_ms", "sdpa_ms"):
        if k in res:
            res[f"speedup_vs_{k[:-3]}"] = res[k] / res["ours_ms"]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
