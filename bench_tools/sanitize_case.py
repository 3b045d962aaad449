"""Tiny invocations of every kernel family for compute-sanitizer (bench_tools/sanitize.sh):
TTT fwd / bwd (bf16 tensor-core path, fp32 check path), the unroll backward, the loss with its
in-place Alg. 3 backward, tree verification and the RoPE split. Small shapes that still span
several tiles, a ragged tail and j > 0 diagonal keys."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_18567_b200 as ttt  # noqa: E402
from paper_2603_18567_b200.inputs import Shape, make_case, make_loss_case, make_tree_case  # noqa: E402


def attn(dtype):
    s = Shape(2, 256, 4, 2, 128, 3)
    c = make_case(s, dtype=dtype, seed=0, lens="ragged")
    d = lambda t: t.cuda().contiguous()
    q, do = [d(x) for x in c.q], [d(x) for x in c.dout]
    k, v = d(c.k_base), d(c.v_base)
    ks, vs = [d(x) for x in c.k_steps], [d(x) for x in c.v_steps]
    desc = ttt.desc_for(q[0], k, seq_lens=[int(x) for x in c.seq_lens])
    S = s.ttt_steps
    out = [torch.empty_like(x) for x in q]
    lo = [torch.empty_like(x) for x in q] if dtype == torch.bfloat16 else None
    lse = [torch.empty(s.batch, s.num_q_heads, s.seq_len, device="cuda") for _ in range(S)]
    for j in range(S):
        ttt.ttt_attn_fwd(desc, j, q[j], k, v, ks, vs, out[j], lse[j], out_lo=lo[j] if lo else None)
    f32 = lambda: torch.zeros(s.kv_shape, device="cuda")
    dq = [torch.empty_like(x) for x in q]
    dk, dv, dks, dvs = f32(), f32(), [f32() for _ in range(S - 1)], [f32() for _ in range(S - 1)]
    ws = torch.empty(max(ttt.ttt_attn_workspace_size(desc, S - 1, True), 16), dtype=torch.uint8, device="cuda")
    for j in reversed(range(S)):
        ttt.ttt_attn_bwd(desc, j, q[j], k, v, ks, vs, out[j], lse[j], do[j], dq[j], dk, dv, dks, dvs,
                         flags=0 if j == S - 1 else ttt.TTT_ACCUMULATE_DKV, workspace=ws,
                         out_lo=lo[j] if lo else None)
    if dtype == torch.bfloat16:
        wsu = torch.empty(ttt.ttt_attn_bwd_unroll_workspace_size(desc, S), dtype=torch.uint8, device="cuda")
        ttt.ttt_attn_bwd_unroll(desc, q, k, v, ks, vs, out, lse, do, dq, dk, dv, dks, dvs, workspace=wsu, out_lo=lo)
    torch.cuda.synchronize()


def loss():
    lc = make_loss_case(64, 1000, dtype=torch.bfloat16, seed=0)
    z, p, m = lc.z.cuda(), lc.p.cuda(), lc.mask.cuda()
    d = ttt.loss_desc_for(z)
    ws = torch.empty(ttt.ttt_loss_workspace_size(d), dtype=torch.uint8, device="cuda")
    st = torch.empty(2, dtype=torch.float64, device="cuda")
    ttt.ttt_loss_fwd(d, z, p, m, st, ws)
    ttt.ttt_loss_bwd_inplace(d, z, p, m, ws)
    z2 = lc.z.cuda()
    ttt.ttt_loss_fwd_bwd_inplace(d, z2, p, m, st, ws)
    torch.cuda.synchronize()


def tree():
    tc = make_tree_case(2, 16, [130, 200], 4, 2, 128, seed=0)
    q, k, v, par = tc.q.cuda(), tc.k.cuda(), tc.v.cuda(), tc.parents.cuda()
    d = ttt.tree_desc(2, 16, k.shape[1], 4, 2, 128, tc.prefix_lens)
    out = torch.empty_like(q)
    lse = torch.empty(2, 4, 16, device="cuda")
    ws = torch.empty(max(ttt.ttt_tree_attn_workspace_size(d), 16), dtype=torch.uint8, device="cuda")
    ttt.ttt_tree_attn_fwd(d, q, k, v, par, out, lse, ws)
    torch.cuda.synchronize()


def rope():
    B, L, Hq, Hkv, D = 2, 64, 4, 2, 128
    qkv = torch.randn(B, L, Hq + 2 * Hkv, D, device="cuda").to(torch.bfloat16)
    q = torch.empty(B, L, Hq, D, dtype=torch.bfloat16, device="cuda")
    k = torch.empty(B, L, Hkv, D, dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    d = ttt.rope_desc(B, L, Hq, Hkv, D)
    ws = torch.empty(ttt.ttt_rope_workspace_size(d), dtype=torch.uint8, device="cuda")
    ttt.ttt_qkv_rope_split(d, qkv, q, k, v, ws)
    dqkv = torch.empty_like(qkv)
    ttt.ttt_qkv_rope_join_bwd(d, q, k, v, dqkv, ws)
    torch.cuda.synchronize()


if __name__ == "__main__":
    which = sys.argv[1:] or ["attn_bf16", "attn_fp32", "loss", "tree", "rope"]
    for w in which:
        {"attn_bf16": lambda: attn(torch.bfloat16), "attn_fp32": lambda: attn(torch.float32), "loss": loss,
         "tree": tree, "rope": rope}[w]()
        print("ok", w, flush=True)
