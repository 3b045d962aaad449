"""One tree-verification call and one qkv RoPE split at the bench shapes, for ncu (dev tool):
ncu --set full -k regex:"ttt_fwd_sm100|ttt_qkv_rope_kernel" -c 2 python bench_tools/prof_next.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_18567_b200 as ttt  # noqa: E402

B, n, P, Hq, Hkv, D = 8, 64, 4096, 32, 8, 128
mk = lambda *s: torch.randn(s, device="cuda").to(torch.bfloat16)
q, k, v = mk(B, n, Hq, D), mk(B, P + n, Hkv, D), mk(B, P + n, Hkv, D)
par = torch.arange(-1, n - 1, device="cuda", dtype=torch.int32).repeat(B, 1).contiguous()
out, lse = torch.empty_like(q), torch.empty(B, Hq, n, device="cuda")
d = ttt.tree_desc(B, n, P + n, Hq, Hkv, D, [P] * B)
ws = torch.empty(ttt.ttt_tree_attn_workspace_size(d), dtype=torch.uint8, device="cuda")
ttt.ttt_tree_attn_fwd(d, q, k, v, par, out, lse, ws)
Lr = 2048
qkv = mk(B, Lr, Hq + 2 * Hkv, D)
rq, rk, rv = mk(B, Lr, Hq, D), mk(B, Lr, Hkv, D), mk(B, Lr, Hkv, D)
rd = ttt.rope_desc(B, Lr, Hq, Hkv, D)
rws = torch.empty(ttt.ttt_rope_workspace_size(rd), dtype=torch.uint8, device="cuda")
ttt.ttt_qkv_rope_split(rd, qkv, rq, rk, rv, rws)
torch.cuda.synchronize()
print("ok")
