"""Run fwd + bwd of one TTT step once (for ncu captures). usage: prof_one.py [config] [step]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_18567_b200 as ttt
from paper_2603_18567_b200.inputs import CONFIGS
cfg = sys.argv[1] if len(sys.argv) > 1 else "llama8b"
j = int(sys.argv[2]) if len(sys.argv) > 2 else 6
s = CONFIGS[cfg]
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
mk = lambda shp: torch.randn(shp, device=dev, generator=g, dtype=torch.float32).to(torch.bfloat16)
q = mk(s.q_shape); k = mk(s.kv_shape); v = mk(s.kv_shape)
ks = [mk(s.kv_shape) for _ in range(s.ttt_steps - 1)]; vs = [mk(s.kv_shape) for _ in range(s.ttt_steps - 1)]
out = torch.empty_like(q); olo = torch.empty_like(q); lse = torch.empty(s.batch, s.num_q_heads, s.seq_len, device=dev)
desc = ttt.make_desc(s.batch, s.seq_len, s.num_q_heads, s.num_kv_heads, s.head_dim)
do = mk(s.q_shape); dq = torch.empty_like(q)
z = lambda: torch.zeros(s.kv_shape, device=dev)
dk, dv = z(), z(); dks = [z() for _ in range(s.ttt_steps - 1)]; dvs = [z() for _ in range(s.ttt_steps - 1)]
ws = torch.empty(ttt.ttt_attn_workspace_size(desc, j, True), dtype=torch.uint8, device=dev)
for _ in range(2):
    ttt.ttt_attn_fwd(desc, j, q, k, v, ks, vs, out, lse, out_lo=olo)
    ttt.ttt_attn_bwd(desc, j, q, k, v, ks, vs, out, lse, do, dq, dk, dv, dks, dvs, flags=0, workspace=ws, out_lo=olo)
torch.cuda.synchronize()
print("done")
