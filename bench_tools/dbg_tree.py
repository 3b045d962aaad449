import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2603_18567_b200 as ttt
from paper_2603_18567_b200.inputs import make_tree_case
from oracle import tree as OT
for (B, n, P, Hq, Hkv) in [(2, 64, [1000, 2047], 32, 8), (1, 64, [1000], 32, 8), (1, 64, [1000], 8, 2), (1, 20, [1000], 8, 2), (2, 64, [1000, 2047], 8, 8)]:
    c = make_tree_case(B, n, P, Hq, Hkv, 128, seed=3, kv_len=max(P) + n + 9)
    d = ttt.tree_desc(B, n, c.k.shape[1], Hq, Hkv, 128, P)
    out = torch.empty(B, n, Hq, 128, dtype=torch.bfloat16, device="cuda"); lse = torch.empty(B, Hq, n, device="cuda")
    ws = torch.zeros(ttt.ttt_tree_attn_workspace_size(d), dtype=torch.uint8, device="cuda")
    ttt.ttt_tree_attn_fwd(d, c.q.cuda(), c.k.cuda(), c.v.cuda(), c.parents.cuda(), out, lse, ws); torch.cuda.synchronize()
    o = out.float().cpu().numpy(); l = lse.cpu().numpy()
    f = lambda t: t.float().numpy()
    oo, ol = OT.tree_attention(f(c.q), f(c.k), f(c.v), P, c.parents.numpy())
    nan = np.argwhere(np.isnan(o).any(-1))
    print((B, n, P, Hq, Hkv), "nan rows", len(nan), nan[:6].tolist(), "max err", np.nanmax(np.abs(o - oo)), "lse err", np.nanmax(np.abs(l - ol)), "lse nan", int(np.isnan(l).sum()))
