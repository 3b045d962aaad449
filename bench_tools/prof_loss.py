"""One fused loss + in-place grad launch at the bench shape, for ncu (dev tool):
ncu --set full -k regex:ttt_loss_kernel -c 1 python bench_tools/prof_loss.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_18567_b200 as ttt  # noqa: E402

rows, vocab = int(sys.argv[1]) if len(sys.argv) > 1 else 16384, int(sys.argv[2]) if len(sys.argv) > 2 else 32000
z = (torch.randn((rows, vocab), device="cuda") * 3).to(torch.bfloat16)
p = torch.rand((rows, vocab), device="cuda") ** 8
p = (p / p.sum(1, keepdim=True)).to(torch.bfloat16)
mask = torch.ones(rows, dtype=torch.uint8, device="cuda")
stats = torch.empty(2, dtype=torch.float64, device="cuda")
d = ttt.loss_desc_for(z)
ws = torch.empty(ttt.ttt_loss_workspace_size(d), dtype=torch.uint8, device="cuda")
for _ in range(3):
    ttt.ttt_loss_fwd_bwd_inplace(d, z, p, mask, stats, ws)
torch.cuda.synchronize()
print("stats", stats.tolist())
