"""Time the fused loss + in-place grad at the bench shape with CUDA events (dev A/B tool):
TTT_ATTN_LIB=build/libtttattn_x.so python bench_tools/time_loss.py [rows vocab]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_18567_b200 as ttt  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
vocab = int(sys.argv[2]) if len(sys.argv) > 2 else 32000
z = (torch.randn((rows, vocab), device="cuda") * 3).to(torch.bfloat16)
p = torch.rand((rows, vocab), device="cuda") ** 8
p = (p / p.sum(1, keepdim=True)).to(torch.bfloat16)
mask = torch.ones(rows, dtype=torch.uint8, device="cuda")
stats = torch.empty(2, dtype=torch.float64, device="cuda")
d = ttt.loss_desc_for(z)
ws = torch.empty(ttt.ttt_loss_workspace_size(d), dtype=torch.uint8, device="cuda")
for _ in range(5):
    ttt.ttt_loss_fwd_bwd_inplace(d, z, p, mask, stats, ws)
torch.cuda.synchronize()
ttt.ttt_attn_profile_begin()
for _ in range(20):
    ttt.ttt_loss_fwd_bwd_inplace(d, z, p, mask, stats, ws)
torch.cuda.synchronize()
k = ttt.ttt_attn_profile_end()
ms, n = k["ttt_loss_kernel"]
gb = rows * vocab * 6 / 1e9
print(f"{os.environ.get('TTT_ATTN_LIB', 'default')}: loss kernel {ms / n * 1e3:.1f} us  {gb / (ms / n / 1e3):.0f} GB/s")
