"""One Llama-shape unroll (7 fwd + one ttt_attn_bwd_unroll or 7 ttt_attn_bwd), for ncu (dev tool).
python bench_tools/prof_unroll.py [percall]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import Unroll  # noqa: E402
from paper_2603_18567_b200.inputs import CONFIGS  # noqa: E402

u = Unroll(CONFIGS["llama8b"], seed=0, dev=torch.device("cuda"), bwd_unroll="percall" not in sys.argv)
s = torch.cuda.current_stream()
for _ in range(2):
    u.step(s)
torch.cuda.synchronize()
print("ok")
