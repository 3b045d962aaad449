"""dev: full-size unroll vs per-call differences (which tensors, how large, which rows)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from tests.test_gpu_bwd_unroll import _run_both
from tests.gpu_helpers import DeviceCase
from paper_2603_18567_b200.inputs import CONFIGS, Shape, make_case
cfg = sys.argv[1] if len(sys.argv) > 1 else "llama8b"
shape = CONFIGS[cfg] if cfg in CONFIGS else Shape(*[int(x) for x in cfg.split(",")])
case = make_case(shape, dtype=torch.bfloat16, seed=0, lens="full")
dc = DeviceCase(case)
S = shape.ttt_steps
dq_a, a, dq_b, b = _run_both(dc, S, False)
dq_a2, a2, _, _ = _run_both(dc, S, False)
for i in range(S - 1):
    for k in ("dk_steps", "dv_steps"):
        d = (a[k][i] - b[k][i]).abs()
        d2 = (a[k][i] - a2[k][i]).abs()
        nz = (d > 0).nonzero()
        print(k, i + 1, "unroll-vs-percall max", d.max().item(), "n", int((d > 0).sum()), "percall-vs-percall max", d2.max().item(),
              "rows", nz[:5, :3].tolist() if len(nz) else [], "ref mag", a[k][i].abs().max().item())
