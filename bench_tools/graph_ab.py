"""dev: one unroll eager vs captured into a CUDA graph and replayed (same buffers)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import Unroll  # noqa: E402
from paper_2603_18567_b200.inputs import CONFIGS  # noqa: E402

u = Unroll(CONFIGS["llama8b"], seed=0, dev=torch.device("cuda"))
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        u.step(s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    u.step(torch.cuda.current_stream())
torch.cuda.synchronize()


def timeit(fn, n=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(n):
            fn()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for r in range(3):
    print("eager", round(timeit(lambda: u.step(s)), 3), "graph", round(timeit(g.replay), 3), flush=True)
# graph result == eager result
with torch.cuda.stream(s):
    u.step(s)
torch.cuda.synchronize()
ref = [t.clone() for t in (u.out[6], u.dq[0], u.dks[0])]
g.replay()
torch.cuda.synchronize()
print("graph out/dk_1 identical:", torch.equal(ref[0], u.out[6]), torch.equal(ref[2], u.dks[0]))
