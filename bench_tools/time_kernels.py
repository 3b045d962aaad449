"""Per-step, per-kernel timing of one unroll (dev tool, not the bench contract).
usage: python bench_tools/time_kernels.py [config] [bwd]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_18567_b200 as ttt
from paper_2603_18567_b200.inputs import CONFIGS

cfg = sys.argv[1] if len(sys.argv) > 1 else "llama8b"
do_bwd = "bwd" in sys.argv
s = CONFIGS[cfg]
B, L, Hq, Hkv, D, S = s.batch, s.seq_len, s.num_q_heads, s.num_kv_heads, s.head_dim, s.ttt_steps
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
mk = lambda shp: torch.randn(shp, device=dev, generator=g, dtype=torch.float32).to(torch.bfloat16)
q = mk(s.q_shape); k = mk(s.kv_shape); v = mk(s.kv_shape)
ks = [mk(s.kv_shape) for _ in range(S - 1)]; vs = [mk(s.kv_shape) for _ in range(S - 1)]
out = torch.empty_like(q); olo = torch.empty_like(q); lse = torch.empty(B, Hq, L, device=dev)
desc = ttt.make_desc(B, L, Hq, Hkv, D)
do = mk(s.q_shape); dq = torch.empty_like(q)
z = lambda: torch.zeros(s.kv_shape, device=dev)
dk, dv = z(), z(); dks = [z() for _ in range(S - 1)]; dvs = [z() for _ in range(S - 1)]
ws = torch.empty(ttt.ttt_attn_workspace_size(desc, S - 1, True), dtype=torch.uint8, device=dev)
tot_f = tot_b = 0.0
ksum = {}
fwd = lambda j: ttt.ttt_attn_fwd(desc, j, q, k, v, ks, vs, out, lse, out_lo=olo)
bwd = lambda j: ttt.ttt_attn_bwd(desc, j, q, k, v, ks, vs, out, lse, do, dq, dk, dv, dks, dvs, flags=1, workspace=ws, out_lo=olo)


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record(); torch.cuda.synchronize()
    ttt.ttt_attn_profile_begin()
    fn()
    torch.cuda.synchronize()
    kern = ttt.ttt_attn_profile_end()
    return e0.elapsed_time(e1) / n, kern


for j in range(S):
    pairs = B * Hq * (L * (L + 1) / 2 + j * L)
    base = B * Hq * L * (L + 1) / 2
    ms, kern = timeit(lambda: fwd(j))
    tot_f += ms
    for n_, v_ in kern.items(): ksum[n_] = ksum.get(n_, 0.0) + v_[0]
    km = " ".join(f"{n.replace('ttt_','').replace('_kernel','')}={v[0]:.3f}" for n, v in kern.items())
    msg = f"{cfg} j={j} fwd {ms:.3f} ms {4*D*pairs/ms/1e9:.1f} TFLOP/s [{km}]"
    if do_bwd:
        msb, kern = timeit(lambda: bwd(j))
        tot_b += msb
        for n_, v_ in kern.items(): ksum[n_] = ksum.get(n_, 0.0) + v_[0]
        mm = kern.get("ttt_bwd_sm100_kernel", (0, 1))[0]
        km = " ".join(f"{n.replace('ttt_','').replace('_kernel','')}={v[0]:.3f}" for n, v in kern.items())
        msg += f" | bwd {msb:.3f} ms {8*D*pairs/msb/1e9:.1f} TFLOP/s [{km}] main {8*D*base/mm/1e9:.0f} TF/s"
    print(msg, flush=True)
P = B * Hq * (S * L * (L + 1) / 2 + L * S * (S - 1) / 2)
print(f"unroll fwd {tot_f:.3f} ms ({4*D*P/tot_f/1e9:.1f} TFLOP/s)" + (f" bwd {tot_b:.3f} ms ({8*D*P/tot_b/1e9:.1f}) total {12*D*P/(tot_f+tot_b)/1e9:.1f} TFLOP/s" if do_bwd else ""))
print("kernels ms/unroll: " + " ".join(f"{n.replace('ttt_','').replace('_kernel','')}={v:.3f}" for n, v in ksum.items()))
