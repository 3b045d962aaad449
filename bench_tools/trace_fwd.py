"""Timeline of one fwd CTA from a -DTTT_TRACE build (dev tool).
usage: TTT_ATTN_LIB=build/libtttattn_variant.so python bench_tools/trace_fwd.py [cta]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_18567_b200 as ttt
from paper_2603_18567_b200 import _lib
from paper_2603_18567_b200.inputs import CONFIGS
cta = int(sys.argv[1]) if len(sys.argv) > 1 else 0
lib = ctypes.CDLL(_lib.LIB_PATH)
buf = np.zeros((4, 1 << 16), dtype=np.uint64)
s = CONFIGS["llama8b"]; dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
mk = lambda shp: torch.randn(shp, device=dev, generator=g, dtype=torch.float32).to(torch.bfloat16)
q = mk(s.q_shape); k = mk(s.kv_shape); v = mk(s.kv_shape)
out = torch.empty_like(q); olo = torch.empty_like(q); lse = torch.empty(s.batch, s.num_q_heads, s.seq_len, device=dev)
desc = ttt.make_desc(s.batch, s.seq_len, s.num_q_heads, s.num_kv_heads, s.head_dim)
J = int(os.environ.get("TTT_TRACE_STEP", "0"))  # TTT step j of the traced forward (diagonal keys)
ks = [mk(s.kv_shape) for _ in range(J)]; vs = [mk(s.kv_shape) for _ in range(J)]
lib.ttt_debug_ftrace_read(ctypes.c_void_p(buf.ctypes.data), ctypes.c_uint(cta))
for _ in range(2):
    ttt.ttt_attn_fwd(desc, J, q, k, v, ks, vs, out, lse, out_lo=olo if 'nolo' not in sys.argv else None)
lib.ttt_debug_ftrace_read(ctypes.c_void_p(buf.ctypes.data), ctypes.c_uint(cta))
names = {0: {9: "mma:start", 8: "mma:got_q_k0", 1: "mma:got_v", 2: "mma:got_p0", 3: "mma:got_p1"},
         1: {9: "cta:start", 10: "cta:end", 1: "s0:got_s", 2: "s0:p_done", 3: "s0:loop_end", 4: "s0:got_o", 5: "s0:epi_done", 6: "s0:epi_math_done", 7: "s0:epi_bar", 8: "s0:tma_issued"},
         2: {1: "s1:got_s", 2: "s1:p_done"},
         3: {1: "dg:stage_full", 2: "dg:done", 3: "dgp:issued", 4: "dg:start"}}
ev = []
for role in range(4):
    for x in buf[role]:
        x = int(x)
        if x == 0: continue
        ev.append((x >> 20, names[role].get((x >> 12) & 0xFF, str((x >> 12) & 0xFF)), x & 0xFFF))
ev.sort()
t0 = ev[0][0]
for t, n, i in ev[:1000]:
    print(f"{t - t0:8d} {n:14s} {i}")
got = [t for t, n, i in ev if n == "s0:got_s"]
st = [t for t, n, i in ev if n == "cta:start"]
en = [t for t, n, i in ev if n == "cta:end"]
if got and st and en:
    d = np.diff(got)
    print(f"CTA {cta}: tiles {len(got)}  start->first S {got[0] - st[0]}  tile period median {np.median(d) if len(d) else 0:.0f}"
          f"  last S -> end {en[0] - got[-1]}  total {en[0] - st[0]}")
