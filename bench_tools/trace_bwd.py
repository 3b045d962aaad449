"""Timeline of one bwd CTA from a -DTTT_TRACE build (dev tool).
usage: TTT_ATTN_LIB=build/libtttattn_variant.so python bench_tools/trace_bwd.py [cta]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_18567_b200 as ttt
from paper_2603_18567_b200 import _lib
from paper_2603_18567_b200.inputs import CONFIGS
cta = int(sys.argv[1]) if len(sys.argv) > 1 else 0
lib = ctypes.CDLL(_lib.LIB_PATH)
buf = np.zeros((4, 1 << 16), dtype=np.uint64)
s = CONFIGS["llama8b"]; dev = "cuda"; j = 0
g = torch.Generator(device=dev).manual_seed(0)
mk = lambda shp: torch.randn(shp, device=dev, generator=g, dtype=torch.float32).to(torch.bfloat16)
q = mk(s.q_shape); k = mk(s.kv_shape); v = mk(s.kv_shape); do = mk(s.q_shape)
out = torch.empty_like(q); olo = torch.empty_like(q); lse = torch.empty(s.batch, s.num_q_heads, s.seq_len, device=dev)
desc = ttt.make_desc(s.batch, s.seq_len, s.num_q_heads, s.num_kv_heads, s.head_dim)
dq = torch.empty_like(q); z = lambda: torch.zeros(s.kv_shape, device=dev); dk, dv = z(), z()
ws = torch.empty(ttt.ttt_attn_workspace_size(desc, 0, True), dtype=torch.uint8, device=dev)
ttt.ttt_attn_fwd(desc, j, q, k, v, [], [], out, lse, out_lo=olo)
lib.ttt_debug_trace_read(ctypes.c_void_p(buf.ctypes.data), ctypes.c_uint(cta))
for _ in range(2):
    ttt.ttt_attn_bwd(desc, j, q, k, v, [], [], out, lse, do, dq, dk, dv, [], [], flags=0, workspace=ws, out_lo=olo)
lib.ttt_debug_trace_read(ctypes.c_void_p(buf.ctypes.data), ctypes.c_uint(cta))
names = {0: {1: "mma:got_p_a", 2: "mma:got_p_b", 3: "mma:got_ds_a", 4: "mma:got_ds_b", 5: "mma:got_dqempty", 6: "mma:dP_issued", 7: "mma:dK_a_issued", 8: "mma:dK_b_issued", 9: "mma:dQ_issued", 10: "mma:S_issued", 11: "mma:got_q", 12: "mma:got_do_a", 13: "mma:got_do_b"},
         1: {1: "cmpA:got_s", 2: "cmpA:p_done", 3: "cmpA:got_dp", 4: "cmpA:ds_done", 5: "cmpA:s_loaded", 6: "cmpA:p_math_done", 7: "cmpA:got_dsempty", 8: "cmpA:got_acc", 9: "cmpA:epi_done", 10: "cmpA:epi_staged", 11: "cmpA:epi_bar", 12: "cmpA:epi_ld0"},
         2: {1: "dq:got_dq", 2: "dq:drained", 11: "prod:q_issue", 12: "prod:do_a_issue", 13: "prod:do_b_issue", 14: "obs:q_arrived", 15: "obs:do_a_arrived", 16: "obs:do_b_arrived"}}
ev = []
for role in range(3):
    for x in buf[role]:
        x = int(x)
        if x == 0: continue
        ev.append((x >> 20, names[role].get((x >> 12) & 0xFF, str((x >> 12) & 0xFF)), x & 0xFFF))
ev.sort()
t0 = ev[0][0]
items = {}
for t, n, i in ev:
    items.setdefault(i, []).append((t - t0, n))
for i in sorted(items)[:3] + sorted(items)[20:24]:
    base = items[i][0][0]
    print(f"item {i}: " + "  ".join(f"{n}@{t-base}" for t, n in items[i]))
# per-item period
starts = sorted((v[0][0], i) for i, v in items.items() if any(n == "cmpA:got_s" for _, n in v))
ts = [t for t, n, i in ev if n == "cmpA:got_s"]
d = np.diff(ts)
print("items", len(ts), "period clk median", np.median(d), "mean", d.mean())
for nm in ["mma:got_p", "mma:got_ds", "mma:got_q", "mma:got_dqempty", "mma:got_do", "cmp:p_done", "cmp:got_dp", "cmp:ds_done", "dq:got_dq", "dq:drained"]:
    pass
# average offsets relative to cmp:got_s of the same item
acc = {}
for i, v in items.items():
    s0 = [t for t, n in v if n == "cmpA:got_s"]
    if not s0: continue
    for t, n in v:
        acc.setdefault(n, []).append(t - s0[0])
for n, xs in sorted(acc.items(), key=lambda kv: np.median(kv[1])):
    print(f"{n:18s} median offset {np.median(xs):8.0f}")
# per-warp phase completion spread (role 3)
w = {}
for x in buf[3]:
    x = int(x)
    if x == 0: continue
    ev_ = (x >> 12) & 0xFF; it = x & 0xFFF
    w.setdefault((it, ev_ >= 16), {})[ev_ % 16] = (x >> 20)
for phase, nm in ((False, "P"), (True, "dS")):
    rel = {k: [] for k in range(4, 12)}
    for (it, ph), d in w.items():
        if ph != phase or len(d) < 8 or it < 4: continue
        t0_ = min(d.values())
        for k, t in d.items(): rel[k].append(t - t0_)
    print(nm, "phase: median lag behind the first warp, by warp:", {k: int(np.median(v)) for k, v in rel.items() if v})

# per-warp arrive times relative to cmpA:got_s of the same tile
gs = {i: t for t, n, i in ev if n == "cmpA:got_s"}
for phase, nm in ((False, "P arrive"), (True, "dS arrive")):
    rel = {}
    for (it, ph), d in w.items():
        if ph != phase or it not in gs or it < 4: continue
        for k, t in d.items(): rel.setdefault(k, []).append(t - gs[it])
    print(nm, "median offset by warp:", {k: int(np.median(v)) for k, v in sorted(rel.items())})

# absolute timeline (all roles) over a window of steady-state items
if "timeline" in sys.argv:
    gs_sorted = sorted(gs.items())
    lo = gs[20] if 20 in gs else ev[0][0]
    hi = gs[23] if 23 in gs else ev[-1][0]
    for t, n, i in ev:
        if lo - 2000 <= t <= hi:
            print(f"{t - lo:7d}  {n:18s} item {i}")

if "epi" in sys.argv:
    for t, n, i in ev:
        if n.startswith("cmpA:epi") or n == "cmpA:got_acc": print(f"{t - ev[0][0]:8d} {n}")
    print("total clk", ev[-1][0] - ev[0][0])
