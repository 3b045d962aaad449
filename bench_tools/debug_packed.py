"""dev: packed vs padded forward per (lens, j) — which rows differ."""
import torch
import paper_2603_18567_b200 as ttt
from paper_2603_18567_b200.inputs import make_packed_case


def run(lens, j, Hq=8, Hkv=2, D=128):
    c = make_packed_case(lens, Hq, Hkv, D, j + 1, seed=5)
    to = lambda t: t.cuda().contiguous()
    q, k, v = to(c.q[j]), to(c.k_base), to(c.v_base)
    ks, vs = [to(x) for x in c.k_steps], [to(x) for x in c.v_steps]
    d = ttt.packed_desc(c.cu, Hq, Hkv, D)
    out = torch.zeros_like(q); lse = torch.zeros((Hq, c.rows), device="cuda")
    ttt.ttt_attn_fwd(d, j, q, k, v, ks, vs, out, lse)
    B = len(lens); L = (max(lens) + 127) // 128 * 128
    def pad(x):
        y = torch.zeros((B, L) + tuple(x.shape[1:]), dtype=x.dtype, device="cuda")
        for b in range(B):
            y[b, :lens[b]] = x[c.cu[b]:c.cu[b + 1]]
        return y
    dd = ttt.desc_for(pad(q), pad(k), seq_lens=list(lens))
    od = torch.zeros_like(pad(q)); ld = torch.zeros((B, Hq, L), device="cuda")
    ttt.ttt_attn_fwd(dd, j, pad(q), pad(k), pad(v), [pad(x) for x in ks], [pad(x) for x in vs], od, ld)
    torch.cuda.synchronize()
    msgs = []
    for b in range(B):
        r0, T = int(c.cu[b]), lens[b]
        e = (out[r0:r0 + T].float() - od[b, :T].float()).abs().amax(dim=(1, 2))
        el = (lse[:, r0:r0 + T] - ld[b, :, :T]).abs().amax(dim=0)
        bad = torch.nonzero(e > 0).flatten().tolist()
        badl = torch.nonzero(el > 0).flatten().tolist()
        msgs.append(f"seq{b}(T={T},r0={r0}): out bad rows {len(bad)} {bad[:6]} lse bad {len(badl)} {badl[:6]}")
    print(f"lens={lens} j={j}:", "; ".join(msgs))


for lens in ([128, 128], [16, 128], [8, 128], [1, 128], [3, 130], [130, 3]):
    for j in (0, 1, 2):
        run(lens, j)
