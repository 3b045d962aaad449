"""CPU-side checks of the C-ABI boundary (no GPU compute): the shared library
loads, exports every function include/ttt_attn.h declares, and rejects bad
arguments with the documented status codes before touching the device."""
import ctypes
import os
import re

import pytest

import paper_2603_18567_b200 as ttt
from paper_2603_18567_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    names = []
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            src = open(os.path.join(ROOT, "include", fn)).read()
            names += re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(ttt_(?:attn|loss|tree|rope|qkv)_\w+)\s*\(", src, re.M)
    return sorted(set(names))


def test_header_symbols_exported():
    names = _declared_functions()
    assert {"ttt_attn_fwd", "ttt_attn_bwd", "ttt_attn_workspace_size", "ttt_attn_strerror",
            "ttt_loss_fwd", "ttt_loss_bwd_inplace", "ttt_loss_fwd_bwd_inplace", "ttt_loss_workspace_size"} <= set(names)
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n


def test_version_and_strerror():
    assert "sm_100a" in ttt.ttt_attn_version()
    for code in range(8):
        assert ttt.ttt_attn_strerror(code)


class FakeT:
    """Stand-in exposing data_ptr() only: validation fails before any CUDA call."""
    def __init__(self, ptr):
        self.p = ptr

    def data_ptr(self):
        return self.p


def _fwd(desc, step, align=16, null=False):
    P = lambda i: FakeT(0 if null and i == 0 else 0x10000000 + 4096 * i + (align % 16))
    ks = [P(10 + i) for i in range(max(step, 0))]
    vs = [P(50 + i) for i in range(max(step, 0))]
    ttt.ttt_attn_fwd(desc, step, P(0), P(1), P(2), ks, vs, P(3), P(4))


@pytest.mark.parametrize("kw,step,code", [
    (dict(head_dim=96), 0, 2),                 # unsupported head_dim
    (dict(seq_len=100), 0, 2),                 # bf16 needs L % 128 == 0
    (dict(num_kv_heads=3), 0, 1),              # Hq % Hkv != 0
    (dict(), -1, 3), (dict(), 32, 3),          # step range
    (dict(seq_lens=[0, 128]), 0, 5),           # degenerate T_b
    (dict(seq_lens=[129, 128]), 0, 5),
    (dict(batch=0), 0, 1),
])
def test_validation_codes(kw, step, code):
    base = dict(batch=2, seq_len=128, num_q_heads=4, num_kv_heads=2, head_dim=64)
    base.update(kw)
    d = ttt.make_desc(**base)
    with pytest.raises(ttt.TTTError) as ei:
        _fwd(d, step)
    assert ei.value.code == code


def test_alignment_and_null():
    d = ttt.make_desc(1, 128, 2, 1, 64)
    with pytest.raises(ttt.TTTError) as ei:
        _fwd(d, 1, align=8)
    assert ei.value.code == 4
    with pytest.raises(ttt.TTTError) as ei:
        _fwd(d, 1, null=True)
    assert ei.value.code == 1


@pytest.mark.parametrize("cu,seq_lens,code", [
    ([0, 3, 3, 9], None, 5),                   # empty sequence
    ([1, 3, 9], None, 1),                      # cu_seqlens[0] != 0
    ([0, 5, 9], [5, 4], 1),                    # seq_lens and cu_seqlens both given
    ([0, 40000000, 80000000], None, 2),        # N x Hq >= 2^31
])
def test_packed_validation_codes(cu, seq_lens, code):
    d = ttt.make_desc(len(cu) - 1, 128, 32, 8, 128, seq_lens=seq_lens, cu_seqlens=cu)
    with pytest.raises(ttt.TTTError) as ei:
        _fwd(d, 0)
    assert ei.value.code == code


def test_packed_desc_and_workspace():
    cu = [0, 5, 133, 300, 301]
    d = ttt.packed_desc(cu, 4, 2, 64)
    assert d.packed_rows == 301 and d.batch == 4 and d.seq_len == 167
    tiles = 1 + 1 + 2 + 1  # T_b = 5, 128, 167, 1
    assert ttt.ttt_attn_workspace_size(d, 2, True) >= 2 * 4 * tiles * 128 * 4 + 4 * tiles * 128 * 64 * 4
    assert ttt.ttt_attn_workspace_size(d, 2, False) == 0
    fp = ttt.packed_desc(cu, 4, 2, 64, dtype=ttt.TTT_FP32_CHECK)
    assert ttt.ttt_attn_workspace_size(fp, 2, True) == (2 + 2 * 2) * 301 * 2 * 64 * 8
    with pytest.raises(ttt.TTTError):
        ttt.make_desc(2, 128, 4, 2, 64, cu_seqlens=[0, 5])  # batch + 1 entries needed


def test_workspace_size():
    d = ttt.make_desc(8, 2048, 32, 8, 128)
    ws = ttt.ttt_attn_workspace_size(d, 6, True)
    rows = 8 * 32 * 2048
    assert ws >= rows * 4 * 2 + rows * 128 * 4
    assert ttt.ttt_attn_workspace_size(d, 6, False) == 0
    assert ttt.ttt_attn_workspace_size(ttt.make_desc(8, 2048, 32, 8, 96), 0, True) == 0


def _loss_desc(rows=16, vocab=32000, dtype=ttt.TTT_BF16):
    d = ttt.LossDesc()
    d.rows, d.vocab, d.dtype = rows, vocab, dtype
    return d


@pytest.mark.parametrize("kw,call,code", [
    (dict(rows=0), "fwd", 1), (dict(vocab=1), "fwd", 1), (dict(dtype=7), "fwd", 1),
    (dict(vocab=262152), "fwd", 2),            # beyond the register-resident row capacity
    (dict(vocab=131076, dtype=1), "bwd", 2),
    (dict(vocab=32769), "bwd", 2),             # odd vocab (element path) capacity 32768
    (dict(), "ws_small", 6), (dict(), "ws_misaligned", 4), (dict(), "flags", 1),
    (dict(), "no_stats", 1), (dict(vocab=33), "z_odd", 4),
])
def test_loss_validation_codes(kw, call, code):
    d = _loss_desc(**kw)
    ws_n = ttt.ttt_loss_workspace_size(d) if call not in ("fwd",) or code != 1 else 0
    ws_n = max(ws_n, 4096)
    z, p, st, m = FakeT(0x10000000), FakeT(0x20000000), FakeT(0x30000000), FakeT(0x40000000)
    ws = FakeT(0x50000000)

    class WS(FakeT):
        def __init__(self, ptr, n):
            super().__init__(ptr)
            self.n = n

        def numel(self):
            return self.n

        def element_size(self):
            return 1
    wsb = WS(0x50000000, ws_n)
    with pytest.raises(ttt.TTTError) as e:
        if call == "fwd":
            ttt.ttt_loss_fwd(d, z, p, m, st, wsb)
        elif call == "bwd":
            ttt.ttt_loss_bwd_inplace(d, z, p, m, wsb)
        elif call == "ws_small":
            ttt.ttt_loss_fwd(d, z, p, m, st, WS(0x50000000, 64))
        elif call == "ws_misaligned":
            ttt.ttt_loss_fwd(d, z, p, m, st, WS(0x50000008, ws_n + 64))
        elif call == "flags":
            ttt.ttt_loss_bwd_inplace(d, z, p, m, wsb, flags=6)
        elif call == "no_stats":
            ttt.ttt_loss_fwd(d, z, p, m, None, wsb)
        elif call == "z_odd":
            ttt.ttt_loss_bwd_inplace(d, FakeT(0x10000001), p, m, wsb)
    assert e.value.code == code
    del ws


def test_loss_workspace_size():
    assert ttt.ttt_loss_workspace_size(_loss_desc(rows=1000)) >= 1000 * 4
    assert ttt.ttt_loss_workspace_size(_loss_desc(rows=0)) == 0


@pytest.mark.parametrize("S,ws,code", [(0, 1 << 30, 3), (9, 1 << 30, 3), (3, 64, 6)])
def test_bwd_unroll_validation_codes(S, ws, code):
    d = ttt.make_desc(1, 256, 4, 2, 128)
    n = max(S, 1)
    P = lambda i: FakeT(0x10000000 + 4096 * i)

    class WS(FakeT):
        def numel(self):
            return ws

        def element_size(self):
            return 1
    with pytest.raises(ttt.TTTError) as e:
        ttt.ttt_attn_bwd_unroll(d, [P(i) for i in range(n)][:S] if S else [], P(20), P(21),
                                [P(30 + i) for i in range(8)], [P(40 + i) for i in range(8)],
                                [P(50 + i) for i in range(n)], [P(60 + i) for i in range(n)],
                                [P(70 + i) for i in range(n)], [P(80 + i) for i in range(n)], P(90), P(91),
                                [P(100 + i) for i in range(8)], [P(110 + i) for i in range(8)],
                                workspace=WS(0x50000000))
    assert e.value.code == code


def test_bwd_unroll_workspace_size():
    d = ttt.make_desc(8, 2048, 32, 8, 128)
    assert ttt.ttt_attn_bwd_unroll_workspace_size(d, 7) == 7 * ttt.ttt_attn_workspace_size(d, 6, True)
    assert ttt.ttt_attn_bwd_unroll_workspace_size(d, 9) == 0


@pytest.mark.parametrize("kw,code", [(dict(num_tree=65), 2), (dict(num_tree=0), 1), (dict(head_dim=96), 2),
                                     (dict(prefix=[100, 4097]), 5), (dict(prefix=[-1, 0]), 5),
                                     (dict(ws=8), 6)])
def test_tree_validation_codes(kw, code):
    n = kw.get("num_tree", 8)
    d = ttt.tree_desc(2, n, 4104, 4, 2, kw.get("head_dim", 128), kw.get("prefix", [100, 200]))
    P = lambda i: FakeT(0x10000000 + 4096 * i)

    class WS(FakeT):
        def numel(self):
            return kw.get("ws", 4096)

        def element_size(self):
            return 1
    with pytest.raises(ttt.TTTError) as e:
        ttt.ttt_tree_attn_fwd(d, P(0), P(1), P(2), P(3), P(4), P(5), WS(0x50000000))
    assert e.value.code == code


def test_rope_validation_codes():
    d = ttt.rope_desc(1, 8, 4, 2, 40)
    P = lambda i: FakeT(0x10000000 + 4096 * i)
    with pytest.raises(ttt.TTTError) as e:
        ttt.ttt_qkv_rope_split(d, P(0), P(1), P(2), P(3), None)
    assert e.value.code == 2  # head_dim % 16
    d = ttt.rope_desc(1, 8, 4, 2, 64)
    with pytest.raises(ttt.TTTError) as e:
        ttt.ttt_qkv_rope_split(d, FakeT(0x10000008), P(1), P(2), P(3), None)
    assert e.value.code == 4
    assert ttt.ttt_rope_workspace_size(d) == 8 * 32 * 8 and ttt.ttt_rope_workspace_size(d, True) == 8 * 32 * 8
