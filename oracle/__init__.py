"""TEST INFRASTRUCTURE — the fp64 CPU oracle for TTT attention (NOT product code).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` leg may import this package. It shares no code with the
CUDA path (``paper_2603_18567_b200``) and never imports it.

Contents
  * ``liboracle.so`` (``ttt_oracle.c``): the plain definition — explicit Alg. 2
    mask, dense logits, softmax over the allowed set,
    analytic backward — in fp64, threaded over (b, kv-group).
  * :func:`alg1_row`: Alg. 1 "TTT Attention" literally, for
    one query row, as an independent third formulation.
  * :func:`fwd_packed` / :func:`bwd_packed`: packed batches (rows of sequence b at
    [cu[b], cu[b+1]), no padding), each sequence alone through fwd / bwd with
    Q_LEN = T_b (pinned in tests/test_oracle_packed.py).

Parity status: every function here is pinned by tests/test_oracle_*.py
(worked examples, closed forms, library routines, finite differences, exact
identities); see DESIGN.md §3. Nothing is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "ttt_oracle.c")

_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain gcc (-O2, no fast-math: IEEE fp64)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fPIC", "-shared",
             "-pthread", "-o", _SO, _SRC, "-lm"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        i, d, p = ctypes.c_int, ctypes.c_double, ctypes.c_void_p
        lib.ttt_oracle_mask.argtypes = [i, i, i, i]
        lib.ttt_oracle_mask.restype = i
        lib.ttt_oracle_mask_dense.argtypes = [i, i, i, p]
        lib.ttt_oracle_mask_dense.restype = None
        lib.ttt_oracle_fwd.argtypes = [i, i, i, i, i, i, p, d, p, p, p, p, p, p, p, p, i]
        lib.ttt_oracle_fwd.restype = i
        lib.ttt_oracle_bwd.argtypes = [i, i, i, i, i, i, p, d, p, p, p, p, p, p, p, p, p, p, p, p, i]
        lib.ttt_oracle_bwd.restype = i
        _lib = lib
    return _lib


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def mask(L: int, T: int, q_i: int, kv_i: int) -> bool:
    """Alg. 2 predicate for one (query, key) pair."""
    return bool(_load().ttt_oracle_mask(L, T, q_i, kv_i))


def mask_dense(L: int, T: int, j: int) -> np.ndarray:
    """Dense L x (j+1)L boolean mask of Alg. 2 for one sequence."""
    m = np.zeros((L, (j + 1) * L), dtype=np.uint8)
    _load().ttt_oracle_mask_dense(L, T, j, m.ctypes.data)
    return m.astype(bool)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def _ptr_array(arrs):
    n = len(arrs)
    arr = (ctypes.c_void_p * max(n, 1))()
    for i, a in enumerate(arrs):
        arr[i] = a.ctypes.data
    return arr


def _lens(seq_lens, B, L):
    if seq_lens is None:
        return None
    s = np.ascontiguousarray(np.asarray(seq_lens, dtype=np.int32))
    assert s.shape == (B,)
    return s


def fwd(q, k_base, v_base, k_steps, v_steps, seq_lens=None, scale=0.0, row_sel=None,
        nthreads=None):
    """Oracle forward of TTT step j = len(k_steps).

    q [B,L,Hq,D]; k_base/v_base/k_steps[i]/v_steps[i] [B,L,Hkv,D] (any float
    dtype holding exact fp32 values). Returns (out fp64 [B,L,Hq,D],
    lse fp64 [B,Hq,L]). Rows not in ``row_sel`` ([B,Hq,L] bool) are NaN.
    """
    q = _f32(q); kb = _f32(k_base); vb = _f32(v_base)
    ks = [_f32(x) for x in k_steps]; vs = [_f32(x) for x in v_steps]
    B, L, Hq, D = q.shape
    Hkv = kb.shape[2]
    j = len(ks)
    assert len(vs) == j
    lens = _lens(seq_lens, B, L)
    sel = None if row_sel is None else np.ascontiguousarray(np.asarray(row_sel, dtype=np.uint8))
    out = np.full((B, L, Hq, D), np.nan, dtype=np.float64)
    lse = np.full((B, Hq, L), np.nan, dtype=np.float64)
    kp, vp = _ptr_array(ks), _ptr_array(vs)
    st = _load().ttt_oracle_fwd(
        B, L, Hq, Hkv, D, j, None if lens is None else lens.ctypes.data, float(scale),
        q.ctypes.data, kb.ctypes.data, vb.ctypes.data, kp, vp,
        None if sel is None else sel.ctypes.data, out.ctypes.data, lse.ctypes.data,
        int(nthreads or default_threads()))
    if st == 1:
        raise ValueError("degenerate row: a query row has no allowed key (T_b < 1)")
    if st != 0:
        raise ValueError(f"oracle fwd: bad arguments (status {st})")
    return out, lse


def bwd(q, k_base, v_base, k_steps, v_steps, dout, seq_lens=None, scale=0.0, row_sel=None,
        nthreads=None):
    """Oracle backward contribution of TTT step j = len(k_steps).

    Returns dict with fp64 arrays dq [B,L,Hq,D], dk_base, dv_base [B,L,Hkv,D],
    dk_steps, dv_steps (lists of j arrays [B,L,Hkv,D]).
    """
    q = _f32(q); kb = _f32(k_base); vb = _f32(v_base); do = _f32(dout)
    ks = [_f32(x) for x in k_steps]; vs = [_f32(x) for x in v_steps]
    B, L, Hq, D = q.shape
    Hkv = kb.shape[2]
    j = len(ks)
    lens = _lens(seq_lens, B, L)
    sel = None if row_sel is None else np.ascontiguousarray(np.asarray(row_sel, dtype=np.uint8))
    dq = np.zeros((B, L, Hq, D), dtype=np.float64)
    dkb = np.zeros((B, L, Hkv, D), dtype=np.float64)
    dvb = np.zeros((B, L, Hkv, D), dtype=np.float64)
    dks = [np.zeros((B, L, Hkv, D), dtype=np.float64) for _ in range(j)]
    dvs = [np.zeros((B, L, Hkv, D), dtype=np.float64) for _ in range(j)]
    st = _load().ttt_oracle_bwd(
        B, L, Hq, Hkv, D, j, None if lens is None else lens.ctypes.data, float(scale),
        q.ctypes.data, kb.ctypes.data, vb.ctypes.data, _ptr_array(ks), _ptr_array(vs),
        do.ctypes.data, None if sel is None else sel.ctypes.data,
        dq.ctypes.data, dkb.ctypes.data, dvb.ctypes.data, _ptr_array(dks), _ptr_array(dvs),
        int(nthreads or default_threads()))
    if st == 1:
        raise ValueError("degenerate row: a query row has no allowed key (T_b < 1)")
    if st != 0:
        raise ValueError(f"oracle bwd: bad arguments (status {st})")
    return {"dq": dq, "dk_base": dkb, "dv_base": dvb, "dk_steps": dks, "dv_steps": dvs}


def _packed_spans(cu_seqlens):
    cu = np.asarray(cu_seqlens, dtype=np.int64)
    assert cu.ndim == 1 and cu[0] == 0 and np.all(np.diff(cu) >= 1)
    return [(int(cu[b]), int(cu[b + 1])) for b in range(len(cu) - 1)]


def fwd_packed(q, k_base, v_base, k_steps, v_steps, cu_seqlens, scale=0.0, nthreads=None):
    """Oracle forward of a PACKED batch: sequence b is rows
    [cu[b], cu[b+1]) of q [N,Hq,D] / k_base, v_base, k_steps[i], v_steps[i] [N,Hkv,D], with no
    padding rows. It is Alg. 2 run on each sequence alone with Q_LEN = T_b = cu[b+1] - cu[b]
    (m_pad is then vacuous) — the plain definition, one sequence at a
    time through :func:`fwd`. Returns (out fp64 [N,Hq,D], lse fp64 [Hq,N])."""
    q = np.asarray(q); Hq = q.shape[1]
    N = q.shape[0]
    out = np.empty((N,) + q.shape[1:], dtype=np.float64)
    lse = np.empty((Hq, N), dtype=np.float64)
    for r0, r1 in _packed_spans(cu_seqlens):
        sl = lambda a: np.asarray(a)[None, r0:r1]
        o, l = fwd(sl(q), sl(k_base), sl(v_base), [sl(x) for x in k_steps], [sl(x) for x in v_steps],
                   scale=scale, nthreads=nthreads)
        out[r0:r1] = o[0]
        lse[:, r0:r1] = l[0]
    return out, lse


def bwd_packed(q, k_base, v_base, k_steps, v_steps, dout, cu_seqlens, scale=0.0, nthreads=None):
    """Oracle backward of a packed batch (see :func:`fwd_packed`): each sequence alone through
    :func:`bwd` with L = T_b. Returns the dict of :func:`bwd` in the packed layout ([N,H,D])."""
    q = np.asarray(q)
    N, Hkv, D = q.shape[0], np.asarray(k_base).shape[1], q.shape[2]
    j = len(k_steps)
    res = {"dq": np.empty(q.shape, dtype=np.float64), "dk_base": np.empty((N, Hkv, D)),
           "dv_base": np.empty((N, Hkv, D)), "dk_steps": [np.empty((N, Hkv, D)) for _ in range(j)],
           "dv_steps": [np.empty((N, Hkv, D)) for _ in range(j)]}
    for r0, r1 in _packed_spans(cu_seqlens):
        sl = lambda a: np.asarray(a)[None, r0:r1]
        g = bwd(sl(q), sl(k_base), sl(v_base), [sl(x) for x in k_steps], [sl(x) for x in v_steps], sl(dout),
                scale=scale, nthreads=nthreads)
        for key in ("dq", "dk_base", "dv_base"):
            res[key][r0:r1] = g[key][0]
        for i in range(j):
            res["dk_steps"][i][r0:r1] = g["dk_steps"][i][0]
            res["dv_steps"][i][r0:r1] = g["dv_steps"][i][0]
    return res


def alg1_row(q_t, K_train, V_train, k_pred, v_pred, scale):
    """Alg. 1 "TTT Attention", literally, for ONE query.

    q_t [D]; K_train/V_train [n, D] (the prefix rows this query sees);
    k_pred/v_pred: lists of [D] cached keys/values k_i, v_i for i = T+1..t-1.
    Returns o_t [D] (fp64).
    """
    q_t = np.asarray(q_t, dtype=np.float64)
    K_train = np.asarray(K_train, dtype=np.float64)
    V_train = np.asarray(V_train, dtype=np.float64)
    S = (q_t @ K_train.T) * scale                       # S <- q_t K^train^T / sqrt(d_k)
    for k_i in k_pred:                                  # for i <- T+1 to t-1
        s_i = float(q_t @ np.asarray(k_i, np.float64)) * scale   # s_i <- q_t . k_i / sqrt(d_k)
        S = np.concatenate([S, [s_i]])                  # S <- concat(S, s_i)
    e = np.exp(S - S.max())
    alpha = e / e.sum()                                 # alpha <- softmax(S)
    n = K_train.shape[0]
    o_t = alpha[:n] @ V_train                           # o_t <- alpha . V^train
    for i, v_i in enumerate(v_pred):                    # for i <- T+1 to t-1
        o_t = o_t + alpha[n + i] * np.asarray(v_i, np.float64)   # o_t <- o_t + alpha_i v_i
    return o_t
