"""ctypes binding of libtttattn.so — argument marshalling only.

Every step of the TTT attention runs in the library's CUDA kernels; this file
turns torch tensors into (device pointer, size) arguments of the C-ABI in
include/ttt_attn.h and raises on a non-zero status. There is no CPU fallback:
if the shared library is missing or was not built, import fails loudly.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TTT_ATTN_LIB") or os.path.join(_HERE, "libtttattn.so")  # env: dev A/B builds only

TTT_BF16 = 0
TTT_FP32_CHECK = 1
TTT_ACCUMULATE_DKV = 1
TTT_MAX_STEPS = 32
TTT_MAX_BATCH = 512
TTT_MAX_UNROLL = 8

STATUS = {
    0: "TTT_OK", 1: "TTT_ERR_INVALID_ARG", 2: "TTT_ERR_UNSUPPORTED", 3: "TTT_ERR_STEP_RANGE",
    4: "TTT_ERR_ALIGNMENT", 5: "TTT_ERR_DEGENERATE", 6: "TTT_ERR_WORKSPACE", 7: "TTT_ERR_CUDA",
}


class TTTError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class Desc(ctypes.Structure):
    _fields_ = [
        ("batch", ctypes.c_int32), ("seq_len", ctypes.c_int32), ("num_q_heads", ctypes.c_int32),
        ("num_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32), ("dtype", ctypes.c_int32),
        ("softmax_scale", ctypes.c_float), ("seq_lens", ctypes.POINTER(ctypes.c_int32)),
        ("cu_seqlens", ctypes.POINTER(ctypes.c_int32)),
    ]

    @property
    def packed_rows(self) -> Optional[int]:
        """N = cu_seqlens[batch] for a packed desc, else None."""
        return self.cu_seqlens[self.batch] if self.cu_seqlens else None


class TreeDesc(ctypes.Structure):
    """ttt_tree_desc (include/ttt_attn.h)."""
    _fields_ = [("batch", ctypes.c_int32), ("num_tree", ctypes.c_int32), ("kv_len", ctypes.c_int32),
                ("num_q_heads", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("softmax_scale", ctypes.c_float), ("dtype", ctypes.c_int32),
                ("prefix_lens", ctypes.POINTER(ctypes.c_int32))]


TTT_MAX_TREE = 64


class RopeDesc(ctypes.Structure):
    """ttt_rope_desc (include/ttt_attn.h)."""
    _fields_ = [("batch", ctypes.c_int32), ("seq_len", ctypes.c_int32), ("num_q_heads", ctypes.c_int32),
                ("num_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32), ("rope_base", ctypes.c_float)]


class LossDesc(ctypes.Structure):
    """ttt_loss_desc (include/ttt_loss.h)."""
    _fields_ = [("rows", ctypes.c_int64), ("vocab", ctypes.c_int32), ("dtype", ctypes.c_int32)]


TTT_LOSS_MEAN = 1


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: build the CUDA library first (`make` or __graft_entry__.build()); "
            "there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    vp, sz, i, u = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint
    pd = ctypes.POINTER(Desc)
    lib.ttt_attn_workspace_size.argtypes = [pd, i, i]
    lib.ttt_attn_workspace_size.restype = sz
    lib.ttt_attn_fwd.argtypes = [pd, i, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    lib.ttt_attn_fwd.restype = i
    lib.ttt_attn_bwd.argtypes = [pd, i, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, u, vp, sz, vp]
    lib.ttt_attn_bwd.restype = i
    lib.ttt_attn_bwd_unroll_workspace_size.argtypes = [pd, i]
    lib.ttt_attn_bwd_unroll_workspace_size.restype = sz
    lib.ttt_attn_bwd_unroll.argtypes = [pd, i, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, u, vp, sz, vp]
    lib.ttt_attn_bwd_unroll.restype = i
    ptd = ctypes.POINTER(TreeDesc)
    lib.ttt_tree_attn_workspace_size.argtypes = [ptd]
    lib.ttt_tree_attn_workspace_size.restype = sz
    lib.ttt_tree_attn_fwd.argtypes = [ptd, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    lib.ttt_tree_attn_fwd.restype = i
    prd = ctypes.POINTER(RopeDesc)
    lib.ttt_rope_workspace_size.argtypes = [prd, i]
    lib.ttt_rope_workspace_size.restype = sz
    lib.ttt_qkv_rope_split.argtypes = [prd, vp, vp, vp, vp, vp, vp, sz, vp]
    lib.ttt_qkv_rope_split.restype = i
    lib.ttt_qkv_rope_join_bwd.argtypes = [prd, vp, vp, vp, vp, vp, vp, sz, vp]
    lib.ttt_qkv_rope_join_bwd.restype = i
    lib.ttt_attn_strerror.argtypes = [i]
    lib.ttt_attn_strerror.restype = ctypes.c_char_p
    lib.ttt_attn_version.argtypes = []
    lib.ttt_attn_version.restype = ctypes.c_char_p
    lib.ttt_attn_profile_begin.argtypes = []
    lib.ttt_attn_profile_begin.restype = i
    lib.ttt_attn_profile_end.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int), i]
    lib.ttt_attn_profile_end.restype = i
    lib.ttt_attn_kernel_name.argtypes = [i]
    lib.ttt_attn_kernel_name.restype = ctypes.c_char_p
    pl = ctypes.POINTER(LossDesc)
    f = ctypes.c_float
    lib.ttt_loss_workspace_size.argtypes = [pl]
    lib.ttt_loss_workspace_size.restype = sz
    lib.ttt_loss_fwd.argtypes = [pl, vp, vp, vp, vp, vp, vp, sz, vp]
    lib.ttt_loss_fwd.restype = i
    lib.ttt_loss_bwd_inplace.argtypes = [pl, vp, vp, vp, vp, f, u, vp, vp, sz, vp]
    lib.ttt_loss_bwd_inplace.restype = i
    lib.ttt_loss_fwd_bwd_inplace.argtypes = [pl, vp, vp, vp, vp, f, u, vp, vp, vp, vp, sz, vp]
    lib.ttt_loss_fwd_bwd_inplace.restype = i
    return lib


_lib = _load()


def ttt_attn_strerror(code: int) -> str:
    return _lib.ttt_attn_strerror(int(code)).decode()


def ttt_attn_version() -> str:
    return _lib.ttt_attn_version().decode()


def make_desc(batch: int, seq_len: int, num_q_heads: int, num_kv_heads: int, head_dim: int,
              dtype: int = TTT_BF16, softmax_scale: float = 0.0,
              seq_lens: Optional[Sequence[int]] = None, cu_seqlens: Optional[Sequence[int]] = None) -> Desc:
    """ttt_attn_desc. cu_seqlens (batch + 1 offsets, host ints) selects the packed layout: q [N, Hq, D],
    k / v [N, Hkv, D], lse [Hq, N] with N = cu_seqlens[-1]; seq_len is then ignored."""
    d = Desc()
    d.batch, d.seq_len, d.num_q_heads, d.num_kv_heads, d.head_dim = (
        int(batch), int(seq_len), int(num_q_heads), int(num_kv_heads), int(head_dim))
    d.dtype, d.softmax_scale = int(dtype), float(softmax_scale)
    if seq_lens is not None:
        arr = (ctypes.c_int32 * int(batch))(*[int(x) for x in seq_lens])
        d._seq_lens_keepalive = arr  # keep the host array alive with the desc
        d.seq_lens = ctypes.cast(arr, ctypes.POINTER(ctypes.c_int32))
    if cu_seqlens is not None:
        cu = [int(x) for x in cu_seqlens]
        if len(cu) != int(batch) + 1:
            raise TTTError(1, f"cu_seqlens needs batch + 1 = {int(batch) + 1} entries (got {len(cu)})")
        carr = (ctypes.c_int32 * len(cu))(*cu)
        d._cu_keepalive = carr
        d.cu_seqlens = ctypes.cast(carr, ctypes.POINTER(ctypes.c_int32))
    return d


def packed_desc(cu_seqlens: Sequence[int], num_q_heads: int, num_kv_heads: int, head_dim: int,
                dtype: int = TTT_BF16, softmax_scale: float = 0.0) -> Desc:
    """Desc of a packed batch: sequence b = rows [cu_seqlens[b], cu_seqlens[b+1])."""
    cu = [int(x) for x in cu_seqlens]
    return make_desc(len(cu) - 1, max(1, max(b - a for a, b in zip(cu[:-1], cu[1:]))), num_q_heads, num_kv_heads,
                     head_dim, dtype, softmax_scale, None, cu)


def desc_for(q: torch.Tensor, k_base: torch.Tensor, seq_lens=None, softmax_scale: float = 0.0) -> Desc:
    """Desc from BSHD tensors: q [B,L,Hq,D], k_base [B,L,Hkv,D]."""
    B, L, Hq, D = q.shape
    dt = TTT_FP32_CHECK if q.dtype == torch.float32 else TTT_BF16
    return make_desc(B, L, Hq, k_base.shape[2], D, dt, softmax_scale, seq_lens)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _ptr_list(ts: Sequence[torch.Tensor]):
    arr = (ctypes.c_void_p * max(len(ts), 1))()
    for n, t in enumerate(ts):
        arr[n] = t.data_ptr()
    return arr


def _stream(stream) -> ctypes.c_void_p:
    if stream is None:
        if not torch.cuda.is_available():  # validation-only calls on a CPU host
            return ctypes.c_void_p(0)
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _check(code: int):
    if code != 0:
        raise TTTError(code, ttt_attn_strerror(code))


def _validate(spec, *, device=None):
    """Host-side checks of the torch tensors handed to a C-ABI call: the C side sees
    only raw pointers, so a non-contiguous view, a dtype mismatch or a tensor on another device
    would otherwise read or write the wrong bytes. `spec`: (name, tensor, dtype | None, shape |
    None) tuples; entries that are not torch tensors (None, or the pointer stand-ins of the
    CPU-only validation tests) are skipped. Raises TTTError(TTT_ERR_INVALID_ARG)."""
    dev = device
    for name, t, dt, shape in spec:
        if not isinstance(t, torch.Tensor):
            continue
        if not t.is_cuda:
            raise TTTError(1, f"{name} must be a CUDA tensor (got {t.device})")
        if dev is None:
            dev = t.device
        elif t.device != dev:
            raise TTTError(1, f"{name} is on {t.device}, the other arguments on {dev}")
        if not t.is_contiguous():
            raise TTTError(1, f"{name} must be contiguous (row-major); pass .contiguous()")
        if dt is not None and t.dtype != dt:
            raise TTTError(1, f"{name} must be {dt} (got {t.dtype})")
        if shape is not None and tuple(t.shape) != tuple(shape):
            raise TTTError(1, f"{name} must have shape {tuple(shape)} (got {tuple(t.shape)})")
    return dev


def _attn_shapes(desc: "Desc"):
    B, L, Hq, Hkv, D = desc.batch, desc.seq_len, desc.num_q_heads, desc.num_kv_heads, desc.head_dim
    dt = torch.float32 if desc.dtype == TTT_FP32_CHECK else torch.bfloat16
    N = desc.packed_rows
    if N is not None:  # packed layout
        return dt, (N, Hq, D), (N, Hkv, D), (Hq, N)
    return dt, (B, L, Hq, D), (B, L, Hkv, D), (B, Hq, L)


def _check_list(name: str, ts, n: int):
    if len(ts) < n:
        raise TTTError(1, f"{name} has {len(ts)} entries, step needs {n}")


TTT_KERNEL_KINDS = 10


def ttt_attn_kernel_name(kind: int) -> str:
    return _lib.ttt_attn_kernel_name(int(kind)).decode()


def ttt_attn_profile_begin() -> None:
    """Arm per-kernel CUDA-event timing for this host thread (include/ttt_attn.h)."""
    rc = _lib.ttt_attn_profile_begin()
    if rc < 0:
        _check(-rc)


def ttt_attn_profile_end() -> dict:
    """Disarm; return {kernel_name: (total_ms, launches)} for kinds that ran."""
    ms = (ctypes.c_double * TTT_KERNEL_KINDS)()
    n = (ctypes.c_int * TTT_KERNEL_KINDS)()
    rc = _lib.ttt_attn_profile_end(ms, n, TTT_KERNEL_KINDS)
    if rc < 0:
        _check(-rc)
    return {ttt_attn_kernel_name(k): (ms[k], n[k]) for k in range(rc) if n[k] > 0}


def ttt_attn_workspace_size(desc: Desc, step: int, is_bwd: bool) -> int:
    return int(_lib.ttt_attn_workspace_size(ctypes.byref(desc), int(step), int(bool(is_bwd))))


def ttt_attn_fwd(desc: Desc, step: int, q, k_base, v_base, k_steps, v_steps, out, lse,
                 out_lo=None, workspace=None, stream=None) -> None:
    """Enqueue ttt_attn_fwd (include/ttt_attn.h) on `stream` (default: current)."""
    dt, qs, kvs, ls = _attn_shapes(desc)
    _check_list("k_steps", k_steps, step)
    _check_list("v_steps", v_steps, step)
    _validate([("q", q, dt, qs), ("k_base", k_base, dt, kvs), ("v_base", v_base, dt, kvs), ("out", out, dt, qs),
               ("out_lo", out_lo, torch.bfloat16, qs), ("lse", lse, torch.float32, ls)]
              + [(f"k_steps[{i}]", k_steps[i], dt, kvs) for i in range(max(step, 0))]
              + [(f"v_steps[{i}]", v_steps[i], dt, kvs) for i in range(max(step, 0))])
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check(_lib.ttt_attn_fwd(ctypes.byref(desc), int(step), _ptr(q), _ptr(k_base), _ptr(v_base),
                             _ptr_list(k_steps[:step]), _ptr_list(v_steps[:step]), _ptr(out), _ptr(out_lo),
                             _ptr(lse), _ptr(workspace), ws_bytes, _stream(stream)))


def ttt_attn_bwd(desc: Desc, step: int, q, k_base, v_base, k_steps, v_steps, out, lse, dout,
                 dq, dk_base, dv_base, dk_steps, dv_steps, flags: int = 0, workspace=None,
                 stream=None, out_lo=None) -> None:
    """Enqueue ttt_attn_bwd (include/ttt_attn.h) on `stream` (default: current)."""
    dt, qs, kvs, ls = _attn_shapes(desc)
    f32 = torch.float32
    for nm, lst in (("k_steps", k_steps), ("v_steps", v_steps), ("dk_steps", dk_steps), ("dv_steps", dv_steps)):
        _check_list(nm, lst, step)
    n = max(step, 0)
    _validate([("q", q, dt, qs), ("k_base", k_base, dt, kvs), ("v_base", v_base, dt, kvs), ("out", out, dt, qs),
               ("out_lo", out_lo, torch.bfloat16, qs), ("lse", lse, f32, ls), ("dout", dout, dt, qs),
               ("dq", dq, dt, qs), ("dk_base", dk_base, f32, kvs), ("dv_base", dv_base, f32, kvs)]
              + [(f"k_steps[{i}]", k_steps[i], dt, kvs) for i in range(n)]
              + [(f"v_steps[{i}]", v_steps[i], dt, kvs) for i in range(n)]
              + [(f"dk_steps[{i}]", dk_steps[i], f32, kvs) for i in range(n)]
              + [(f"dv_steps[{i}]", dv_steps[i], f32, kvs) for i in range(n)]
              + [("workspace", workspace, None, None)])
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check(_lib.ttt_attn_bwd(ctypes.byref(desc), int(step), _ptr(q), _ptr(k_base), _ptr(v_base),
                             _ptr_list(k_steps[:step]), _ptr_list(v_steps[:step]), _ptr(out), _ptr(out_lo),
                             _ptr(lse), _ptr(dout), _ptr(dq), _ptr(dk_base), _ptr(dv_base),
                             _ptr_list(dk_steps[:step]), _ptr_list(dv_steps[:step]), int(flags),
                             _ptr(workspace), ws_bytes, _stream(stream)))



def ttt_attn_bwd_unroll_workspace_size(desc: Desc, num_steps: int) -> int:
    return int(_lib.ttt_attn_bwd_unroll_workspace_size(ctypes.byref(desc), int(num_steps)))


def ttt_attn_bwd_unroll(desc: Desc, q: Sequence, k_base, v_base, k_steps, v_steps, out: Sequence, lse: Sequence,
                        dout: Sequence, dq: Sequence, dk_base, dv_base, dk_steps, dv_steps, flags: int = 0,
                        workspace=None, stream=None, out_lo: Optional[Sequence] = None) -> None:
    """Enqueue ttt_attn_bwd_unroll (include/ttt_attn.h): the S = len(q) backward calls of one
    unroll (j = S-1 .. 0) in one call; per-step lists q / out / out_lo / lse / dout / dq."""
    S = len(q)
    dt, qs, kvs, ls = _attn_shapes(desc)
    f32 = torch.float32
    for nm, lst in (("out", out), ("lse", lse), ("dout", dout), ("dq", dq)):
        _check_list(nm, lst, S)
    if out_lo is not None:
        _check_list("out_lo", out_lo, S)
    for nm, lst in (("k_steps", k_steps), ("v_steps", v_steps), ("dk_steps", dk_steps), ("dv_steps", dv_steps)):
        _check_list(nm, lst, S - 1)
    spec = [("k_base", k_base, dt, kvs), ("v_base", v_base, dt, kvs), ("dk_base", dk_base, f32, kvs),
            ("dv_base", dv_base, f32, kvs), ("workspace", workspace, None, None)]
    for j in range(S):
        spec += [(f"q[{j}]", q[j], dt, qs), (f"out[{j}]", out[j], dt, qs), (f"lse[{j}]", lse[j], f32, ls),
                 (f"dout[{j}]", dout[j], dt, qs), (f"dq[{j}]", dq[j], dt, qs)]
        if out_lo is not None:
            spec.append((f"out_lo[{j}]", out_lo[j], torch.bfloat16, qs))
    for i in range(max(S - 1, 0)):
        spec += [(f"k_steps[{i}]", k_steps[i], dt, kvs), (f"v_steps[{i}]", v_steps[i], dt, kvs),
                 (f"dk_steps[{i}]", dk_steps[i], f32, kvs), (f"dv_steps[{i}]", dv_steps[i], f32, kvs)]
    _validate(spec)
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check(_lib.ttt_attn_bwd_unroll(
        ctypes.byref(desc), S, _ptr_list(q), _ptr(k_base), _ptr(v_base), _ptr_list(k_steps[:S - 1]),
        _ptr_list(v_steps[:S - 1]), _ptr_list(out), None if out_lo is None else _ptr_list(out_lo), _ptr_list(lse),
        _ptr_list(dout), _ptr_list(dq), _ptr(dk_base), _ptr(dv_base), _ptr_list(dk_steps[:S - 1]),
        _ptr_list(dv_steps[:S - 1]), int(flags), _ptr(workspace), ws_bytes, _stream(stream)))



def tree_desc(batch: int, num_tree: int, kv_len: int, num_q_heads: int, num_kv_heads: int, head_dim: int,
              prefix_lens: Sequence[int], softmax_scale: float = 0.0, dtype: int = TTT_BF16) -> TreeDesc:
    d = TreeDesc()
    d.dtype = int(dtype)
    d.batch, d.num_tree, d.kv_len = int(batch), int(num_tree), int(kv_len)
    d.num_q_heads, d.num_kv_heads, d.head_dim = int(num_q_heads), int(num_kv_heads), int(head_dim)
    d.softmax_scale = float(softmax_scale)
    arr = (ctypes.c_int32 * int(batch))(*[int(x) for x in prefix_lens])
    d._keepalive = arr
    d.prefix_lens = ctypes.cast(arr, ctypes.POINTER(ctypes.c_int32))
    return d


def ttt_tree_attn_workspace_size(desc: TreeDesc) -> int:
    return int(_lib.ttt_tree_attn_workspace_size(ctypes.byref(desc)))


def ttt_tree_attn_fwd(desc: TreeDesc, q, k_cache, v_cache, parents, out, lse, workspace, stream=None) -> None:
    """Enqueue ttt_tree_attn_fwd (include/ttt_attn.h): tree-attention verification forward."""
    dt = torch.float32 if desc.dtype == TTT_FP32_CHECK else torch.bfloat16
    B, n, KV, Hq, Hkv, D = desc.batch, desc.num_tree, desc.kv_len, desc.num_q_heads, desc.num_kv_heads, desc.head_dim
    _validate([("q", q, dt, (B, n, Hq, D)), ("k_cache", k_cache, dt, (B, KV, Hkv, D)),
               ("v_cache", v_cache, dt, (B, KV, Hkv, D)), ("parents", parents, torch.int32, (B, n)),
               ("out", out, dt, (B, n, Hq, D)), ("lse", lse, torch.float32, (B, Hq, n)),
               ("workspace", workspace, None, None)])
    _check(_lib.ttt_tree_attn_fwd(ctypes.byref(desc), _ptr(q), _ptr(k_cache), _ptr(v_cache), _ptr(parents),
                                  _ptr(out), _ptr(lse), _ptr(workspace), _nbytes(workspace), _stream(stream)))



def rope_desc(batch: int, seq_len: int, num_q_heads: int, num_kv_heads: int, head_dim: int,
              rope_base: float = 500000.0) -> RopeDesc:
    d = RopeDesc()
    d.batch, d.seq_len, d.num_q_heads, d.num_kv_heads, d.head_dim = (
        int(batch), int(seq_len), int(num_q_heads), int(num_kv_heads), int(head_dim))
    d.rope_base = float(rope_base)
    return d


def ttt_rope_workspace_size(desc: RopeDesc, per_sequence_positions: bool = False) -> int:
    return int(_lib.ttt_rope_workspace_size(ctypes.byref(desc), int(bool(per_sequence_positions))))


def ttt_qkv_rope_split(desc: RopeDesc, qkv, q, k_slot, v_slot, workspace, positions=None, stream=None) -> None:
    """Enqueue ttt_qkv_rope_split (include/ttt_attn.h): RoPE'd q and the step's K / V slots from a
    fused q/k/v projection output, one HBM pass."""
    B, Lr, Hq, Hkv, D = desc.batch, desc.seq_len, desc.num_q_heads, desc.num_kv_heads, desc.head_dim
    bf = torch.bfloat16
    _validate([("qkv", qkv, bf, (B, Lr, Hq + 2 * Hkv, D)), ("positions", positions, torch.int32, (B, Lr)),
               ("q", q, bf, (B, Lr, Hq, D)), ("k_slot", k_slot, bf, (B, Lr, Hkv, D)),
               ("v_slot", v_slot, bf, (B, Lr, Hkv, D)), ("workspace", workspace, None, None)])
    _check(_lib.ttt_qkv_rope_split(ctypes.byref(desc), _ptr(qkv), _ptr(positions), _ptr(q), _ptr(k_slot),
                                   _ptr(v_slot), _ptr(workspace), _nbytes(workspace), _stream(stream)))



def ttt_qkv_rope_join_bwd(desc: RopeDesc, dq, dk_slot, dv_slot, dqkv, workspace, positions=None, stream=None) -> None:
    """Enqueue ttt_qkv_rope_join_bwd: the adjoint of ttt_qkv_rope_split (gradients -> dqkv)."""
    B, Lr, Hq, Hkv, D = desc.batch, desc.seq_len, desc.num_q_heads, desc.num_kv_heads, desc.head_dim
    bf = torch.bfloat16
    _validate([("dq", dq, bf, (B, Lr, Hq, D)), ("dk_slot", dk_slot, bf, (B, Lr, Hkv, D)),
               ("dv_slot", dv_slot, bf, (B, Lr, Hkv, D)), ("positions", positions, torch.int32, (B, Lr)),
               ("dqkv", dqkv, bf, (B, Lr, Hq + 2 * Hkv, D)), ("workspace", workspace, None, None)])
    _check(_lib.ttt_qkv_rope_join_bwd(ctypes.byref(desc), _ptr(dq), _ptr(dk_slot), _ptr(dv_slot), _ptr(positions),
                                      _ptr(dqkv), _ptr(workspace), _nbytes(workspace), _stream(stream)))


# ---- masked soft-label log-softmax loss + Alg. 3 in-place backward (include/ttt_loss.h) ----

def loss_desc_for(z: torch.Tensor) -> LossDesc:
    """LossDesc from logits z [..., V] (rows = product of the leading dims)."""
    d = LossDesc()
    d.vocab = int(z.shape[-1])
    d.rows = int(z.numel() // max(d.vocab, 1))
    d.dtype = TTT_FP32_CHECK if z.dtype == torch.float32 else TTT_BF16
    return d


def ttt_loss_workspace_size(desc: LossDesc) -> int:
    return int(_lib.ttt_loss_workspace_size(ctypes.byref(desc)))


def _nbytes(t) -> int:
    return 0 if t is None else t.numel() * t.element_size()


def _loss_validate(desc: LossDesc, z, p, mask, g_rows=None, grad=None, lse=None, stats=None, workspace=None):
    dt = torch.float32 if desc.dtype == TTT_FP32_CHECK else torch.bfloat16
    N, V = desc.rows, desc.vocab
    _validate([("z", z, dt, None), ("p", p, dt, None), ("grad", grad, dt, None), ("mask", mask, torch.uint8, None),
               ("g_rows", g_rows, torch.float32, None), ("lse", lse, torch.float32, None),
               ("stats", stats, torch.float64, None), ("workspace", workspace, None, None)])
    for nm, t, n in (("z", z, N * V), ("p", p, N * V), ("grad", grad, N * V), ("mask", mask, N),
                     ("g_rows", g_rows, N), ("lse", lse, N), ("stats", stats, 2)):
        if isinstance(t, torch.Tensor) and t.numel() != n:
            raise TTTError(1, f"{nm} has {t.numel()} elements, expected {n}")


def ttt_loss_fwd(desc: LossDesc, z, p, mask, stats, workspace, lse=None, stream=None) -> None:
    """Enqueue ttt_loss_fwd: stats (fp64 [2]) = {masked mean loss, masked-row count}."""
    _loss_validate(desc, z, p, mask, lse=lse, stats=stats, workspace=workspace)
    _check(_lib.ttt_loss_fwd(ctypes.byref(desc), _ptr(z), _ptr(p), _ptr(mask), _ptr(lse), _ptr(stats),
                             _ptr(workspace), _nbytes(workspace), _stream(stream)))


def ttt_loss_bwd_inplace(desc: LossDesc, z, p, mask, workspace, g_scale: float = 1.0, flags: int = TTT_LOSS_MEAN,
                         g_rows=None, grad=None, stream=None) -> None:
    """Enqueue Alg. 3: z <- dL/dz in place (or into `grad` when given)."""
    _loss_validate(desc, z, p, mask, g_rows=g_rows, grad=grad, workspace=workspace)
    _check(_lib.ttt_loss_bwd_inplace(ctypes.byref(desc), _ptr(z), _ptr(p), _ptr(mask), _ptr(g_rows),
                                     float(g_scale), int(flags), _ptr(grad), _ptr(workspace), _nbytes(workspace),
                                     _stream(stream)))


def ttt_loss_fwd_bwd_inplace(desc: LossDesc, z, p, mask, stats, workspace, g_scale: float = 1.0,
                             flags: int = TTT_LOSS_MEAN, g_rows=None, grad=None, lse=None, stream=None) -> None:
    """Enqueue the fused loss + Alg. 3 backward (one pass: z, p read once, gradient written over z)."""
    _loss_validate(desc, z, p, mask, g_rows=g_rows, grad=grad, lse=lse, stats=stats, workspace=workspace)
    _check(_lib.ttt_loss_fwd_bwd_inplace(ctypes.byref(desc), _ptr(z), _ptr(p), _ptr(mask), _ptr(g_rows),
                                         float(g_scale), int(flags), _ptr(grad), _ptr(lse), _ptr(stats),
                                         _ptr(workspace), _nbytes(workspace), _stream(stream)))
