"""paper_2603_18567_b200 — B200-native (sm_100a) TTT attention for EAGLE-3 draft
training (SpecForge, arXiv 2603.18567).

The compute lives in libtttattn.so (tcgen05/TMEM/TMA kernels + an fp32 CUDA-core
check mode) behind the C-ABI of include/ttt_attn.h; this package is its thin
Python binding (same names) plus the seeded input generator and the
data-parallel harness.

The library is loaded on first use of any binding name (PEP 562 module
__getattr__), so `paper_2603_18567_b200.inputs` (the seeded generators, no method
arithmetic) can be imported without mapping libtttattn.so — the bench's
reference (oracle) arm does exactly that. The first binding access without the
built library raises ImportError: there is no CPU fallback.
"""
from __future__ import annotations

import importlib

_EXPORTS = (
    "TTT_ACCUMULATE_DKV", "TTT_BF16", "TTT_FP32_CHECK", "TTT_MAX_BATCH", "TTT_MAX_STEPS", "Desc", "TTTError",
    "desc_for", "make_desc", "packed_desc", "ttt_attn_bwd", "ttt_attn_fwd", "ttt_attn_strerror", "ttt_attn_version",
    "ttt_attn_workspace_size", "ttt_attn_profile_begin", "ttt_attn_profile_end", "ttt_attn_kernel_name",
    "TTT_LOSS_MEAN", "LossDesc", "loss_desc_for", "ttt_loss_workspace_size", "ttt_loss_fwd", "ttt_loss_bwd_inplace",
    "ttt_loss_fwd_bwd_inplace", "TTT_MAX_UNROLL", "ttt_attn_bwd_unroll", "ttt_attn_bwd_unroll_workspace_size",
    "TTT_MAX_TREE", "TreeDesc", "tree_desc", "ttt_tree_attn_fwd", "ttt_tree_attn_workspace_size",
    "RopeDesc", "rope_desc", "ttt_qkv_rope_split", "ttt_rope_workspace_size", "ttt_qkv_rope_join_bwd",
)

__all__ = list(_EXPORTS)


def __getattr__(name: str):
    if name in _EXPORTS:
        lib = importlib.import_module("._lib", __name__)  # loads libtttattn.so (raises if missing)
        return getattr(lib, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")


def __dir__():
    return sorted(list(globals()) + list(_EXPORTS))
