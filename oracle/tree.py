"""TEST INFRASTRUCTURE — fp64 CPU oracle of tree-attention verification (SURVEY.md
§8(f) NEXT #4). NOT product code; only tests/ and bench.py's cpu leg may use it. It
shares no code with the CUDA path and never imports it.

What it follows
  * PAPER.md:135 (§2.2, Stage 2, Tree Attention): "a masked attention structure constrains
    each candidate token to attend only to its ancestors, allowing the model to evaluate
    multiple hypotheses in parallel"; PAPER.md:133 (tree attention masks in TTT).
  * SPEC.md:507-509 (DraftTree): nodes in topological order, parent index, the root being
    the verified context tip; SPEC.md:528 (verify: one target forward over context + tree
    with ancestor attention masking).
  Readings (R21-R22): node t attends every context (prefix) key of its sequence
  and the tree keys of its ancestors AND itself (as a token attends itself in causal
  attention); parent[t] = -1 means the node hangs off the context tip directly.

Layout: q [B, n, Hq, D] (the n tree tokens), k/v [B, Lk, Hkv, D] with the prefix in rows
[0, P_b) and the tree tokens' own keys in rows [P_b, P_b + n); GQA kv head = h // (Hq/Hkv).
fp64 numpy on the exact input values. Pinned by tests/test_oracle_tree.py.
"""
from __future__ import annotations

import numpy as np


def ancestors_or_self(parents) -> list:
    """Per node t: the set {t, parent(t), parent(parent(t)), ...} (parents
    precede children). Raises on a parent index that is not earlier in the order."""
    parents = [int(x) for x in parents]
    out = []
    for t, p in enumerate(parents):
        if p >= t or p < -1:
            raise ValueError(f"node {t}: parent {p} must be -1 or an earlier node")
        s = {t}
        while p != -1:
            s.add(p)
            p = parents[p]
        out.append(s)
    return out


def tree_mask(prefix_len: int, parents, n_keys: int) -> np.ndarray:
    """Boolean [n, n_keys]: node t may attend key k iff k < prefix_len, or k - prefix_len is
    an ancestor of t or t itself."""
    anc = ancestors_or_self(parents)
    n = len(anc)
    m = np.zeros((n, n_keys), dtype=bool)
    for t in range(n):
        m[t, :prefix_len] = True
        for u in anc[t]:
            m[t, prefix_len + u] = True
    return m


def tree_attention(q, k, v, prefix_lens, parents, scale=0.0):
    """Dense masked softmax attention over the tree mask, fp64.
    q [B, n, Hq, D]; k, v [B, Lk, Hkv, D]; prefix_lens [B]; parents [B, n].
    Returns (out [B, n, Hq, D], lse [B, Hq, n]) with lse the natural-log logsumexp."""
    q = np.asarray(q, np.float64)
    k = np.asarray(k, np.float64)
    v = np.asarray(v, np.float64)
    B, n, Hq, D = q.shape
    Lk, Hkv = k.shape[1], k.shape[2]
    G = Hq // Hkv
    c = scale if scale else 1.0 / np.sqrt(D)
    out = np.zeros((B, n, Hq, D))
    lse = np.zeros((B, Hq, n))
    for b in range(B):
        P = int(prefix_lens[b])
        m = tree_mask(P, parents[b], Lk)
        for h in range(Hq):
            g = h // G
            s = c * (q[b, :, h, :] @ k[b, :, g, :].T)          # [n, Lk], every key (dense)
            s = np.where(m, s, -np.inf)
            mx = s.max(axis=1, keepdims=True)
            e = np.exp(s - mx)
            l = e.sum(axis=1, keepdims=True)
            out[b, :, h, :] = (e / l) @ v[b, :, g, :]
            lse[b, h, :] = (mx + np.log(l))[:, 0]
    return out, lse
