"""CPU oracle for tree attention and the KV-cache commit — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module.  It shares no code with
``paper_2505_14969_b200`` and the product path never imports it.

SURVEY.md §8(f) NEXT #3: the attention layers of a hybrid SSM/Transformer stack
(MambaInLlama) verify the same packed tree with a
topology-aware mask: node i attends to every committed
cache position and to the tree nodes on its own root-to-i path.  The paper gives no
formula (it cites SpecInfer); the plain definition written here is DESIGN.md reading
R-attn:

    keys(i)   = k_cache[b][0 : cache_len[b]]  ++  k_new[b][path(i)]      (path(i) root .. i)
    s_ij      = scale * <q[b][i][h], key_j>                            (kv head = h // (Hq/Hkv))
    o[b][i][h] = sum_j softmax_j(s_ij) * value_j

and the KV commit (the attention analogue of activation replay):

    cache[b][cache_len[b] + r] = new[b][path[r]]   for r < path_len[b];   cache_len[b] += path_len[b]

Everything is float64 (bf16 inputs widened exactly by the caller); path(i) is found
by walking parent pointers here, independently of any mask builder.  Pins:
tests/test_attn_oracle.py (textbook causal attention on chains and on every unrolled
root-to-leaf sequence, T = 1, ancestor-only dependence by brute force, commit-then-decode
equals decode-from-scratch).

Status codes per tree: 0 ok, 1 bad root, 2 bad parent, 3 invalid path, 5 cache capacity.
"""
from __future__ import annotations

import numpy as np


def _tree_status(par: np.ndarray) -> int:
    """PAPER.md:90 ordering precondition (R5)."""
    if len(par) == 0:
        return 0
    if par[0] != -1:
        return 1
    for i in range(1, len(par)):
        if not (0 <= par[i] < i):
            return 2
    return 0


def _path(par: np.ndarray, i: int) -> list[int]:
    """Root-to-i path s_i."""
    p = []
    while i >= 0:
        p.append(i)
        i = int(par[i])
    return p[::-1]


def tree_attn(q, k_new, v_new, k_cache, v_cache, cache_len, parent, scale):
    """q [B][T][Hq][D], k_new/v_new [B][T][Hkv][D], k_cache/v_cache [B][S][Hkv][D],
    cache_len [B], parent [B][T] -> (o float64 [B][T][Hq][D], status [B]).
    A tree with an invalid parent array gets o = 0 and its status."""
    q, k_new, v_new, k_cache, v_cache = (np.asarray(a, dtype=np.float64) for a in (q, k_new, v_new, k_cache, v_cache))
    parent = np.asarray(parent, dtype=np.int64)
    B, T, Hq, D = q.shape
    Hkv = k_new.shape[2]
    grp = Hq // Hkv
    o = np.zeros((B, T, Hq, D), np.float64)
    st = np.zeros(B, np.int32)
    for b in range(B):
        st[b] = _tree_status(parent[b])
        if st[b]:
            continue
        L = int(cache_len[b])
        for i in range(T):
            pth = _path(parent[b], i)
            for h in range(Hq):
                g = h // grp
                keys = np.concatenate([k_cache[b, :L, g, :], k_new[b, pth, g, :]], axis=0)
                vals = np.concatenate([v_cache[b, :L, g, :], v_new[b, pth, g, :]], axis=0)
                s = scale * (keys @ q[b, i, h, :])
                w = np.exp(s - s.max())
                o[b, i, h, :] = (w @ vals) / w.sum()
    return o, st


def kv_commit(k_new, v_new, k_cache, v_cache, cache_len, path, path_len, parent=None):
    """Returns (k_cache', v_cache', cache_len', status [B]) as new float64 arrays; the inputs
    are not modified.  A tree whose path is invalid (not root-anchored, not parent-linked when
    parent is given, length outside [1, T]) or would overflow the cache keeps its cache."""
    k_new, v_new = np.asarray(k_new, np.float64), np.asarray(v_new, np.float64)
    kc, vc = np.array(k_cache, np.float64), np.array(v_cache, np.float64)
    cl = np.array(cache_len, np.int64)
    B, T = k_new.shape[:2]
    S = kc.shape[1]
    st = np.zeros(B, np.int32)
    for b in range(B):
        r = int(path_len[b])
        pth = [int(v) for v in path[b][:max(r, 0)]]
        ok = 1 <= r <= T and pth[0] == 0 and all(0 <= v < T for v in pth)
        if ok and parent is not None:
            ok = _tree_status(np.asarray(parent[b])) == 0 and all(
                int(parent[b][pth[s]]) == pth[s - 1] for s in range(1, r))
        if not ok:
            st[b] = 3
            continue
        if cl[b] + r > S:
            st[b] = 5
            continue
        for s, node in enumerate(pth):
            kc[b, cl[b] + s] = k_new[b, node]
            vc[b, cl[b] + s] = v_new[b, node]
        cl[b] += r
    return kc, vc, cl, st
