"""CPU oracle for multi-step speculative sampling (MSS) verification — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference``
legs may import this module.  It shares no code with ``paper_2505_14969_b200`` and the product path
never imports it.

SURVEY.md §8(f) NEXT #4.  STree verifies sampled (temperature > 0) trees with SpecInfer's multi-step
speculative sampling (SPEC.md:365-373 verify_mss).  The plain algorithm, DESIGN.md
reading R-mss, in float64:

    cur = root; p = p_target[cur]                         (target distribution after node cur)
    loop:
        for each child c of cur, in increasing node index (draft-rank order):
            t = tokens[c];  q = q_draft[cur]            (the draft distribution the children of cur
                                                          were drawn from)
            accept c iff  u_accept[c] * q[t] < p[t]     (i.e. u < min(1, p[t]/q[t]), u in [0, 1))
            if accepted:  path += c; cur = c; p = p_target[c]; restart the loop at the new node
            else:         r = max(0, p - q);  if sum(r) > 0: p = r / sum(r)   (else p is kept)
        no child accepted: stop
    bonus = smallest v with  sum_{w <= v} p[w]  >  u_bonus * sum_w p[w]   (inverse CDF of p;
            if rounding leaves no such v, the last v with p[v] > 0)

path_len counts the root (as stree_accept).  Every decision is a comparison of two floats; the
oracle also returns each decision's margin so a test can tell a genuine disagreement from a
rounding-order tie (several results are possible only at exact ties).
Pins: tests/test_mss_oracle.py (SPEC.md:370-372 examples, and Monte Carlo losslessness: the first
emitted token is distributed exactly as p_target[root] when the children are drawn from q).
"""
from __future__ import annotations

import numpy as np


def _children(parent, T):
    kids = [[] for _ in range(T)]
    for i in range(1, T):
        kids[int(parent[i])].append(i)
    return kids


def verify_mss_tree(tokens, parent, p_target, q_draft, u_accept, u_bonus):
    """One tree.  Returns (path list, bonus, margins list).  margins: relative distance of every
    decision from its threshold (acceptance: |u q - p| / max(p, q); bonus: distance of the threshold
    to the nearest CDF step, relative to sum p)."""
    T = len(parent)
    kids = _children(parent, T)
    cur = 0
    path = [0]
    p = np.asarray(p_target[0], np.float64)
    margins = []
    while True:
        q = np.asarray(q_draft[cur], np.float64)
        acc = None
        for c in kids[cur]:
            t = int(tokens[c])
            lhs, rhs = float(u_accept[c]) * q[t], p[t]
            margins.append(abs(lhs - rhs) / max(p[t], q[t], 1e-300))
            if lhs < rhs:
                acc = c
                break
            r = np.maximum(0.0, p - q)
            z = r.sum()
            if z > 0:
                p = r / z
        if acc is None:
            break
        path.append(acc)
        cur = acc
        p = np.asarray(p_target[cur], np.float64)
    z = p.sum()
    thr = float(u_bonus) * z
    cdf = np.cumsum(p)
    idx = np.nonzero(cdf > thr)[0]
    pos = np.nonzero(p > 0)[0]
    if len(idx):
        v = int(idx[0])
    else:
        v = int(pos[-1]) if len(pos) else 0
    lo = cdf[v - 1] if v > 0 else 0.0
    margins.append(min(abs(cdf[v] - thr), abs(thr - lo)) / max(z, 1e-300))
    return path, v, margins


def verify_mss(tokens, parent, p_target, q_draft, u_accept, u_bonus):
    """Batched: tokens/parent [B][T], p_target/q_draft [B][T][V], u_accept [B][T], u_bonus [B]
    -> (path [B][T] -1 padded, path_len [B], bonus [B], status [B], min_margin [B])."""
    parent = np.asarray(parent)
    B, T = parent.shape
    path = np.full((B, T), -1, np.int32)
    plen = np.zeros(B, np.int32)
    bonus = np.full(B, -1, np.int32)
    st = np.zeros(B, np.int32)
    mm = np.full(B, np.inf)
    for b in range(B):
        par = parent[b]
        if par[0] != -1:
            st[b] = 1
            continue
        if any(not (0 <= par[i] < i) for i in range(1, T)):
            st[b] = 2
            continue
        pth, v, m = verify_mss_tree(tokens[b], par, p_target[b], q_draft[b], u_accept[b], u_bonus[b])
        path[b, :len(pth)] = pth
        plen[b] = len(pth)
        bonus[b] = v
        mm[b] = min(m) if m else np.inf
    return path, plen, bonus, st, mm
