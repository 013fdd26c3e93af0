"""Seeded tree-shape generators.

Shared by the oracle side and the CUDA side as *inputs only*: this module
holds tree topologies (parent arrays) and nothing of the method's arithmetic.

Every generator returns ``parent`` as an ``int32`` array with ``parent[0] == -1``
and ``0 <= parent[i] < i`` for ``i >= 1`` (topological order, PAPER.md:90
"we can always organize the tokens in the sequence such that L_{t,i}=0 for i>t").
"""
from __future__ import annotations

import numpy as np


def heap_kary(n: int, k: int) -> np.ndarray:
    """Heap-ordered k-ary tree: parent(i) = (i-1)//k.  n=2^L-1, k=2 is the
    full binary tree with L levels used at PAPER.md:218 (15/31/63 tokens)."""
    if n < 1:
        return np.zeros(0, dtype=np.int32)
    p = (np.arange(n, dtype=np.int64) - 1) // k
    p[0] = -1
    return p.astype(np.int32)


def chain(n: int) -> np.ndarray:
    """Chain (a plain sequence): parent(i) = i-1.  Its mask is the causal
    lower-triangular mask of PAPER.md:104."""
    p = np.arange(n, dtype=np.int64) - 1
    return p.astype(np.int32)


def star(n: int) -> np.ndarray:
    """Root with n-1 children (depth 1)."""
    p = np.zeros(n, dtype=np.int32)
    if n:
        p[0] = -1
    return p


def beam(m_beams: int, n_steps: int, rng: np.random.Generator) -> np.ndarray:
    """Beam-search tree of PAPER.md:309: root + n_steps layers of m_beams
    nodes; the root gives the first layer, each later node picks a (seeded)
    parent in the previous layer.  1 + M*N nodes (M=3,N=4 -> 13)."""
    parent = [-1]
    prev = [0]
    for _ in range(n_steps):
        layer = []
        for _m in range(m_beams):
            parent.append(int(prev[int(rng.integers(len(prev)))]) if len(prev) > 1 else prev[0])
            layer.append(len(parent) - 1)
        prev = layer
    return np.asarray(parent, dtype=np.int32)


# Static trees A-E of PAPER.md:411-415 (tab:static-configs) as BFS layer widths
# (max width, drafted depth excluding the root, tokens incl. the root).
# The adjacency is figure-only; SURVEY.md Appendix A fixes
# these widths, children distributed left-first.
STATIC_LAYER_WIDTHS = {
    "A": (3, 3, 3, 3),       # (3,4,13)
    "B": (4, 8, 16),         # (16,3,29)
    "C": (3, 6, 6),          # (6,3,16)
    "D": (4, 4, 2, 2),       # (4,4,13)
    "E": (3, 3, 3, 3, 3),    # (3,5,16)
}


def static_tree(name: str) -> np.ndarray:
    widths = STATIC_LAYER_WIDTHS[name]
    parent = [-1]
    prev = [0]
    for w in widths:
        q = -(-w // len(prev))  # ceil: children per parent, left-first
        layer = []
        for c in range(w):
            parent.append(prev[c // q])
            layer.append(len(parent) - 1)
        prev = layer
    return np.asarray(parent, dtype=np.int32)


def random_recursive(n: int, b_max: int, rng: np.random.Generator) -> np.ndarray:
    """parent(i) uniform over earlier nodes that have fewer than b_max children."""
    parent = np.empty(n, dtype=np.int32)
    if n == 0:
        return parent
    parent[0] = -1
    nchild = np.zeros(n, dtype=np.int64)
    for i in range(1, n):
        cand = np.flatnonzero(nchild[:i] < b_max)
        p = int(cand[int(rng.integers(len(cand)))])
        parent[i] = p
        nchild[p] += 1
    return parent


def random_parent_array(n: int, rng: np.random.Generator) -> np.ndarray:
    """Uniform over all topologically ordered trees: parent(i) ~ U{0..i-1}."""
    parent = np.empty(n, dtype=np.int32)
    if n:
        parent[0] = -1
    for i in range(1, n):
        parent[i] = int(rng.integers(i))
    return parent


def make_tree(kind: str, n: int = 0, k: int = 2, seed: int = 0, **kw) -> np.ndarray:
    """Dispatch by name: heap/chain/star/beam/static/random/recursive."""
    rng = np.random.default_rng(seed)
    if kind == "heap":
        return heap_kary(n, k)
    if kind == "chain":
        return chain(n)
    if kind == "star":
        return star(n)
    if kind == "beam":
        return beam(kw["m"], kw["steps"], rng)
    if kind == "static":
        return static_tree(kw["name"])
    if kind == "recursive":
        return random_recursive(n, kw.get("b_max", 4), rng)
    if kind == "random":
        return random_parent_array(n, rng)
    raise ValueError(f"unknown tree kind {kind!r}")


def children_lists(parent: np.ndarray) -> list[list[int]]:
    ch: list[list[int]] = [[] for _ in range(len(parent))]
    for i in range(1, len(parent)):
        ch[int(parent[i])].append(i)
    return ch


def pad_batch(parents: list[np.ndarray], T: int) -> np.ndarray:
    """Stack trees of equal size T into [B][T]."""
    out = np.stack([np.asarray(p, dtype=np.int32) for p in parents])
    assert out.shape[1] == T
    return out
