"""Seeded synthetic inputs for MSS verification.  Random values only.

Recipe: target logits ~ N(0, sigma^2) per (tree, node) over the vocabulary (sigma = 3: a peaked
distribution, top token ~ a few % of the mass at V = 50,280); draft logits = target logits + N(0, 1)
(a draft model close to the target); both softmaxed in float64 and stored float32.  Children's tokens
are drawn from the draft distribution of their parent (i.i.d., so siblings may repeat, as in
SpecInfer's MSS), u_accept ~ U[0, 1) per node, u_bonus ~ U[0, 1) per tree.
Seeds: BASE_SEED + 200 + case.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from . import trees
from .inputs import BASE_SEED, VOCAB


@dataclasses.dataclass
class MssProblem:
    tokens: np.ndarray      # [B][T] int32
    parent: np.ndarray      # [B][T] int32
    p_target: np.ndarray    # [B][T][V] float32
    q_draft: np.ndarray     # [B][T][V] float32
    u_accept: np.ndarray    # [B][T] float32
    u_bonus: np.ndarray     # [B] float32


def _softmax(x):
    x = x - x.max(axis=-1, keepdims=True)
    e = np.exp(x)
    return e / e.sum(axis=-1, keepdims=True)


def make_mss_problem(parent: np.ndarray, vocab: int, seed: int, sigma: float = 3.0, draft_noise: float = 1.0,
                     same=False) -> MssProblem:
    rng = np.random.default_rng(seed)
    parent = np.asarray(parent, np.int32)
    B, T = parent.shape
    p = np.empty((B, T, vocab), np.float32)
    q = np.empty((B, T, vocab), np.float32)
    tokens = np.zeros((B, T), np.int32)
    for b in range(B):   # per tree: bounded float64 temporaries
        lt = rng.standard_normal((T, vocab)) * sigma
        pb = _softmax(lt)
        qb = pb if same else _softmax(lt + rng.standard_normal((T, vocab)) * draft_noise)
        p[b], q[b] = pb, qb
        cdf = np.cumsum(qb, axis=1)
        for i in range(1, T):
            row = cdf[parent[b, i]]
            tokens[b, i] = min(int(np.searchsorted(row, rng.random() * row[-1], side="right")), vocab - 1)
        tokens[b, 0] = rng.integers(0, vocab)
    u_acc = rng.random((B, T)).astype(np.float32)
    u_bon = rng.random(B).astype(np.float32)
    return MssProblem(tokens, parent, p, q, u_acc, u_bon)


def mss_config(name: str) -> MssProblem:
    """'c4': the bench workload — the 16 random recursive 64-node trees, V = 50,280."""
    if name == "c4":
        seed = BASE_SEED + 200
        par = np.stack([trees.random_recursive(64, 4, np.random.default_rng(seed * 1000 + b)) for b in range(16)])
        return make_mss_problem(par, VOCAB, seed)
    raise KeyError(name)
