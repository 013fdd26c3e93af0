"""Seeded synthetic inputs for the tree-verify hot path.

Shared by both sides as INPUTS only: value distributions, shapes and the
bf16 storage format.  No arithmetic of the method lives here (no decay, no
segsum, no scan, no acceptance rule).

Value recipe (Mamba-2 init ranges):
  A_h  = -U[1, 16]                       (per head, fp32)
  dt   ~ log-uniform[1e-3, 1e-1]         (per node and head, fp32, post-softplus)
  x, B, C ~ N(0, 1) then cast to the io dtype (bf16 = round-to-nearest-even)
  D_h  = 1 + 0.1 N(0, 1)
  h0   ~ N(0, 1)                          (fp32 state)
Seeds: 250514969 + config index, one sub-seed per tree.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from . import trees

BASE_SEED = 250514969
VOCAB = 50280


# ----------------------------------------------------------------------------
# bf16 storage format (raw uint16 bit patterns), round-to-nearest-even.
# ----------------------------------------------------------------------------
def f32_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rnd = ((u >> 16) & 1) + 0x7FFF
    out = ((u + rnd) >> 16).astype(np.uint16)
    nan = np.isnan(np.asarray(a, dtype=np.float32))
    if nan.any():
        out[nan] = 0x7FC0
    return out


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


@dataclasses.dataclass
class Dims:
    batch: int
    n_nodes: int
    n_heads: int
    head_dim: int
    d_state: int
    n_groups: int = 1
    io_dtype: str = "bf16"  # "bf16" or "f32"


@dataclasses.dataclass
class Problem:
    """One layer's tree-verify inputs.  Arrays are numpy, row-major:
    x[B][T][H][P] (io), dt[B][T][H] f32, A[H] f32, Bm/Cm[B][T][G][N] (io),
    D[H] f32, h0[B][H][P][N] f32, parent[B][T] i32.
    io arrays are float32 when io_dtype == 'f32' and uint16 bf16 bits otherwise."""
    dims: Dims
    x: np.ndarray
    dt: np.ndarray
    A: np.ndarray
    Bm: np.ndarray
    Cm: np.ndarray
    D: np.ndarray
    h0: np.ndarray
    parent: np.ndarray

    def io_as_f32(self, name: str) -> np.ndarray:
        a = getattr(self, name)
        return bf16_bits_to_f32(a) if self.dims.io_dtype == "bf16" else a


def _io(a: np.ndarray, io_dtype: str) -> np.ndarray:
    a = a.astype(np.float32)
    return f32_to_bf16_bits(a) if io_dtype == "bf16" else a


def make_problem(dims: Dims, parent: np.ndarray, seed: int,
                 dt_range=(1e-3, 1e-1), A_range=(1.0, 16.0),
                 x_scale: float = 1.0, h0_zero: bool = False, D_none: bool = False) -> Problem:
    """Values for a given batch of parent arrays ([B][T])."""
    rng = np.random.default_rng(seed)
    B, T, H, P, N, G = dims.batch, dims.n_nodes, dims.n_heads, dims.head_dim, dims.d_state, dims.n_groups
    parent = np.asarray(parent, dtype=np.int32).reshape(B, T)
    A = (-rng.uniform(A_range[0], A_range[1], size=H)).astype(np.float32)
    lo, hi = np.log(dt_range[0]), np.log(dt_range[1])
    dt = np.exp(rng.uniform(lo, hi, size=(B, T, H))).astype(np.float32)
    x = _io(x_scale * rng.standard_normal((B, T, H, P)), dims.io_dtype)
    Bm = _io(rng.standard_normal((B, T, G, N)), dims.io_dtype)
    Cm = _io(rng.standard_normal((B, T, G, N)), dims.io_dtype)
    D = (1.0 + 0.1 * rng.standard_normal(H)).astype(np.float32)
    if D_none:
        D = np.zeros(H, dtype=np.float32)
    h0 = rng.standard_normal((B, H, P, N)).astype(np.float32)
    if h0_zero:
        h0[:] = 0
    return Problem(dims, x, dt, A, Bm, Cm, D, h0, parent)


# ----------------------------------------------------------------------------
# Acceptance inputs: draft tokens with distinct siblings and verifier tokens.
# ----------------------------------------------------------------------------
def make_tokens(parent: np.ndarray, rng: np.random.Generator, vocab: int = VOCAB,
                dup_siblings: bool = False) -> np.ndarray:
    """tokens[i] for one tree; siblings distinct unless dup_siblings."""
    T = len(parent)
    tok = np.zeros(T, dtype=np.int32)
    if T == 0:
        return tok
    tok[0] = int(rng.integers(vocab))
    for kids in trees.children_lists(parent):
        if not kids:
            continue
        vals = rng.choice(vocab, size=len(kids), replace=False)
        if dup_siblings and len(kids) >= 2:
            vals[int(rng.integers(1, len(kids)))] = vals[0]
        tok[kids] = vals
    return tok


def make_verifier_tokens(parent: np.ndarray, tokens: np.ndarray, p_match: float,
                         rng: np.random.Generator, vocab: int = VOCAB) -> np.ndarray:
    """vtok[i] = the token of a random child of i with probability p_match,
    else a token carried by no child of i (SURVEY.md §8(d) acceptance inputs)."""
    T = len(parent)
    vt = np.zeros(T, dtype=np.int32)
    ch = trees.children_lists(parent)
    for i in range(T):
        kids = ch[i]
        kid_toks = set(int(tokens[c]) for c in kids)
        if kids and rng.random() < p_match:
            vt[i] = tokens[kids[int(rng.integers(len(kids)))]]
        else:
            while True:
                t = int(rng.integers(vocab))
                if t not in kid_toks:
                    break
            vt[i] = t
    return vt


def make_accept_inputs(parent_b: np.ndarray, seed: int, p_match: float = 0.9,
                       dup_siblings: bool = False):
    rng = np.random.default_rng(seed)
    B, T = parent_b.shape
    tokens = np.stack([make_tokens(parent_b[b], rng, dup_siblings=dup_siblings) for b in range(B)]) \
        if B else np.zeros((0, T), np.int32)
    vtok = np.stack([make_verifier_tokens(parent_b[b], tokens[b], p_match, rng) for b in range(B)]) \
        if B else np.zeros((0, T), np.int32)
    return tokens.astype(np.int32), vtok.astype(np.int32)


# ----------------------------------------------------------------------------
# Named configurations (BASELINE.json configs[0..4]).
# ----------------------------------------------------------------------------
def config_trees(cfg: str, seed: int) -> tuple[Dims, np.ndarray]:
    """Dims and [B][T] parent arrays for c1..c4 (c5 is a sweep, see sweep_cases)."""
    if cfg == "c1":  # toy: 1 head, P=N=4, binary depth 2 (7 nodes), fp32
        d = Dims(1, 7, 1, 4, 4, 1, "f32")
        return d, trees.heap_kary(7, 2)[None]
    if cfg == "c2":  # Mamba-2 130M layer, 32-node heap-binary tree
        d = Dims(1, 32, 24, 64, 128, 1, "bf16")
        return d, trees.heap_kary(32, 2)[None]
    if cfg == "c3":  # Mamba-2 2.7B layer, 64-node heap-binary tree
        d = Dims(1, 64, 80, 64, 128, 1, "bf16")
        return d, trees.heap_kary(64, 2)[None]
    if cfg == "c4":  # 2.7B layer, 16 distinct random recursive trees (branching <= 4)
        d = Dims(16, 64, 80, 64, 128, 1, "bf16")
        par = np.stack([trees.random_recursive(64, 4, np.random.default_rng(seed * 1000 + b))
                        for b in range(16)])
        return d, par
    raise ValueError(cfg)


def config_problem(cfg: str, io_dtype: str | None = None, batch: int | None = None) -> Problem:
    idx = {"c1": 0, "c2": 1, "c3": 2, "c4": 3}[cfg]
    seed = BASE_SEED + idx
    d, par = config_trees(cfg, seed)
    if io_dtype is not None:
        d.io_dtype = io_dtype
    if batch is not None and batch != d.batch:
        reps = -(-batch // d.batch)
        par = np.concatenate([par] * reps)[:batch]
        d.batch = batch
    return make_problem(d, par, seed)


def sweep_cases():
    """c5: T in {16..256} x heap k-ary k in {2,4,8}, plus chains and the
    paper's shapes (full binary 15/31/63, beam 1+M*N, static A-E)."""
    cases = []
    for T in (16, 32, 64, 128, 256):
        for k in (2, 4, 8):
            cases.append((f"heap{k}_T{T}", trees.heap_kary(T, k)))
        cases.append((f"chain_T{T}", trees.chain(T)))
    for L in (4, 5, 6):
        cases.append((f"fullbin_L{L}", trees.heap_kary(2 ** L - 1, 2)))
    for M in (2, 3, 4, 5):
        for N in (4, 8, 16):
            if 1 + M * N <= 256:
                cases.append((f"beam_M{M}N{N}", trees.beam(M, N, np.random.default_rng(M * 100 + N))))
    for name in "ABCDE":
        cases.append((f"static_{name}", trees.static_tree(name)))
    return cases
