"""Seeded synthetic inputs for tree attention + KV commit.

Holds none of the method's arithmetic: random values, bf16 bit patterns and shapes only.
Shapes follow the attention layers of the hybrid MambaInLlama-8B target (
Llama-3.1-8B attention: 32 query heads, 8 KV heads, head dim 128).  Values: q, k, v ~ N(0, 1)
cast to the io dtype (scores s = <q,k>/sqrt(D) ~ N(0, 1)); committed prefix lengths ragged,
cache_len ~ U[lo, hi] per tree.  Seeds: BASE_SEED + 100 + case index.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from . import trees
from .inputs import BASE_SEED, bf16_bits_to_f32, f32_to_bf16_bits


@dataclasses.dataclass
class AttnDims:
    batch: int
    n_nodes: int
    n_q_heads: int = 32
    n_kv_heads: int = 8
    head_dim: int = 128
    cache_cap: int = 2048
    io_dtype: str = "bf16"


@dataclasses.dataclass
class AttnProblem:
    """q[B][T][Hq][D], k_new/v_new[B][T][Hkv][D], k_cache/v_cache[B][S][Hkv][D] (io: float32, or
    uint16 bf16 bits), cache_len[B] i32, parent[B][T] i32, scale (1/sqrt(D))."""
    dims: AttnDims
    q: np.ndarray
    k_new: np.ndarray
    v_new: np.ndarray
    k_cache: np.ndarray
    v_cache: np.ndarray
    cache_len: np.ndarray
    parent: np.ndarray
    scale: float

    def as_f32(self, name: str) -> np.ndarray:
        a = getattr(self, name)
        return bf16_bits_to_f32(a) if self.dims.io_dtype == "bf16" else a


def _io(a, io_dtype):
    a = np.asarray(a, np.float32)
    return f32_to_bf16_bits(a) if io_dtype == "bf16" else a


def make_attn_problem(dims: AttnDims, parent: np.ndarray, seed: int, cache_len=None,
                      len_range=(768, 1280), q_scale: float = 1.0) -> AttnProblem:
    rng = np.random.default_rng(seed)
    B, T, Hq, Hkv, D, S = dims.batch, dims.n_nodes, dims.n_q_heads, dims.n_kv_heads, dims.head_dim, dims.cache_cap
    parent = np.asarray(parent, np.int32).reshape(B, T)
    if cache_len is None:
        cache_len = rng.integers(len_range[0], len_range[1] + 1, size=B)
    cache_len = np.minimum(np.asarray(cache_len, np.int64).reshape(B), S).astype(np.int32)
    q = _io(q_scale * rng.standard_normal((B, T, Hq, D)), dims.io_dtype)
    k_new = _io(rng.standard_normal((B, T, Hkv, D)), dims.io_dtype)
    v_new = _io(rng.standard_normal((B, T, Hkv, D)), dims.io_dtype)
    k_cache = np.zeros((B, S, Hkv, D), np.float32)
    v_cache = np.zeros((B, S, Hkv, D), np.float32)
    for b in range(B):
        n = int(cache_len[b])
        k_cache[b, :n] = rng.standard_normal((n, Hkv, D))
        v_cache[b, :n] = rng.standard_normal((n, Hkv, D))
    return AttnProblem(dims, q, k_new, v_new, _io(k_cache, dims.io_dtype), _io(v_cache, dims.io_dtype),
                       cache_len, parent, float(1.0 / np.sqrt(D)))


def attn_config(name: str, io_dtype: str = "bf16", batch: int | None = None) -> AttnProblem:
    """Named cases.  'hyb8b': the bench workload — 16 random recursive 64-node trees (branching
    <= 4, the c4 trees), MambaInLlama-8B attention shape, prefixes of 768..1280 committed tokens."""
    if name == "hyb8b":
        B = batch or 16
        seed = BASE_SEED + 100
        par = np.stack([trees.random_recursive(64, 4, np.random.default_rng(seed * 1000 + b)) for b in range(B)])
        return make_attn_problem(AttnDims(B, 64, io_dtype=io_dtype), par, seed)
    if name == "toy":
        par = trees.heap_kary(7, 2)[None]
        return make_attn_problem(AttnDims(1, 7, 2, 1, 4, 16, io_dtype), par, BASE_SEED + 101, len_range=(3, 5))
    raise KeyError(name)
