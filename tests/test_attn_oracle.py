"""Pins for the tree-attention / KV-commit oracle (oracle/attn.py, reading R-attn) — CPU only.

Each pin checks the oracle against something other than itself:
  * textbook causal attention (a full score matrix with a lower-triangular -inf mask, written here
    independently) on a chain tree — a chain mask is the causal mask;
  * the same textbook attention on every unrolled root-to-leaf sequence: every node must equal
    causal attention over (prefix ++ its root path) ("avoiding repeated
    computation when naively unrolling the tree");
  * T = 1 with an empty cache: softmax over one position returns that value;
  * equal keys: uniform softmax, o = mean of the values (closed form);
  * brute force on small random trees: o[i] changes under a perturbation of node j's k/v iff j is an
    ancestor of i (or i itself) — the mask is exactly the ancestor relation;
  * commit-then-decode equals decode-from-scratch on the accepted text.
"""
import numpy as np
import pytest

from gen import trees
from gen.attn import AttnDims, attn_config, make_attn_problem
from oracle import attn as oattn


def causal_attention_textbook(qs, ks, vs, scale):
    """Standard causal multi-head attention with GQA over one sequence:
    qs [n][Hq][D], ks/vs [n][Hkv][D] -> [n][Hq][D];  A = softmax(scale*QK^T + M), M_ij = -inf for j > i."""
    n, Hq, D = qs.shape
    Hkv = ks.shape[1]
    kr = np.repeat(ks, Hq // Hkv, axis=1)
    vr = np.repeat(vs, Hq // Hkv, axis=1)
    S = scale * np.einsum("ihd,jhd->hij", qs, kr)
    M = np.triu(np.full((n, n), -np.inf), k=1)
    S = S + M[None]
    S = S - S.max(axis=2, keepdims=True)
    P = np.exp(S)
    P /= P.sum(axis=2, keepdims=True)
    return np.einsum("hij,jhd->ihd", P, vr)


def _f64(prob, name):
    return prob.as_f32(name).astype(np.float64)


def _run(prob):
    return oattn.tree_attn(_f64(prob, "q"), _f64(prob, "k_new"), _f64(prob, "v_new"), _f64(prob, "k_cache"),
                           _f64(prob, "v_cache"), prob.cache_len, prob.parent, prob.scale)


def _small(parent, seed, L, Hq=4, Hkv=2, D=8, S=32):
    parent = np.asarray(parent, np.int32)[None]
    return make_attn_problem(AttnDims(1, parent.shape[1], Hq, Hkv, D, S, "f32"), parent, seed, cache_len=[L])


@pytest.mark.parametrize("L", [0, 1, 5])
def test_chain_equals_causal_attention(L):
    T = 9
    prob = _small(trees.chain(T), 11 + L, L)
    o, st = _run(prob)
    assert st[0] == 0
    # the full sequence: prefix (no queries needed) then the chain tokens
    ks = np.concatenate([_f64(prob, "k_cache")[0, :L], _f64(prob, "k_new")[0]])
    vs = np.concatenate([_f64(prob, "v_cache")[0, :L], _f64(prob, "v_new")[0]])
    qs = np.concatenate([np.zeros((L,) + prob.q.shape[2:]), _f64(prob, "q")[0]])
    ref = causal_attention_textbook(qs, ks, vs, prob.scale)[L:]
    np.testing.assert_allclose(o[0], ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("kind,seed", [("random", 1), ("random", 2), ("heap", 3), ("star", 4)])
def test_every_node_equals_unrolled_leaf_sequence(kind, seed):
    T, L = 12, 6
    rng = np.random.default_rng(seed)
    par = {"random": lambda: trees.random_recursive(T, 3, rng), "heap": lambda: trees.heap_kary(T, 2),
           "star": lambda: trees.star(T)}[kind]()
    prob = _small(par, 100 + seed, L)
    o, st = _run(prob)
    assert st[0] == 0
    kids = trees.children_lists(par)
    leaves = [i for i in range(T) if not kids[i]]
    seen = np.zeros(T, bool)
    for leaf in leaves:
        path = [leaf]
        while par[path[-1]] >= 0:
            path.append(int(par[path[-1]]))
        path = path[::-1]
        ks = np.concatenate([_f64(prob, "k_cache")[0, :L], _f64(prob, "k_new")[0, path]])
        vs = np.concatenate([_f64(prob, "v_cache")[0, :L], _f64(prob, "v_new")[0, path]])
        qs = np.concatenate([np.zeros((L,) + prob.q.shape[2:]), _f64(prob, "q")[0, path]])
        ref = causal_attention_textbook(qs, ks, vs, prob.scale)[L:]
        np.testing.assert_allclose(o[0, path], ref, rtol=1e-12, atol=1e-12)
        seen[path] = True
    assert seen.all()


def test_single_node_empty_cache_returns_its_value():
    prob = _small([-1], 7, 0, Hq=6, Hkv=3)
    o, _ = _run(prob)
    v = _f64(prob, "v_new")[0, 0]
    np.testing.assert_allclose(o[0, 0], np.repeat(v, 2, axis=0), rtol=0, atol=1e-15)


def test_equal_keys_give_mean_of_values():
    par = trees.heap_kary(7, 2)
    prob = _small(par, 8, 3, Hq=2, Hkv=1)
    prob.k_cache[:] = 0.5
    prob.k_new[:] = 0.5
    o, _ = _run(prob)
    for i in range(7):
        path = [i]
        while par[path[-1]] >= 0:
            path.append(int(par[path[-1]]))
        vals = np.concatenate([_f64(prob, "v_cache")[0, :3, 0], _f64(prob, "v_new")[0, path, 0]])
        np.testing.assert_allclose(o[0, i, 0], vals.mean(axis=0), rtol=1e-13, atol=1e-13)


def test_bruteforce_dependence_is_exactly_the_ancestor_relation():
    rng = np.random.default_rng(5)
    for trial in range(6):
        T = 7
        par = trees.random_parent_array(T, rng)
        prob = _small(par, 200 + trial, 2)
        o0, _ = _run(prob)
        anc = [set() for _ in range(T)]
        for i in range(T):
            j = i
            while j >= 0:
                anc[i].add(j)
                j = int(par[j])
        for j in range(T):
            pk = make_attn_problem(prob.dims, prob.parent, 0, cache_len=prob.cache_len)
            for f in ("q", "k_new", "v_new", "k_cache", "v_cache"):
                setattr(pk, f, getattr(prob, f).copy())
            pk.k_new[0, j] += 1.0
            pk.v_new[0, j] -= 2.0
            o1, _ = _run(pk)
            for i in range(T):
                changed = not np.array_equal(o0[0, i], o1[0, i])
                assert changed == (j in anc[i]), (trial, i, j)


def test_invalid_tree_status():
    prob = _small([-1, 0, 2], 9, 1)
    o, st = _run(prob)
    assert st[0] == 2 and not o.any()
    prob = _small([0, 0, 1], 9, 1)
    assert _run(prob)[1][0] == 1


def test_commit_then_decode_equals_decode_from_scratch():
    """Verify a tree, commit the accepted path, then decode one more token (a 1-node tree):
    the result equals causal attention over the linear text prefix ++ accepted ++ new token."""
    rng = np.random.default_rng(12)
    T, L, S = 10, 4, 32
    par = trees.random_recursive(T, 3, rng)
    prob = _small(par, 300, L, S=S)
    # an accepted root-to-node path
    node = T - 1
    path = [node]
    while par[path[-1]] >= 0:
        path.append(int(par[path[-1]]))
    path = path[::-1]
    r = len(path)
    pp = np.full((1, T), -1, np.int32)
    pp[0, :r] = path
    kc, vc, cl, st = oattn.kv_commit(_f64(prob, "k_new"), _f64(prob, "v_new"), _f64(prob, "k_cache"),
                                     _f64(prob, "v_cache"), prob.cache_len, pp, [r], parent=prob.parent)
    assert st[0] == 0 and cl[0] == L + r
    nxt = _small([-1], 301, 0, S=S)
    o, _ = oattn.tree_attn(_f64(nxt, "q"), _f64(nxt, "k_new"), _f64(nxt, "v_new"), kc, vc, cl, nxt.parent,
                           nxt.scale)
    ks = np.concatenate([_f64(prob, "k_cache")[0, :L], _f64(prob, "k_new")[0, path], _f64(nxt, "k_new")[0]])
    vs = np.concatenate([_f64(prob, "v_cache")[0, :L], _f64(prob, "v_new")[0, path], _f64(nxt, "v_new")[0]])
    qs = np.zeros((len(ks),) + nxt.q.shape[2:])
    qs[-1] = _f64(nxt, "q")[0, 0]
    ref = causal_attention_textbook(qs, ks, vs, nxt.scale)[-1]
    np.testing.assert_allclose(o[0, 0], ref, rtol=1e-12, atol=1e-12)


def test_kv_commit_rejects_bad_paths_and_overflow():
    par = trees.heap_kary(7, 2)
    prob = _small(par, 13, 30, S=32)
    args = (_f64(prob, "k_new"), _f64(prob, "v_new"), _f64(prob, "k_cache"), _f64(prob, "v_cache"), prob.cache_len)
    kc0 = _f64(prob, "k_cache")
    for path, r, code in [([1, 3], 2, 3), ([0, 2, 3], 3, 3), ([0], 0, 3), ([0, 1, 3], 3, 5)]:
        pp = np.full((1, 7), -1, np.int32)
        pp[0, :len(path)] = path
        kc, vc, cl, st = oattn.kv_commit(*args, pp, [r], parent=prob.parent)
        assert st[0] == code and cl[0] == 30 and np.array_equal(kc, kc0)
    pp = np.full((1, 7), -1, np.int32)
    pp[0, :2] = [0, 2]
    kc, vc, cl, st = oattn.kv_commit(*args, pp, [2], parent=prob.parent)
    assert st[0] == 0 and cl[0] == 32
    np.testing.assert_array_equal(kc[0, 30], _f64(prob, "k_new")[0, 0])
    np.testing.assert_array_equal(vc[0, 31], _f64(prob, "v_new")[0, 2])


def test_named_configs_shapes():
    p = attn_config("toy", "f32")
    assert p.q.shape == (1, 7, 2, 4) and p.k_cache.shape == (1, 16, 1, 4)
    o, st = _run(p)
    assert st[0] == 0 and np.isfinite(o).all()
