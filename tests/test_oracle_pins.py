"""Pins for the CPU oracle (oracle/stree_oracle.c) — CPU only.

Each pin checks the oracle against something other than itself: values the
paper (or SPEC's worked examples) print, closed forms, the paper's matrix
form re-derived here in numpy, the textbook Mamba-2 chain
scan, invariants and brute force over all small trees.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle
from gen import inputs, trees

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------------------
# Independent helpers (NOT the oracle): the paper's matrix form.
# ---------------------------------------------------------------------------
def mask_by_closure(parent):
    """L row(i) = row(parent(i)) ∪ {i}  (SPEC.md:35 invariant)."""
    T = len(parent)
    L = np.zeros((T, T), dtype=np.int64)
    for i in range(T):
        if i > 0:
            L[i] = L[parent[i]]
        L[i, i] = 1
    return L


def matrix_form_scan(x, dt, A, Bm, Cm, D, h0, parent):
    """PAPER.md:86-102 for one tree, per head (Mamba-2 scalar-per-head decay):
    A_log[t] = dt_t*A_h;  A_tree = L @ A_log  (Eq. a_tree);
    y_i = C_i (exp(A_tree_i) h0)  +  sum_j L_ij exp(A_tree_i - A_tree_j) (C_i·B_j) dt_j x_j  + D x_i.
    x[T][H][P], dt[T][H], Bm/Cm[T][N] (G=1), h0[H][P][N]."""
    T, H, P = x.shape
    L = mask_by_closure(parent).astype(np.float64)
    y = np.zeros((T, H, P))
    G = Cm @ Bm.T                                   # C_i · B_j
    for h in range(H):
        alog = dt[:, h] * A[h]
        atree = L @ alog
        diff = atree[:, None] - atree[None, :]
        Mu = L * np.exp(np.where(L > 0, diff, 0.0)) * G * dt[None, :, h]
        Mx = np.exp(atree)[:, None] * (Cm @ h0[h].T)  # (M_x)_i x0 = C_i diag(e^{A_tree_i}) x0
        y[:, h, :] = Mx + Mu @ x[:, h, :] + D[h] * x[:, h, :]
    return y


def ssd_chain_textbook(x, dt, A, Bm, Cm, D, h0):
    """Mamba-2 SSD quadratic ('dual') form on a plain sequence with an initial
    state: segsum with -inf above the diagonal,
    Y = (exp(segsum) ∘ C Bᵀ)(dt X) + exp(cumsum) C h0ᵀ + D X;  final state
    h_T = exp(cs_T) h0 + sum_j exp(cs_T - cs_j) dt_j x_j B_jᵀ."""
    T, H, P = x.shape
    y = np.zeros((T, H, P))
    hT = np.zeros_like(h0)
    for h in range(H):
        a = dt[:, h] * A[h]
        cs = np.cumsum(a)
        seg = cs[:, None] - cs[None, :]
        seg = np.where(np.tril(np.ones((T, T), bool)), seg, -np.inf)
        Lm = np.exp(seg)
        y[:, h] = (Lm * (Cm @ Bm.T)) @ (dt[:, h, None] * x[:, h]) \
            + np.exp(cs)[:, None] * (Cm @ h0[h].T) + D[h] * x[:, h]
        w = np.exp(cs[-1] - cs) * dt[:, h]
        hT[h] = np.exp(cs[-1]) * h0[h] + np.einsum("t,tp,tn->pn", w, x[:, h], Bm)
    return y, hT


def rand_case(parent, H=2, P=3, N=4, seed=0, dt_hi=1e-1):
    rng = np.random.default_rng(seed)
    T = len(parent)
    x = rng.standard_normal((1, T, H, P))
    dt = np.exp(rng.uniform(np.log(1e-3), np.log(dt_hi), (1, T, H)))
    A = -rng.uniform(1, 16, H)
    Bm = rng.standard_normal((1, T, 1, N))
    Cm = rng.standard_normal((1, T, 1, N))
    D = 1 + 0.1 * rng.standard_normal(H)
    h0 = rng.standard_normal((1, H, P, N))
    return x, dt, A, Bm, Cm, D, h0, np.asarray(parent, np.int32)[None]


def group_of(h, H, G, convention="contiguous"):
    """Head -> group map.  Mamba-2 (the paper is silent): the heads of a group are
    contiguous, head h reads B/C of group h // (H/G).  'strided' (h % G) is the plausible mistake the
    grouped pins must reject."""
    return h // (H // G) if convention == "contiguous" else h % G


def matrix_form_scan_grouped(x, dt, A, Bm, Cm, D, h0, parent, convention="contiguous"):
    """matrix_form_scan with n_groups = G: Bm/Cm [T][G][N]; head h uses group group_of(h)."""
    T, H, P = x.shape
    G = Bm.shape[1]
    y = np.zeros((T, H, P))
    for h in range(H):
        g = group_of(h, H, G, convention)
        y[:, h:h + 1] = matrix_form_scan(x[:, h:h + 1], dt[:, h:h + 1], A[h:h + 1], Bm[:, g], Cm[:, g], D[h:h + 1],
                                         h0[h:h + 1], parent)
    return y


def commit_matrix_form_grouped(x, dt, A, Bm, h0, path, convention="contiguous"):
    """h_new = e^{Λ_k} h0 + Σ_{j∈path} e^{Λ_k-Λ_j} dt_j x_j B_jᵀ (the matrix form on the path),
    Bm [T][G][N], head h uses group group_of(h)."""
    T, H, P = x.shape
    G = Bm.shape[1]
    out = np.zeros_like(h0)
    for h in range(H):
        g = group_of(h, H, G, convention)
        lam = np.cumsum(dt[path, h] * A[h])
        w = np.exp(lam[-1] - lam) * dt[path, h]
        out[h] = np.exp(lam[-1]) * h0[h] + np.einsum("m,mp,mn->pn", w, x[path, h], Bm[path, g])
    return out


def rand_case_grouped(parent, H, G, P=3, N=4, seed=0):
    x, dt, A, _, _, D, h0, par = rand_case(parent, H=H, P=P, N=N, seed=seed)
    rng = np.random.default_rng(seed + 7)
    T = len(parent)
    return x, dt, A, rng.standard_normal((1, T, G, N)), rng.standard_normal((1, T, G, N)), D, h0, par


def relerr(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ---------------------------------------------------------------------------
# Mask
# ---------------------------------------------------------------------------
def _rows(mask_b, T):
    return ["".join("1" if (mask_b[i, j // 32] >> (j % 32)) & 1 else "0" for j in range(T))
            for i in range(T)]


def test_mask_spec_examples():
    for case in _gold("mask_examples.json")["cases"]:
        par = np.array(case["parent"], np.int32)[None]
        m, d, st = oracle.build_mask(par)
        assert st[0] == 0
        assert _rows(m[0], par.shape[1]) == case["rows"]
        assert list(d[0]) == [r.count("1") - 1 for r in case["rows"]]


def all_parent_arrays(T):
    return itertools.product(*[range(i) for i in range(1, T)])


def test_mask_bruteforce_all_trees_T_le_7():
    for T in range(1, 8):
        for tail in all_parent_arrays(T):
            par = np.array((-1,) + tail, np.int32)
            m, d, st = oracle.build_mask(par[None])
            L = mask_by_closure(par)
            got = np.array([[(m[0, i, j // 32] >> (j % 32)) & 1 for j in range(T)] for i in range(T)])
            assert st[0] == 0
            assert np.array_equal(got, L)
            assert np.array_equal(d[0], L.sum(1) - 1)


def test_mask_chain_is_causal_and_multiword():
    for T in (33, 64, 100, 256):
        m, d, st = oracle.build_mask(trees.chain(T)[None])
        got = np.array([[(m[0, i, j // 32] >> (j % 32)) & 1 for j in range(T)] for i in range(T)])
        assert np.array_equal(got, np.tril(np.ones((T, T), int)))
        assert np.array_equal(d[0], np.arange(T))


def test_mask_invalid_trees():
    bad = np.array([[0, 0, 0], [-1, 1, 0], [-1, 0, 5], [-1, -1, 0]], np.int32)
    _, _, st = oracle.build_mask(bad)
    assert list(st) == [1, 2, 2, 2]


def test_fig3_counts_and_table_shapes():
    g = _gold("fig3_counts.json")
    for c in g["cases"]:
        par = trees.heap_kary(2 ** c["levels"] - 1, 2)
        m, d, st = oracle.build_mask(par[None])
        has_child = np.zeros(len(par), bool)
        has_child[par[1:]] = True
        leaves = np.flatnonzero(~has_child)
        assert len(par) == c["packed_tokens"]
        assert len(leaves) == c["unrolled_states"]
        assert int((d[0][leaves] + 1).sum()) == c["unrolled_tokens"]
    for name, (width, depth, tok) in g["static_configs"].items():
        par = trees.static_tree(name)
        _, d, _ = oracle.build_mask(par[None])
        assert len(par) == tok and d[0].max() == depth
        assert max(np.bincount(d[0])) == width
    M, N, tok = g["beam"]
    par = trees.beam(M, N, np.random.default_rng(0))
    _, d, _ = oracle.build_mask(par[None])
    assert len(par) == tok and d[0].max() == N and max(np.bincount(d[0])[1:]) == M


# ---------------------------------------------------------------------------
# Scan
# ---------------------------------------------------------------------------
def test_matrix_form_helper_atree_spec_example():
    """parent=[-,0,0,1], a_log=ln .5 -> A_tree = [ln.5, 2ln.5, 2ln.5, 3ln.5]."""
    L = mask_by_closure([-1, 0, 0, 1])
    assert np.allclose(L @ np.full(4, math.log(0.5)), np.log(0.5) * np.array([1, 2, 2, 3]))


def test_scan_hand_example():
    g = _gold("hand_example.json")
    T = len(g["parent"])
    x = np.array(g["x"]).reshape(1, T, 1, 1)
    dt = np.array(g["dt"]).reshape(1, T, 1)
    Bm = np.array(g["B"]).reshape(1, T, 1, 1)
    Cm = np.array(g["C"]).reshape(1, T, 1, 1)
    h0 = np.full((1, 1, 1, 1), g["h0"])
    par = np.array(g["parent"], np.int32)[None]
    A = np.array(g["A"])
    for Dv, key in ((0.0, "y_D0"), (1.0, "y_D1")):
        y, st = oracle.tree_scan(x, dt, A, Bm, Cm, np.array([Dv]), h0, par)
        assert st[0] == 0
        np.testing.assert_allclose(y.ravel(), g[key], rtol=1e-14, atol=0)
    hn, st = oracle.commit(x, dt, A, Bm, h0, np.array([[0, 1, 3, -1]], np.int32), np.array([3], np.int32), par)
    assert st[0] == 0 and abs(hn.ravel()[0] - g["h_new"]) < 1e-14


def test_scan_vs_matrix_form_random_trees():
    """C1 (per-leaf recurrence) vs C2 over 200 random trees."""
    rng = np.random.default_rng(1)
    worst = 0.0
    for k in range(200):
        T = int(rng.integers(1, 64))
        par = trees.random_parent_array(T, rng) if k % 2 else trees.random_recursive(T, 3, rng)
        x, dt, A, Bm, Cm, D, h0, P = rand_case(par, H=2, P=int(rng.integers(1, 9)),
                                             N=int(rng.integers(1, 17)), seed=k)
        y, st = oracle.tree_scan(x, dt, A, Bm, Cm, D, h0, P)
        ref = matrix_form_scan(x[0], dt[0], A, Bm[0, :, 0], Cm[0, :, 0], D, h0[0], par)
        worst = max(worst, relerr(y[0], ref))
    assert worst < 1e-12, worst


def test_scan_bruteforce_all_trees_T_le_7():
    """Every topologically ordered tree with T <= 7 (873 trees; BASELINE north_star invariant 3)."""
    k = 0
    for T in range(1, 8):
        for tail in all_parent_arrays(T):
            par = np.array((-1,) + tail, np.int32)
            x, dt, A, Bm, Cm, D, h0, P = rand_case(par, H=2, P=3, N=4, seed=k, dt_hi=1.0)
            y, st = oracle.tree_scan(x, dt, A, Bm, Cm, D, h0, P)
            ref = matrix_form_scan(x[0], dt[0], A, Bm[0, :, 0], Cm[0, :, 0], D, h0[0], par)
            assert relerr(y[0], ref) < 1e-12, (par, relerr(y[0], ref))
            k += 1


@pytest.mark.parametrize("H,G", [(4, 2), (6, 3), (8, 4), (6, 2), (5, 5)])
def test_scan_grouped_heads_vs_matrix_form(H, G):
    """n_groups > 1 (Mamba-2: heads of a group contiguous): the oracle equals the matrix form
    with B/C of group h // (H/G) for every head, and differs from the strided h % G reading by far more
    than rounding — so a mis-grouped oracle fails this pin."""
    rng = np.random.default_rng(H * 10 + G)
    for k in range(12):
        T = int(rng.integers(2, 40))
        par = trees.random_recursive(T, 3, rng) if k % 2 else trees.random_parent_array(T, rng)
        x, dt, A, Bm, Cm, D, h0, P = rand_case_grouped(par, H, G, seed=50 + k)
        y, st = oracle.tree_scan(x, dt, A, Bm, Cm, D, h0, P, n_groups=G)
        assert st[0] == 0
        ref = matrix_form_scan_grouped(x[0], dt[0], A, Bm[0], Cm[0], D, h0[0], par)
        assert relerr(y[0], ref) < 1e-12
        if 1 < G < H:
            wrong = matrix_form_scan_grouped(x[0], dt[0], A, Bm[0], Cm[0], D, h0[0], par, convention="strided")
            assert relerr(y[0], wrong) > 1e-2


@pytest.mark.parametrize("H,G", [(4, 2), (6, 3), (8, 4)])
def test_grouped_equals_per_head_replication(H, G):
    """G groups == H groups (one per head, where every convention is the identity) with B/C replicated to
    the heads of each group (Mamba-2's repeat of B/C over the heads of a group): scan and commit."""
    rng = np.random.default_rng(G)
    par = trees.random_recursive(30, 3, rng)
    x, dt, A, Bm, Cm, D, h0, P = rand_case_grouped(par, H, G, seed=G)
    rep = lambda a: np.repeat(a, H // G, axis=2)   # noqa: E731  group g -> heads g*H/G .. (g+1)*H/G - 1
    y, _ = oracle.tree_scan(x, dt, A, Bm, Cm, D, h0, P, n_groups=G)
    yr, _ = oracle.tree_scan(x, dt, A, rep(Bm), rep(Cm), D, h0, P, n_groups=H)
    assert np.array_equal(y, yr)
    tok, vt = inputs.make_accept_inputs(P, seed=3, p_match=1.0)
    path, plen, _, _ = oracle.accept(tok, P, vt)
    hn, _ = oracle.commit(x, dt, A, Bm, h0, path, plen, P, n_groups=G)
    hr, _ = oracle.commit(x, dt, A, rep(Bm), h0, path, plen, P, n_groups=H)
    assert np.array_equal(hn, hr)


@pytest.mark.parametrize("H,G", [(4, 2), (6, 3), (6, 2)])
def test_commit_grouped_heads_vs_matrix_form(H, G):
    """oracle.commit with n_groups > 1 equals the path matrix form with B of group h // (H/G),
    and not the strided reading."""
    rng = np.random.default_rng(100 + H + G)
    for k in range(10):
        par = trees.random_recursive(int(rng.integers(2, 40)), 3, rng)
        x, dt, A, Bm, Cm, D, h0, P = rand_case_grouped(par, H, G, seed=70 + k)
        tok, vt = inputs.make_accept_inputs(P, seed=k, p_match=0.9)
        path, plen, _, _ = oracle.accept(tok, P, vt)
        hn, st = oracle.commit(x, dt, A, Bm, h0, path, plen, P, n_groups=G)
        pth = path[0, :plen[0]]
        ref = commit_matrix_form_grouped(x[0], dt[0], A, Bm[0], h0[0], pth)
        assert st[0] == 0 and relerr(hn[0], ref) < 1e-12
        wrong = commit_matrix_form_grouped(x[0], dt[0], A, Bm[0], h0[0], pth, convention="strided")
        assert relerr(hn[0], wrong) > 1e-3


def test_chain_grouped_equals_textbook_mamba2_scan():
    """PAPER.md:104 at n_groups = 2: a chain equals the textbook SSD form per head with its group's B/C."""
    H, G, T = 4, 2, 24
    par = trees.chain(T)
    x, dt, A, Bm, Cm, D, h0, P = rand_case_grouped(par, H, G, P=5, N=6, seed=9)
    y, _ = oracle.tree_scan(x, dt, A, Bm, Cm, D, h0, P, n_groups=G)
    for h in range(H):
        g = h // (H // G)
        yr, hT = ssd_chain_textbook(x[0][:, h:h + 1], dt[0][:, h:h + 1], A[h:h + 1], Bm[0, :, g], Cm[0, :, g],
                                    D[h:h + 1], h0[0][h:h + 1])
        assert relerr(y[0][:, h:h + 1], yr) < 1e-12


def test_chain_equals_textbook_mamba2_scan():
    """causal L -> Mamba-2 with a non-zero initial state."""
    for T in (1, 2, 7, 33, 128):
        par = trees.chain(T)
        x, dt, A, Bm, Cm, D, h0, P = rand_case(par, H=3, P=5, N=6, seed=T)
        y, _ = oracle.tree_scan(x, dt, A, Bm, Cm, D, h0, P)
        yr, hT = ssd_chain_textbook(x[0], dt[0], A, Bm[0, :, 0], Cm[0, :, 0], D, h0[0])
        assert relerr(y[0], yr) < 1e-12
        path = np.arange(T, dtype=np.int32)[None]
        hn, st = oracle.commit(x, dt, A, Bm, h0, path, np.array([T], np.int32), P)
        assert st[0] == 0 and relerr(hn[0], hT) < 1e-12


def test_unrolled_paths_reproduce_nodes_bitwise():
    """Each root-to-leaf path scanned as its own chain reproduces the packed
    tree's outputs bit-identically (BASELINE north_star invariant 1)."""
    rng = np.random.default_rng(7)
    for k in range(20):
        par = trees.random_recursive(40, 3, rng)
        x, dt, A, Bm, Cm, D, h0, P = rand_case(par, H=2, P=4, N=5, seed=100 + k)
        y, _ = oracle.tree_scan(x, dt, A, Bm, Cm, D, h0, P)
        has_child = np.zeros(len(par), bool)
        has_child[par[1:]] = True
        for leaf in np.flatnonzero(~has_child):
            path = [int(leaf)]
            while par[path[-1]] >= 0:
                path.append(int(par[path[-1]]))
            path = path[::-1]
            sub = lambda a: a[:, path]  # noqa: E731
            yc, _ = oracle.tree_scan(sub(x), sub(dt), A, sub(Bm), sub(Cm), D, h0,
                                     trees.chain(len(path))[None])
            assert np.array_equal(yc[0], y[0, path])


def test_scan_special_cases():
    rng = np.random.default_rng(3)
    # T = 1: y = e^{dt A} C h0ᵀ + dt (C·B) x + D x   (SPEC.md:150 with h0)
    x, dt, A, Bm, Cm, D, h0, P = rand_case([-1], H=2, P=3, N=4, seed=5)
    y, _ = oracle.tree_scan(x, dt, A, Bm, Cm, D, h0, P)
    for h in range(2):
        exp = np.exp(dt[0, 0, h] * A[h]) * (h0[0, h] @ Cm[0, 0, 0]) \
            + dt[0, 0, h] * (Cm[0, 0, 0] @ Bm[0, 0, 0]) * x[0, 0, h] + D[h] * x[0, 0, h]
        np.testing.assert_allclose(y[0, 0, h], exp, rtol=1e-13)
    par = trees.random_recursive(20, 3, rng)
    x, dt, A, Bm, Cm, D, h0, P = rand_case(par, H=2, P=3, N=4, seed=6)
    # dt = 0: no decay, no input -> y_i = C_i h0ᵀ + D x_i
    y, _ = oracle.tree_scan(x, 0 * dt, A, Bm, Cm, D, h0, P)
    exp = np.einsum("tn,hpn->thp", Cm[0, :, 0], h0[0]) + D[None, :, None] * x[0]
    np.testing.assert_allclose(y[0], exp, rtol=1e-13, atol=1e-13)
    # linearity in (x, h0) (D = 0)
    Dz = np.zeros_like(D)
    y1, _ = oracle.tree_scan(x, dt, A, Bm, Cm, Dz, h0, P)
    y2, _ = oracle.tree_scan(2 * x, dt, A, Bm, Cm, Dz, 0 * h0, P)
    y3, _ = oracle.tree_scan(0 * x, dt, A, Bm, Cm, Dz, 3 * h0, P)
    np.testing.assert_allclose(y1, y2 / 2 + y3 / 3, rtol=1e-11, atol=1e-12)
    # A = 0: no decay -> y_i = C_i (h0 + sum_{j in path} dt_j x_j B_jᵀ) + D x_i
    y, _ = oracle.tree_scan(x, dt, 0 * A, Bm, Cm, D, h0, P)
    L = mask_by_closure(par)
    for i in range(len(par)):
        js = np.flatnonzero(L[i])
        S = h0[0] + np.einsum("j,jhp,jn->hpn", np.ones(len(js)), dt[0, js, :, None] * x[0, js], Bm[0, js, 0])
        np.testing.assert_allclose(y[0, i], S @ Cm[0, i, 0] + D[:, None] * x[0, i], rtol=1e-12, atol=1e-12)


def test_subtree_locality_bitwise():
    """perturbing x_j for j ∉ path(i) leaves y_i bit-identical."""
    rng = np.random.default_rng(11)
    par = trees.random_recursive(48, 4, rng)
    x, dt, A, Bm, Cm, D, h0, P = rand_case(par, seed=12)
    y, _ = oracle.tree_scan(x, dt, A, Bm, Cm, D, h0, P)
    L = mask_by_closure(par)
    j = 17
    x2 = x.copy()
    x2[0, j] += 1.0
    y2, _ = oracle.tree_scan(x2, dt, A, Bm, Cm, D, h0, P)
    for i in range(len(par)):
        if L[i, j] == 0:
            assert np.array_equal(y[0, i], y2[0, i])
        else:
            assert not np.array_equal(y[0, i], y2[0, i])


def test_scan_invalid_tree_zero_filled():
    x, dt, A, Bm, Cm, D, h0, P = rand_case([-1, 0, 1], seed=1)
    bad = np.array([[-1, 2, 0]], np.int32)
    y, st = oracle.tree_scan(x, dt, A, Bm, Cm, D, h0, bad)
    assert st[0] == 2 and not y.any()


# ---------------------------------------------------------------------------
# Accept
# ---------------------------------------------------------------------------
def naive_walk(tokens, parent, vtok):
    """Independent restatement of PAPER.md:309 (children scanned by a dict)."""
    kids = {}
    for c in range(1, len(parent)):
        kids.setdefault(int(parent[c]), []).append(c)
    path, cur = [0], 0
    while True:
        m = [c for c in kids.get(cur, []) if tokens[c] == vtok[cur]]
        if not m:
            return path, int(vtok[cur])
        cur = min(m)
        path.append(cur)


def test_accept_spec_examples_and_hand_example():
    for c in _gold("accept_examples.json")["cases"]:
        path, plen, bonus, st = oracle.accept(np.array([c["tokens"]]), np.array([c["parent"]]),
                                              np.array([c["vtok"]]))
        assert st[0] == 0 and plen[0] == c["len"] and bonus[0] == c["bonus"]
        assert list(path[0][: plen[0]]) == c["path"] and (path[0][plen[0]:] == -1).all()
    g = _gold("hand_example.json")
    path, plen, bonus, st = oracle.accept(np.array([g["tokens"]]), np.array([g["parent"]]), np.array([g["vtok"]]))
    assert list(path[0][: plen[0]]) == g["accept_path"] and plen[0] == g["accept_len"] \
        and bonus[0] == g["accept_bonus"]


def test_accept_chain_full_and_none():
    T = 10
    par = trees.chain(T)
    tok = np.arange(100, 100 + T, dtype=np.int32)
    vt = np.roll(tok, -1)
    vt[-1] = 5
    path, plen, bonus, _ = oracle.accept(tok[None], par[None], vt[None])
    assert plen[0] == T and bonus[0] == 5 and list(path[0]) == list(range(T))
    vt2 = np.full(T, 1, np.int32)
    path, plen, bonus, _ = oracle.accept(tok[None], par[None], vt2[None])
    assert plen[0] == 1 and bonus[0] == 1


def test_accept_bruteforce_with_duplicate_siblings():
    rng = np.random.default_rng(5)
    for k in range(300):
        T = int(rng.integers(1, 80))
        par = trees.random_recursive(T, 4, rng)
        p_match = [0.0, 0.5, 0.9, 1.0][k % 4]
        tok = inputs.make_tokens(par, rng, vocab=50, dup_siblings=(k % 3 == 0))
        vt = inputs.make_verifier_tokens(par, tok, p_match, rng, vocab=50)
        path, plen, bonus, st = oracle.accept(tok[None], par[None], vt[None])
        ep, eb = naive_walk(tok, par, vt)
        assert list(path[0][: plen[0]]) == ep and bonus[0] == eb
        _, d, _ = oracle.build_mask(par[None])
        assert 1 <= plen[0] <= d[0].max() + 1
        for a, b in zip(ep[:-1], ep[1:]):
            assert par[b] == a


# ---------------------------------------------------------------------------
# Commit (activation replay)
# ---------------------------------------------------------------------------
def test_commit_root_only_closed_form():
    x, dt, A, Bm, Cm, D, h0, P = rand_case([-1, 0, 0], H=2, P=3, N=4, seed=9)
    hn, st = oracle.commit(x, dt, A, Bm, h0, np.array([[0, -1, -1]], np.int32), np.array([1], np.int32), P)
    for h in range(2):
        exp = np.exp(dt[0, 0, h] * A[h]) * h0[0, h] + dt[0, 0, h] * np.outer(x[0, 0, h], Bm[0, 0, 0])
        np.testing.assert_allclose(hn[0, h], exp, rtol=1e-14)


def test_commit_invalid_paths_keep_h0():
    x, dt, A, Bm, Cm, D, h0, P = rand_case([-1, 0, 0, 1], seed=2)
    bad = [([1, 3, -1, -1], 2), ([0, 2, 3, -1], 3), ([0, 1, 3, -1], 0), ([0, 1, 1, -1], 3)]
    for p, r in bad:
        hn, st = oracle.commit(x, dt, A, Bm, h0, np.array([p], np.int32), np.array([r], np.int32), P)
        assert st[0] == 3 and np.array_equal(hn, h0)


def test_graft_invariant():
    """Losslessness across iterations (Alg. 1): scanning
    tree2 from h0 = commit(tree1, path to k) equals scanning tree1 with tree2
    grafted below k (tree2's root is the bonus token, a new child of k)."""
    rng = np.random.default_rng(21)
    for k in range(10):
        T1, T2 = 20, 12
        p1 = trees.random_recursive(T1, 3, rng)
        p2 = trees.random_recursive(T2, 3, rng)
        kk = int(rng.integers(T1))
        path = [kk]
        while p1[path[-1]] >= 0:
            path.append(int(p1[path[-1]]))
        path = path[::-1]
        pg = np.concatenate([p1, [kk], p2[1:] + T1]).astype(np.int32)
        x, dt, A, Bm, Cm, D, h0, Pg = rand_case(pg, H=2, P=3, N=4, seed=200 + k)
        yg, _ = oracle.tree_scan(x, dt, A, Bm, Cm, D, h0, Pg)
        pa = np.full((1, T1), -1, np.int32)
        pa[0, : len(path)] = path
        s1 = lambda a: a[:, :T1]  # noqa: E731
        s2 = lambda a: a[:, T1:]  # noqa: E731
        hk, st = oracle.commit(s1(x), s1(dt), A, s1(Bm), h0, pa, np.array([len(path)], np.int32), p1[None])
        assert st[0] == 0
        y2, _ = oracle.tree_scan(s2(x), s2(dt), A, s2(Bm), s2(Cm), D, hk, p2[None])
        np.testing.assert_allclose(y2[0], yg[0, T1:], rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------------------
# Tree-causal depthwise conv1d (reading R-conv)
# Pins: the chain reduces to the library causal conv1d (torch CPU, grouped conv,
# state as left context); every node equals the library conv run on its own
# root-to-node path; W = 1 is pointwise; the commit is list slicing.
# ---------------------------------------------------------------------------
def _torch_causal_conv(seq, weight, bias, act):
    """Library reference: depthwise causal conv1d over seq [L][C] (no padding: seq already holds the
    left context), torch.nn.functional.conv1d on CPU in float64; returns [L - W + 1][C]."""
    import torch
    C, W = weight.shape
    x = torch.from_numpy(np.ascontiguousarray(seq.T[None]))                 # [1][C][L]
    w = torch.from_numpy(np.ascontiguousarray(weight[:, None, :]))          # [C][1][W]
    b = None if bias is None else torch.from_numpy(bias)
    z = torch.nn.functional.conv1d(x, w, b, groups=C)[0].T                  # [L-W+1][C]
    if act:
        z = torch.nn.functional.silu(z)
    return z.numpy()


def _conv_inputs(B, T, C, W, seed):
    rng = np.random.default_rng(seed)
    u = rng.standard_normal((B, T, C))
    weight = rng.standard_normal((C, W)) * 0.5
    bias = rng.standard_normal(C) * 0.1
    state = rng.standard_normal((B, W - 1, C))
    return u, weight, bias, state


@pytest.mark.parametrize("W,act", [(4, True), (4, False), (2, True), (3, True)])
def test_conv_chain_equals_library_causal_conv(W, act):
    B, T, C = 2, 23, 5
    u, weight, bias, state = _conv_inputs(B, T, C, W, seed=W)
    par = np.stack([trees.chain(T)] * B)
    out, st = oracle.tree_conv(u, weight, bias, state, par, act=act)
    assert not st.any()
    for b in range(B):
        ref = _torch_causal_conv(np.concatenate([state[b], u[b]]), weight, bias, act)
        np.testing.assert_allclose(out[b], ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("kind", ["random", "heap2", "star"])
def test_conv_every_node_is_the_conv_of_its_path(kind):
    B, T, C, W = 3, 31, 4, 4
    rng = np.random.default_rng(7)
    mk = {"random": lambda: trees.random_recursive(T, 3, rng), "heap2": lambda: trees.heap_kary(T, 2),
          "star": lambda: np.array([-1] + [0] * (T - 1), np.int32)}[kind]
    par = np.stack([mk() for _ in range(B)])
    u, weight, bias, state = _conv_inputs(B, T, C, W, seed=11)
    out, st = oracle.tree_conv(u, weight, bias, state, par)
    assert not st.any()
    for b in range(B):
        for i in range(T):
            path = []
            v = i
            while v >= 0:
                path.append(v)
                v = int(par[b, v])
            seq = np.concatenate([state[b], u[b, path[::-1]]])
            ref = _torch_causal_conv(seq, weight, bias, True)[-1]
            np.testing.assert_allclose(out[b, i], ref, rtol=1e-12, atol=1e-12)


def test_conv_special_cases():
    B, T, C = 2, 9, 3
    u, weight, bias, state = _conv_inputs(B, T, C, 1, seed=3)
    par = np.stack([trees.random_recursive(T, 3, np.random.default_rng(1)) for _ in range(B)])
    out, _ = oracle.tree_conv(u, weight, bias, None, par, act=False)
    np.testing.assert_allclose(out, u * weight[None, None, :, 0] + bias, rtol=1e-14)   # W = 1: pointwise
    u, weight, bias, state = _conv_inputs(B, T, C, 4, seed=4)
    o1, _ = oracle.tree_conv(u, weight, None, None, par, act=False)
    o2, _ = oracle.tree_conv(u, weight, None, np.zeros_like(state), par, act=False)
    assert np.array_equal(o1, o2)                                                       # NULL state = zeros
    bad = par.copy()
    bad[1, 4] = 6
    o3, st = oracle.tree_conv(u, weight, bias, state, bad)
    assert list(st) == [0, 2] and not o3[1].any()


def test_conv_commit_is_slicing_of_state_and_path():
    B, T, C, W = 3, 12, 4, 4
    u, _, _, state = _conv_inputs(B, T, C, W, seed=5)
    par = np.stack([trees.chain(T)] * B)
    path = np.full((B, T), -1, np.int32)
    plen = np.array([12, 2, 1], np.int32)
    for b in range(B):
        path[b, : plen[b]] = np.arange(plen[b])
    new, st = oracle.conv_commit(u, state, path, plen, W, parent=par)
    assert not st.any()
    for b in range(B):
        full = np.concatenate([state[b], u[b, path[b, : plen[b]]]])
        np.testing.assert_array_equal(new[b], full[-(W - 1):])
    path2 = path.copy()
    path2[1, 1] = 3                                    # not parent-linked
    new2, st2 = oracle.conv_commit(u, state, path2, plen, W, parent=par)
    assert list(st2) == [0, 3, 0]
    np.testing.assert_array_equal(new2[1], state[1])


def test_conv_commit_then_conv_equals_grafted_tree():
    """Losslessness of the conv state across iterations (the conv analogue of Alg. 1): the conv of a
    second tree from the committed state equals the conv of that tree grafted under the last accepted
    node of the first tree, from the original state."""
    C, W = 3, 4
    rng = np.random.default_rng(9)
    T1, T2 = 10, 8
    p1 = trees.random_recursive(T1, 3, rng)
    p2 = trees.random_recursive(T2, 3, rng)
    u1 = rng.standard_normal((1, T1, C))
    u2 = rng.standard_normal((1, T2, C))
    weight = rng.standard_normal((C, W))
    bias = rng.standard_normal(C)
    state = rng.standard_normal((1, W - 1, C))
    k = T1 - 1
    path = []
    v = k
    while v >= 0:
        path.append(v)
        v = int(p1[v])
    path = path[::-1]
    pa = np.full((1, T1), -1, np.int32)
    pa[0, : len(path)] = path
    s1, _ = oracle.conv_commit(u1, state, pa, np.array([len(path)], np.int32), W, parent=p1[None])
    o2, _ = oracle.tree_conv(u2, weight, bias, s1, p2[None])
    pg = np.concatenate([p1, np.where(p2 < 0, k, p2 + T1)]).astype(np.int32)
    og, _ = oracle.tree_conv(np.concatenate([u1, u2], 1), weight, bias, state, pg[None])
    np.testing.assert_allclose(o2[0], og[0, T1:], rtol=1e-12, atol=1e-12)


# ---- scan options (include/stree.h stree_scan_opts; SURVEY §8(f) unranked variants) ----
def test_opts_softplus_inverse_and_bias_reduce_to_plain_scan():
    """softplus(log(e^dt - 1)) = dt and (dt - b) + b = dt: the options fed the pre-images of dt give the plain
    scan and commit (pins the transform's direction, its argument order and that it reaches every dt)."""
    rng = np.random.default_rng(3)
    x, dt, A, Bm, Cm, D, h0, par = rand_case(trees.random_recursive(9, 3, rng), H=3, P=2, N=3, seed=5)
    bias = rng.uniform(-2, 2, 3)
    raw = np.log(np.expm1(dt)) - bias[None, None, :]
    y0, _ = oracle.tree_scan(x, dt, A, Bm, Cm, D, h0, par)
    y1, _ = oracle.tree_scan_ex(x, raw, A, Bm, Cm, D, h0, par, dt_bias=bias, dt_softplus=True)
    y2, _ = oracle.tree_scan_ex(x, dt - bias[None, None, :], A, Bm, Cm, D, h0, par, dt_bias=bias)
    assert relerr(y1, y0) < 1e-12 and relerr(y2, y0) < 1e-12
    path = np.array([[0, 1, -1, -1, -1, -1, -1, -1, -1]], np.int32) if par[0, 1] == 0 else None
    if path is not None:
        pl = np.array([2], np.int32)
        c0, _ = oracle.commit(x, dt, A, Bm, h0, path, pl, par)
        c1, _ = oracle.commit_ex(x, raw, A, Bm, h0, path, pl, par, dt_bias=bias, dt_softplus=True)
        assert relerr(c1, c0) < 1e-12


def test_opts_single_node_closed_form():
    """T = 1 from h0 = 0: y = softplus(dt + b)·x·(B·C) + D[h][p]·x, per head and channel — the recurrence
    and the options written out by hand for one step (PAPER.md:44-45 per R1)."""
    H, P, N = 2, 3, 4
    rng = np.random.default_rng(11)
    x = rng.standard_normal((1, 1, H, P))
    raw = rng.uniform(-3, 3, (1, 1, H))
    bias = rng.uniform(-1, 1, H)
    A = -rng.uniform(1, 5, H)
    Bm, Cm = rng.standard_normal((1, 1, 1, N)), rng.standard_normal((1, 1, 1, N))
    Dhp = rng.standard_normal((H, P))
    y, st = oracle.tree_scan_ex(x, raw, A, Bm, Cm, Dhp, None, np.array([[-1]], np.int32), dt_bias=bias,
                                dt_softplus=True, d_per_channel=True)
    bc = float(sum(Bm[0, 0, 0, n] * Cm[0, 0, 0, n] for n in range(N)))
    for h in range(H):
        sp = math.log1p(math.exp(raw[0, 0, h] + bias[h]))
        for p in range(P):
            want = sp * x[0, 0, h, p] * bc + Dhp[h, p] * x[0, 0, h, p]
            assert abs(y[0, 0, h, p] - want) <= 1e-12 * max(1.0, abs(want))
    assert not st.any()


def test_opts_per_channel_d_reduces_and_is_linear():
    """D[h][p] = D_h for every p equals the per-head D; y(D1 + D2) - y(D1) = D2 ∘ x (the skip term is
    additive and per channel); invalid trees stay zero."""
    rng = np.random.default_rng(7)
    par = np.stack([trees.random_recursive(11, 3, rng), trees.chain(11)]).astype(np.int32)
    cases = [rand_case(par[k], H=2, P=3, N=2, seed=8 + k) for k in range(2)]
    x, dt, Bm, Cm, h0 = (np.concatenate([c[i] for c in cases]) for i in (0, 1, 3, 4, 6))
    A, D = cases[0][2], cases[0][5]
    Dhp = np.repeat(D[:, None], 3, axis=1)
    ya, _ = oracle.tree_scan(x, dt, A, Bm, Cm, D, h0, par)
    yb, _ = oracle.tree_scan_ex(x, dt, A, Bm, Cm, Dhp, h0, par, d_per_channel=True)
    assert relerr(yb, ya) < 1e-12
    D2 = rng.standard_normal((2, 3))
    yc, _ = oracle.tree_scan_ex(x, dt, A, Bm, Cm, Dhp + D2, h0, par, d_per_channel=True)
    assert np.abs((yc - yb) - D2[None, None] * x).max() < 1e-12
    bad = par.copy()
    bad[1, 4] = 7
    yz, st = oracle.tree_scan_ex(x, dt, A, Bm, Cm, Dhp, h0, bad, d_per_channel=True)
    assert st[1] == 2 and not yz[1].any()


def test_variable_T_by_padding_leaves():
    """Variable T per tree: a tree of n < T nodes is padded with leaves under the root; every
    real node's output is unchanged (outputs depend on ancestors only), and a padding leaf
    whose token never matches is never accepted, so the committed state is unchanged too."""
    rng = np.random.default_rng(21)
    n, T = 9, 16
    p9 = trees.random_recursive(n, 3, rng)
    x, dt, A, Bm, Cm, D, h0, p16 = rand_case(np.concatenate([p9, np.zeros(T - n, np.int32)]), H=2, P=2, N=3,
                                             seed=4)
    y16, _ = oracle.tree_scan(x, dt, A, Bm, Cm, D, h0, p16)
    y9, _ = oracle.tree_scan(x[:, :n], dt[:, :n], A, Bm[:, :n], Cm[:, :n], D, h0, p9[None])
    assert np.array_equal(y16[:, :n], y9)
    tok = np.concatenate([rng.integers(0, 50, n), -np.ones(T - n, np.int64)]).astype(np.int32)[None]
    vt = tok.copy()
    vt[0, :n] = rng.integers(0, 50, n)
    path16, pl16, b16, _ = oracle.accept(tok, p16, vt)
    path9, pl9, b9, _ = oracle.accept(tok[:, :n], p9[None], vt[:, :n])
    assert pl16[0] == pl9[0] and b16[0] == b9[0] and np.array_equal(path16[0, :pl16[0]], path9[0, :pl9[0]])
