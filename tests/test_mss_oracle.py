"""Pins for the MSS verification oracle (oracle/mss.py, reading R-mss) — CPU only.

  * SPEC.md:370  q = p everywhere -> every drafted token is accepted (u < 1 = p/q);
  * SPEC.md:371  single child t with p(t) = 0.2, q(t) = 0.8 -> acceptance rate 0.25 (Monte Carlo);
  * SPEC.md:372  V = {a, b}, p = (0.5, 0.5), q = (1, 0), single child a rejected -> residual (0, 1),
                 bonus = b always;
  * losslessness of multi-step speculative sampling (SpecInfer, cited at PAPER.md:355): with the
    children drawn i.i.d. from q, the first emitted token (the first accepted child's token, else the
    bonus) is distributed exactly as p_target[root] — a dropped residual, a wrong normalisation or the
    wrong q would all skew the histogram;
  * the bonus at a leaf is the inverse-CDF sample of the fresh target distribution (closed form).
"""
import numpy as np

from gen import trees
from gen.mss import make_mss_problem, mss_config
from oracle import mss


def _star_problem(p_root, q_root, child_tokens, vocab):
    T = 1 + len(child_tokens)
    par = np.array([-1] + [0] * len(child_tokens), np.int32)
    p = np.zeros((T, vocab)); q = np.zeros((T, vocab))
    p[0], q[0] = p_root, q_root
    p[1:] = 1.0 / vocab; q[1:] = 1.0 / vocab
    tok = np.array([0] + list(child_tokens), np.int32)
    return tok, par, p, q


def test_q_equals_p_accepts_whole_chain():
    prob = make_mss_problem(trees.chain(12)[None], 64, 3, same=True)
    path, plen, bonus, st, _ = mss.verify_mss(prob.tokens, prob.parent, prob.p_target, prob.q_draft,
                                               prob.u_accept, prob.u_bonus)
    assert st[0] == 0 and plen[0] == 12 and list(path[0]) == list(range(12))


def test_single_child_acceptance_rate():
    rng = np.random.default_rng(0)
    V = 4
    p_root = np.array([0.2, 0.3, 0.3, 0.2]); q_root = np.array([0.8, 0.1, 0.05, 0.05])
    tok, par, p, q = _star_problem(p_root, q_root, [0], V)
    n, acc = 10000, 0
    for _ in range(n):
        pth, _, _ = mss.verify_mss_tree(tok, par, p, q, rng.random(2), rng.random())
        acc += len(pth) > 1
    assert abs(acc / n - 0.25) < 0.02


def test_residual_by_hand():
    tok, par, p, q = _star_problem(np.array([0.5, 0.5]), np.array([1.0, 0.0]), [0], 2)
    rng = np.random.default_rng(1)
    for _ in range(200):
        u = rng.random(2)
        u[1] = 0.5 + 0.5 * u[1]          # reject: u * 1 >= 0.5
        pth, v, _ = mss.verify_mss_tree(tok, par, p, q, u, rng.random())
        assert pth == [0] and v == 1


def test_leaf_bonus_is_inverse_cdf_of_target():
    p_root = np.array([0.1, 0.2, 0.3, 0.4])
    tok, par, p, q = _star_problem(p_root, p_root, [], 4)
    for u, want in [(0.05, 0), (0.1, 1), (0.29, 1), (0.31, 2), (0.61, 3), (0.999, 3)]:
        _, v, _ = mss.verify_mss_tree(tok, par, p, q, np.zeros(1), u)
        assert v == want, (u, v)


def test_losslessness_first_token_distribution():
    """Children drawn i.i.d. from q_root; the first emitted token must follow p_root exactly."""
    rng = np.random.default_rng(7)
    V, k, n = 6, 3, 40000
    p_root = rng.dirichlet(np.ones(V) * 0.7)
    q_root = rng.dirichlet(np.ones(V) * 0.7)
    counts = np.zeros(V)
    for _ in range(n):
        kids = rng.choice(V, size=k, p=q_root)
        tok, par, p, q = _star_problem(p_root, q_root, kids, V)
        pth, v, _ = mss.verify_mss_tree(tok, par, p, q, rng.random(k + 1), rng.random())
        first = int(tok[pth[1]]) if len(pth) > 1 else v
        counts[first] += 1
    freq = counts / n
    sigma = np.sqrt(p_root * (1 - p_root) / n)
    assert np.all(np.abs(freq - p_root) < 4.5 * sigma + 1e-4), (freq, p_root)


def test_losslessness_catches_a_wrong_residual():
    """Control for the pin above: skipping the residual update (p stays the target) skews the histogram."""
    rng = np.random.default_rng(8)
    V, k, n = 6, 3, 20000
    p_root = rng.dirichlet(np.ones(V) * 0.7)
    q_root = rng.dirichlet(np.ones(V) * 0.7)
    counts = np.zeros(V)
    for _ in range(n):
        kids = rng.choice(V, size=k, p=q_root)
        u = rng.random(k)
        first = None
        for j, t in enumerate(kids):   # buggy variant: no residual
            if u[j] * q_root[t] < p_root[t]:
                first = t
                break
        if first is None:
            first = int(np.searchsorted(np.cumsum(p_root), rng.random(), side="right"))
        counts[first] += 1
    freq = counts / n
    sigma = np.sqrt(p_root * (1 - p_root) / n)
    assert np.any(np.abs(freq - p_root) > 4.5 * sigma + 1e-4)


def test_invalid_tree_status():
    prob = make_mss_problem(trees.heap_kary(7, 2)[None], 16, 4)
    prob.parent[0, 4] = 6
    _, plen, _, st, _ = mss.verify_mss(prob.tokens, prob.parent, prob.p_target, prob.q_draft, prob.u_accept,
                                       prob.u_bonus)
    assert st[0] == 2 and plen[0] == 0


def test_bench_config_shapes_and_acceptance():
    prob = mss_config("c4")
    assert prob.p_target.shape == (16, 64, 50280)
    path, plen, bonus, st, mm = mss.verify_mss(prob.tokens, prob.parent, prob.p_target, prob.q_draft,
                                               prob.u_accept, prob.u_bonus)
    assert (st == 0).all() and (plen >= 1).all() and (bonus >= 0).all() and (bonus < 50280).all()
    for b in range(16):   # root-anchored, parent-linked
        assert path[b, 0] == 0
        for s in range(1, plen[b]):
            assert prob.parent[b, path[b, s]] == path[b, s - 1]
