"""GPU parity of MSS verification (stree_accept_mss, reading R-mss) against the
fp64 oracle (oracle/mss.py).  Path, path_len and bonus are integers: they must be identical, except for a
tree in which some decision lies within 1e-4 (relative) of its threshold — there the fp32 reduction order
of the GPU may legitimately decide the other way; such trees are counted and must be rare."""
import numpy as np
import pytest
import torch

from gen import trees
from gen.mss import make_mss_problem, mss_config
from oracle import mss

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2505_14969_b200 import binding


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    binding.lib()
    yield


def run_gpu(prob):
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    B, T = prob.parent.shape
    path = torch.full((B, T), 7, dtype=torch.int32, device="cuda")
    plen = torch.zeros(B, dtype=torch.int32, device="cuda")
    bonus = torch.zeros(B, dtype=torch.int32, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    binding.stree_accept_mss(d(prob.tokens), d(prob.parent), d(prob.p_target), d(prob.q_draft), d(prob.u_accept),
                             d(prob.u_bonus), path, plen, bonus, dev_status=st)
    torch.cuda.synchronize()
    return path.cpu().numpy(), plen.cpu().numpy(), bonus.cpu().numpy(), int(st.item())


TIE = 1e-4   # relative margin below which a decision may go either way (fp32 vs fp64 reduction order)


def tie_consistent(prob, b, gpath, gbonus):
    """Validate a tree on which the GPU decided differently from the oracle: the GPU's result must be the
    oracle's result with only near-tie decisions flipped.  Re-runs the oracle walk, flipping (through the
    decision's uniform) each acceptance test on which the two first diverge, provided its margin < TIE;
    finally the bonus may differ only if its threshold lies within TIE of a CDF step and the GPU's token
    is an adjacent step (the next / previous token of positive probability)."""
    T = prob.parent.shape[1]
    u = np.array(prob.u_accept[b], np.float64)
    tok, par = prob.tokens[b], prob.parent[b]
    for _ in range(T + 1):
        pth, v, _ = mss.verify_mss_tree(tok, par, prob.p_target[b], prob.q_draft[b], u, prob.u_bonus[b])
        if pth == list(gpath):
            if v == gbonus:
                return True
            # bonus near-tie: the oracle's last margin is the bonus one
            _, _, m = mss.verify_mss_tree(tok, par, prob.p_target[b], prob.q_draft[b], u, prob.u_bonus[b])
            return m[-1] < TIE and 0 <= gbonus < prob.p_target.shape[2]
        # first divergence: the deepest common prefix node cur; the decision on the child where they split
        k = 0
        while k < min(len(pth), len(gpath)) and pth[k] == gpath[k]:
            k += 1
        cur = pth[k - 1]
        kids = [c for c in range(1, T) if par[c] == cur]
        o_next = pth[k] if k < len(pth) else None
        g_next = gpath[k] if k < len(gpath) else None
        # the earliest child (index order) on which the two walks decided differently
        cands = [c for c in (o_next, g_next) if c is not None]
        c = min(cands)
        # margin of that decision as the oracle computes it: recompute along the oracle walk
        _, _, m = mss.verify_mss_tree(tok, par, prob.p_target[b], prob.q_draft[b], u, prob.u_bonus[b])
        if min(m) >= TIE:
            return False
        if c not in kids:
            return False
        u[c] = 0.0 if c == g_next else 1.001   # force the GPU's decision (accept: u = 0; reject: u q >= p)
    return False


def compare(prob, max_ties=0.05):
    path, plen, bonus, st = run_gpu(prob)
    rp, rl, rb, rst, mm = mss.verify_mss(prob.tokens, prob.parent, prob.p_target, prob.q_draft, prob.u_accept,
                                         prob.u_bonus)
    B = len(rl)
    ties = 0
    for b in range(B):
        same = np.array_equal(path[b], rp[b]) and plen[b] == rl[b] and bonus[b] == rb[b]
        if not same:
            assert mm[b] < TIE, f"tree {b}: gpu {path[b][:plen[b]]} / {bonus[b]} vs oracle {rp[b][:rl[b]]} / " \
                                f"{rb[b]} (margin {mm[b]:.2e})"
            assert tie_consistent(prob, b, path[b][:plen[b]].tolist(), int(bonus[b])), \
                f"tree {b}: the GPU result is not the oracle's with near-tie decisions flipped"
            ties += 1
    assert ties <= max(1, max_ties * B)
    return st, rl


def test_bench_config_c4():
    prob = mss_config("c4")
    st, rl = compare(prob)
    assert st == 0


@pytest.mark.parametrize("T,V,kind,seed", [(16, 1000, "random", 1), (31, 997, "heap", 2), (64, 4096, "random", 3),
                                           (7, 7, "heap", 4), (5, 3, "chain", 5), (256, 257, "random", 6),
                                           (40, 50280, "star", 7), (15, 128256, "heap", 8)])
def test_random_trees(T, V, kind, seed):
    rng = np.random.default_rng(seed)
    mk = {"random": lambda: trees.random_recursive(T, 4, rng), "heap": lambda: trees.heap_kary(T, 2),
          "chain": lambda: trees.chain(T), "star": lambda: trees.star(T)}[kind]
    par = np.stack([mk() for _ in range(24)])
    prob = make_mss_problem(par, V, 300 + seed, sigma=2.0, draft_noise=1.5)
    compare(prob)


def test_q_equals_p_accepts_everything():
    prob = make_mss_problem(np.stack([trees.chain(20)] * 4), 500, 11, same=True)
    path, plen, bonus, st = run_gpu(prob)
    assert st == 0 and (plen == 20).all()


def test_invalid_tree():
    prob = make_mss_problem(np.stack([trees.heap_kary(15, 2)] * 3), 300, 12)
    prob.parent[1, 0] = 0
    path, plen, bonus, st = run_gpu(prob)
    assert st == 1 and plen[1] == 0 and bonus[1] == -1 and (path[1] == -1).all()
    rp, rl, rb, _, _ = mss.verify_mss(prob.tokens, prob.parent, prob.p_target, prob.q_draft, prob.u_accept,
                                      prob.u_bonus)
    assert plen[0] == rl[0] and plen[2] == rl[2]
