"""PDL / EARLY-promise safety (include/stree.h, "Launch options"): eager decode loops with the launch
order of a real verifier, every kernel of an iteration enqueued back to back on one stream with no host
synchronisation, compared iteration by iteration with the oracle (commit then scan, PAPER.md:113,
Alg. 1 l.123-125).  The accepted path changes every iteration, so a kernel that read a path, a state or
a cache before its dependency had completed would commit the wrong state."""
import numpy as np
import pytest
import torch

import oracle
from gen import inputs, trees
from tests.helpers import TOL_BF16, TOL_F32, assert_h_close, assert_y_close

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2505_14969_b200 import api, binding


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    binding.lib()
    yield
    binding.stree_set_launch_flags(binding.STREE_LAUNCH_PDL)


ALL = 31   # PDL | EARLY_STATE | EARLY_REPLAY | EARLY_TREE | EARLY_DT


def _iter_problems(B, T, H, L, K, seed):
    """K iterations x L layers of seeded inputs (one tree per iteration, shared by the layers of that
    iteration), plus acceptance inputs that change every iteration."""
    rng = np.random.default_rng(seed)
    its = []
    for it in range(K):
        par = np.stack([trees.random_recursive(T, 3, rng) for _ in range(B)])
        lay = [inputs.make_problem(inputs.Dims(B, T, H, 64, 128, 1, "bf16"), par, seed=seed + 100 * it + l)
               for l in range(L)]
        if its:   # A and D are the layer's weights: the same in every iteration
            for l in range(L):
                lay[l].A, lay[l].D = its[0][1][l].A, its[0][1][l].D
        tok, vt = inputs.make_accept_inputs(par, seed=seed + 7 * it + 1, p_match=0.8)
        its.append((par, lay, tok, vt))
    return its


@pytest.mark.parametrize("flags,mask_between", [(ALL, True), (1 | 2, False), (0, False)])
def test_eager_decode_loop_replay_scan(flags, mask_between):
    """accept -> [build_mask] -> L x replay_scan -> accept -> ... with the EARLY promises where they hold:
    EARLY_REPLAY needs a kernel between accept and the first replay (the next iteration's mask build)."""
    B, T, H, L, K = 4, 64, 16, 3, 5
    its = _iter_problems(B, T, H, L, K, seed=4242 + flags)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    binding.stree_set_launch_flags(flags)
    try:
        dev = [[api.upload(p) for p in lay] for _, lay, _, _ in its]
        h = [dev[0][l]["h0"].clone() for l in range(L)]
        toks = [(torch.from_numpy(tok).cuda(), torch.from_numpy(vt).cuda()) for _, _, tok, vt in its]
        W = (T + 31) // 32
        mask = torch.empty((B, T, W), dtype=torch.int32, device="cuda")
        path = torch.empty((B, T), dtype=torch.int32, device="cuda")
        plen = torch.empty((B,), dtype=torch.int32, device="cuda")
        bonus = torch.empty((B,), dtype=torch.int32, device="cuda")
        ys, paths = [], []
        torch.cuda.synchronize()
        # iteration 0: plain scans from the initial state, then accept
        binding.stree_build_mask(dev[0][0]["parent"], mask, None, st)
        ys.append([_scan(dev[0][l], h[l], st) for l in range(L)])
        binding.stree_accept(toks[0][0], dev[0][0]["parent"], toks[0][1], path, plen, bonus, st)
        for it in range(1, K):
            paths.append((path.clone(), plen.clone()))   # snapshot on the stream (a device copy kernel)
            if mask_between:
                binding.stree_build_mask(dev[it][0]["parent"], mask, None, st)
            yi = []
            for l in range(L):
                y = torch.empty_like(dev[it][l]["x"])
                api.replay_scan(dev[it - 1][l], path, plen, dev[it][l], h[l], dev_status=st, y=y)
                yi.append(y)
            ys.append(yi)
            binding.stree_accept(toks[it][0], dev[it][0]["parent"], toks[it][1], path, plen, bonus, st)
        torch.cuda.synchronize()
        assert st.item() == 0
    finally:
        binding.stree_set_launch_flags(binding.STREE_LAUNCH_PDL)
    # oracle, iteration by iteration
    hr = [its[0][1][l].h0.astype(np.float64) for l in range(L)]
    for l in range(L):
        p = its[0][1][l]
        yr, _ = oracle.scan_problem(p)
        assert_y_close(ys[0][l].float().cpu().numpy(), yr, TOL_BF16)
    rpath, rplen, _, _ = oracle.accept(its[0][2], its[0][0], its[0][3])
    for it in range(1, K):
        gp, gl = paths[it - 1]
        assert np.array_equal(gp.cpu().numpy(), rpath) and np.array_equal(gl.cpu().numpy(), rplen)
        for l in range(L):
            prev, new = its[it - 1][1][l], its[it][1][l]
            hk, hst = oracle.commit(prev.io_as_f32("x"), prev.dt, prev.A, prev.io_as_f32("Bm"), hr[l], rpath, rplen,
                                    parent=prev.parent)
            assert not hst.any()
            yr, _ = oracle.tree_scan(new.io_as_f32("x"), new.dt, new.A, new.io_as_f32("Bm"), new.io_as_f32("Cm"),
                                     new.D, hk, new.parent)
            hr[l] = hk
            assert_y_close(ys[it][l].float().cpu().numpy(), yr, TOL_BF16)
        rpath, rplen, _, _ = oracle.accept(its[it][2], its[it][0], its[it][3])
    for l in range(L):
        # the last iteration's commit is still pending in the decode loop: h holds the state after it-1
        assert_h_close(h[l].cpu().numpy(), hr[l], TOL_F32)


def _scan(t, h, st):
    y = torch.empty_like(t["x"])
    binding.stree_tree_scan(t["x"], t["dt"], t["A"], t["Bm"], t["Cm"], t["D"], h, t["parent"], y, st)
    return y


@pytest.mark.parametrize("flags", [ALL, 0])
def test_eager_accept_then_commit(flags):
    """accept -> stree_commit directly (the unfused order) with every flag set: stree_commit must not take
    the EARLY_REPLAY promise (its path is written by the accept kernel immediately before it)."""
    B, T, H, K = 8, 64, 24, 6
    rng = np.random.default_rng(77)
    par = np.stack([trees.random_recursive(T, 3, rng) for _ in range(B)])
    prob = inputs.make_problem(inputs.Dims(B, T, H, 64, 128, 1, "bf16"), par, seed=78)
    d = binding.stree_dims(B, T, H, 64, 128, 1, 1)
    assert binding.stree_commit_kernel_for(d, True) == 2
    t = api.upload(prob)
    h = t["h0"].clone()
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    acc = [inputs.make_accept_inputs(par, seed=500 + k, p_match=0.85) for k in range(K)]
    dacc = [(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()) for a, b in acc]
    path = torch.empty((B, T), dtype=torch.int32, device="cuda")
    plen = torch.empty((B,), dtype=torch.int32, device="cuda")
    bonus = torch.empty((B,), dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    binding.stree_set_launch_flags(flags)
    try:
        for k in range(K):   # K commits of the same cache along changing paths, state in place
            binding.stree_accept(dacc[k][0], t["parent"], dacc[k][1], path, plen, bonus, st)
            binding.stree_commit(t["x"], t["dt"], t["A"], t["Bm"], h, t["parent"], path, plen, h, st)
        torch.cuda.synchronize()
    finally:
        binding.stree_set_launch_flags(binding.STREE_LAUNCH_PDL)
    assert st.item() == 0
    hr = prob.h0.astype(np.float64)
    for k in range(K):
        rp, rl, _, _ = oracle.accept(acc[k][0], par, acc[k][1])
        hr, hst = oracle.commit(prob.io_as_f32("x"), prob.dt, prob.A, prob.io_as_f32("Bm"), hr, rp, rl, parent=par)
        assert not hst.any()
    assert_h_close(h.cpu().numpy(), hr, TOL_F32)


def test_ring_commit_small_headdim_long_chain():
    """CUDA-core ring commit with P = 8 < heads per CTA (16) and a fully accepted 256-chain: the long-path
    coefficients (16 heads x 256 floats) are wider than the staging region of short paths; the B rows,
    decays, path and barriers must sit past both."""
    B, T, H, P, N = 16, 256, 160, 8, 128
    par = np.stack([trees.chain(T)] * B)
    prob = inputs.make_problem(inputs.Dims(B, T, H, P, N, 1, "bf16"), par, seed=91)
    d = binding.stree_dims(B, T, H, P, N, 1, 1)
    assert binding.stree_commit_kernel_for(d, True) == 1
    t = api.upload(prob)
    path = torch.from_numpy(np.tile(np.arange(T, dtype=np.int32), (B, 1))).cuda()
    plen = torch.full((B,), T, dtype=torch.int32, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    for inplace in (False, True):
        h = t["h0"].clone()
        out = h if inplace else torch.empty_like(h)
        binding.stree_commit(t["x"], t["dt"], t["A"], t["Bm"], h, t["parent"], path, plen, out, st)
        torch.cuda.synchronize()
        assert st.item() == 0
        hr, _ = oracle.commit_problem(prob, path.cpu().numpy(), plen.cpu().numpy())
        assert_h_close(out.cpu().numpy(), hr, TOL_F32)
