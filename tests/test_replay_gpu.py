"""GPU parity of the fused replay + scan call (stree_replay_scan, §8(f) NEXT #1):
result == oracle.commit(previous tree, accepted path, h) followed by
oracle.tree_scan(new tree, h0 = committed state)."""
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


def make_pair(B, Tp, T, H, P, N, G, io, seed, prev_kind="recursive", p_match=0.9):
    rng = np.random.default_rng(seed)
    if prev_kind == "chain":
        pp = np.stack([trees.chain(Tp)] * B)
    else:
        pp = np.stack([trees.random_recursive(Tp, 3, rng) for _ in range(B)])
    pn = np.stack([trees.random_recursive(T, 4, rng) for _ in range(B)])
    prev = inputs.make_problem(inputs.Dims(B, Tp, H, P, N, G, io), pp, seed=seed)
    new = inputs.make_problem(inputs.Dims(B, T, H, P, N, G, io), pn, seed=seed + 1)
    new.A, new.D, new.h0 = prev.A, prev.D, prev.h0   # same layer, same state
    if prev_kind == "chain":
        tok = np.tile(np.arange(100, 100 + Tp, dtype=np.int32), (B, 1))
        vt = np.roll(tok, -1, axis=1)
    else:
        tok, vt = inputs.make_accept_inputs(pp, seed=seed + 2, p_match=p_match)
    path, plen, _, _ = oracle.accept(tok, pp, vt)
    return prev, new, path, plen


def run_fused(prev, new, path, plen, use_parent=True):
    tp = api.upload(prev)
    tn = api.upload(new)
    h = tp["h0"].clone()
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    y = api.replay_scan(tp, torch.from_numpy(path).cuda(), torch.from_numpy(plen).cuda(), tn, h, dev_status=st,
                        use_parent=use_parent)
    torch.cuda.synchronize()
    return y.float().cpu().numpy(), h.cpu().numpy(), int(st.item())


def oracle_pair(prev, new, path, plen):
    hk, hst = oracle.commit_problem(prev, path, plen)
    y, yst = oracle.tree_scan(new.io_as_f32("x"), new.dt, new.A, new.io_as_f32("Bm"), new.io_as_f32("Cm"), new.D,
                              hk, new.parent, n_groups=new.dims.n_groups)
    return y, hk, hst, yst


@pytest.mark.parametrize("shape", [(16, 64, 64, 80, 64, 128, 1), (1, 64, 64, 80, 64, 128, 1),
                                   (3, 40, 24, 16, 64, 64, 1), (4, 32, 50, 24, 64, 128, 2),
                                   (2, 13, 64, 12, 64, 128, 1), (16, 64, 50, 80, 64, 128, 1), (12, 30, 37, 96, 64, 128, 1)])
@pytest.mark.parametrize("impl", ["auto", "pipeline"])
def test_replay_scan_matches_oracle(shape, impl):
    B, Tp, T, H, P, N, G = shape
    prev, new, path, plen = make_pair(B, Tp, T, H, P, N, G, "bf16", seed=Tp * 7 + T)
    d = binding.stree_dims(B, T, H, P, N, G, 1)
    binding.stree_set_scan_impl(binding.STREE_SCAN_TC_PIPELINE if impl == "pipeline" else binding.STREE_SCAN_AUTO)
    try:
        # a fused tcgen05 kernel serves this shape: the small-batch one (4) when B·H <= #SMs
        assert binding.stree_scan_kernel_for(d) in ((2,) if impl == "pipeline" else (2, 4))
        y, h, st = run_fused(prev, new, path, plen)
    finally:
        binding.stree_set_scan_impl(binding.STREE_SCAN_AUTO)
    yr, hr, hst, yst = oracle_pair(prev, new, path, plen)
    assert st == 0 and not hst.any() and not yst.any()
    assert_h_close(h, hr, TOL_F32)
    assert_y_close(y, yr, TOL_BF16)


@pytest.mark.parametrize("flags", [0, 7, 15, 31])
@pytest.mark.parametrize("B", [16, 1])
def test_replay_launch_flags(flags, B):
    """PDL off, and PDL with the EARLY_STATE + EARLY_REPLAY promises (state ring and replay prologue
    ahead of the dependency wait): same result, including an invalid path's status."""
    prev, new, path, plen = make_pair(B, 64, 64, 80, 64, 128, 1, "bf16", seed=31)
    path = path.copy()
    bad = min(3, B - 1)
    path[bad, 0] = 2
    binding.stree_set_launch_flags(flags)
    try:
        y, h, st = run_fused(prev, new, path, plen)
    finally:
        binding.stree_set_launch_flags(binding.STREE_LAUNCH_PDL)
    yr, hr, hst, _ = oracle_pair(prev, new, path, plen)
    assert st == 3 and hst[bad] == 3
    assert_h_close(h, hr, TOL_F32)
    assert_y_close(y, yr, TOL_BF16)


@pytest.mark.parametrize("B,H,Tp", [(2, 8, 64), (2, 8, 200), (16, 80, 130), (1, 80, 256)])
def test_replay_long_paths_use_l2_path(B, H, Tp):
    """Accepted paths longer than the staged nodes (full chains), including previous trees of more than 64
    accepted nodes (the chunked path-cumsum), through both fused kernels (small-batch: B·H <= #SMs)."""
    prev, new, path, plen = make_pair(B, Tp, 64, H, 64, 128, 1, "bf16", seed=5 + Tp, prev_kind="chain")
    assert (plen == Tp).all()
    y, h, st = run_fused(prev, new, path, plen, use_parent=False)
    yr, hr, _, _ = oracle_pair(prev, new, path, plen)
    assert_h_close(h, hr, TOL_F32)
    assert_y_close(y, yr, TOL_BF16)


def test_replay_invalid_path_keeps_state():
    prev, new, path, plen = make_pair(3, 32, 32, 8, 64, 128, 1, "bf16", seed=9)
    path = path.copy()
    path[1, 0] = 3            # not root-anchored
    y, h, st = run_fused(prev, new, path, plen)
    assert st == 3
    hr, hst = oracle.commit_problem(prev, path, plen)
    assert list(hst) == [0, 3, 0]
    assert np.array_equal(h[1], prev.h0[1])
    assert_h_close(h, hr, TOL_F32)
    yr, _ = oracle.tree_scan(new.io_as_f32("x"), new.dt, new.A, new.io_as_f32("Bm"), new.io_as_f32("Cm"), new.D,
                             hr, new.parent)
    assert_y_close(y, yr, TOL_BF16)


def test_replay_invalid_new_tree_zero_y_state_committed():
    prev, new, path, plen = make_pair(3, 32, 32, 8, 64, 128, 1, "bf16", seed=11)
    new.parent = new.parent.copy()
    new.parent[2, 5] = 30
    y, h, st = run_fused(prev, new, path, plen)
    assert st == 2 and not y[2].any()
    yr, hr, _, _ = oracle_pair(prev, new, path, plen)
    assert_h_close(h, hr, TOL_F32)
    assert_y_close(y[:2], yr[:2], TOL_BF16)


def test_replay_fp32_falls_back_to_two_launches():
    prev, new, path, plen = make_pair(2, 24, 24, 4, 64, 128, 1, "f32", seed=13)
    y, h, st = run_fused(prev, new, path, plen)
    yr, hr, _, _ = oracle_pair(prev, new, path, plen)
    assert_h_close(h, hr, TOL_F32)
    assert_y_close(y, yr, TOL_F32)


def test_replay_equals_separate_commit_then_scan():
    prev, new, path, plen = make_pair(16, 64, 64, 80, 64, 128, 1, "bf16", seed=21)
    yf, hf, _ = run_fused(prev, new, path, plen)
    tp, tn = api.upload(prev), api.upload(new)
    hs = api.commit(tp, torch.from_numpy(path).cuda(), torch.from_numpy(plen).cuda())
    tn["h0"] = hs
    ys = api.tree_scan(tn).float().cpu().numpy()
    assert_h_close(hf, hs.cpu().numpy(), 1e-5)
    assert_y_close(yf, ys, 1e-2)


def test_replay_kernel_selection_boundaries():
    """Around the small-batch kernel's grid limits (one head per CTA: B·H <= #SMs; one CTA per SM when
    2·B·H <= #SMs, two per SM above): the fused call at B·H = #SMs/2, #SMs/2 + 2, #SMs and #SMs + 2 (the last
    one on the pipeline kernel), each against the oracle."""
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    for units, expect in ((nsm // 2, 4), (nsm // 2 + 2, 4), (nsm, 4), (nsm + 2, 2)):
        B = 2
        H = units // B
        prev, new, path, plen = make_pair(B, 40, 48, H, 64, 128, 1, "bf16", seed=units)
        d = binding.stree_dims(B, 48, H, 64, 128, 1, 1)
        assert binding.stree_scan_kernel_for(d) == expect, (units, expect)
        y, h, st = run_fused(prev, new, path, plen)
        yr, hr, hst, yst = oracle_pair(prev, new, path, plen)
        assert st == 0 and not hst.any() and not yst.any()
        assert_h_close(h, hr, TOL_F32)
        assert_y_close(y, yr, TOL_BF16)
