"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same
seeded inputs.  Mask / depth / accept path are bit-exact; y and h_new within
the north_star tolerances (1e-4 fp32 path, 2e-2 bf16 inputs)."""
import itertools

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


def dev_status():
    return torch.zeros(1, dtype=torch.int32, device="cuda")


def y_of(y):
    return y.float().cpu().numpy()


def scan_both(prob, impl=None):
    if impl is not None:
        binding.stree_set_scan_impl(impl)
    try:
        t = api.upload(prob)
        st = dev_status()
        y = api.tree_scan(t, st)
        torch.cuda.synchronize()
    finally:
        binding.stree_set_scan_impl(binding.STREE_SCAN_AUTO)
    ref, rst = oracle.scan_problem(prob)
    return y_of(y), ref, int(st.item()), rst


def tol_of(prob):
    return TOL_BF16 if prob.dims.io_dtype == "bf16" else TOL_F32


# ---------------------------------------------------------------------------
# K1 mask
# ---------------------------------------------------------------------------
def _mask_check(parent_b):
    par = torch.from_numpy(parent_b).cuda()
    st = dev_status()
    m, d = api.build_mask(par, st)
    torch.cuda.synchronize()
    rm, rd, rst = oracle.build_mask(parent_b)
    assert np.array_equal(m.cpu().numpy().view(np.uint32), rm)
    assert np.array_equal(d.cpu().numpy(), rd)
    return int(st.item()), rst


def test_mask_configs_and_sweep():
    for cfg in ("c1", "c2", "c3", "c4"):
        _, par = inputs.config_trees(cfg, 1)
        assert _mask_check(par)[0] == 0
    for name, par in inputs.sweep_cases():
        assert _mask_check(par[None])[0] == 0, name


def test_mask_bruteforce_all_trees_T_le_7():
    for T in range(1, 8):
        pars = np.array([(-1,) + tail for tail in itertools.product(*[range(i) for i in range(1, T)])], np.int32)
        assert _mask_check(pars)[0] == 0


def test_mask_invalid_trees_flagged():
    good = trees.heap_kary(10, 2)
    bad = good.copy()
    bad[5] = 7
    st, rst = _mask_check(np.stack([good, bad, good]))
    assert st == 2 and list(rst) == [0, 2, 0]
    root = good.copy()
    root[0] = 0
    st, rst = _mask_check(root[None])
    assert st == 1 and rst[0] == 1


# ---------------------------------------------------------------------------
# K2 scan
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("cfg,io", [("c1", None), ("c2", "bf16"), ("c2", "f32"), ("c3", "bf16"), ("c3", "f32"),
                                    ("c4", "bf16")])
def test_scan_configs(cfg, io):
    prob = inputs.config_problem(cfg, io_dtype=io)
    y, ref, st, rst = scan_both(prob)
    assert st == 0 and not rst.any()
    assert_y_close(y, ref, tol_of(prob))


@pytest.mark.parametrize("impl", [1, 0])
def test_scan_sweep_c5(impl):
    for k, (name, par) in enumerate(inputs.sweep_cases()):
        d = inputs.Dims(1, len(par), 8, 64, 128, 1, "bf16")
        prob = inputs.make_problem(d, par[None], seed=inputs.BASE_SEED + 4 + k)
        y, ref, st, _ = scan_both(prob, impl)
        assert st == 0
        assert_y_close(y, ref, TOL_BF16)


def test_scan_sweep_c5_fp32():
    for k, (name, par) in enumerate(inputs.sweep_cases()[::3]):
        d = inputs.Dims(1, len(par), 4, 64, 128, 1, "f32")
        prob = inputs.make_problem(d, par[None], seed=inputs.BASE_SEED + 40 + k)
        y, ref, st, _ = scan_both(prob)
        assert_y_close(y, ref, TOL_F32)


@pytest.mark.parametrize("shape", [(3, 5, 2, 3, 7, 1), (2, 33, 6, 16, 16, 2), (2, 70, 4, 96, 40, 4),
                                   (1, 1, 3, 64, 128, 1), (2, 129, 2, 64, 128, 1), (1, 256, 2, 130, 8, 1)])
@pytest.mark.parametrize("io", ["f32", "bf16"])
def test_scan_odd_shapes(shape, io):
    B, T, H, P, N, G = shape
    rng = np.random.default_rng(T * 7 + P)
    par = np.stack([trees.random_recursive(T, 3, rng) for _ in range(B)])
    prob = inputs.make_problem(inputs.Dims(B, T, H, P, N, G, io), par, seed=T + P + N)
    y, ref, st, _ = scan_both(prob)
    assert_y_close(y, ref, tol_of(prob))


@pytest.mark.parametrize("variant", ["stress_decay", "no_decay", "large_x", "h0_zero", "D_none"])
@pytest.mark.parametrize("io", ["f32", "bf16"])
def test_scan_stress_variants(variant, io):
    d = inputs.Dims(2, 64, 8, 64, 128, 1, io)
    par = np.stack([trees.heap_kary(64, 2), trees.chain(64)])
    kw = dict(stress_decay=dict(dt_range=(0.5, 1.0), A_range=(16.0, 16.0)),
              no_decay=dict(dt_range=(1e-6, 1e-5)),
              large_x=dict(x_scale=100.0), h0_zero=dict(h0_zero=True), D_none=dict(D_none=True))[variant]
    prob = inputs.make_problem(d, par, seed=99, **kw)
    y, ref, st, _ = scan_both(prob)
    assert_y_close(y, ref, tol_of(prob))


def test_scan_null_h0_and_D():
    prob = inputs.config_problem("c2", io_dtype="f32")
    t = api.upload(prob)
    y = torch.empty_like(t["x"])
    binding.stree_tree_scan(t["x"], t["dt"], t["A"], t["Bm"], t["Cm"], None, None, t["parent"], y)
    ref, _ = oracle.tree_scan(prob.x, prob.dt, prob.A, prob.Bm, prob.Cm, None, None, prob.parent)
    assert_y_close(y_of(y), ref, TOL_F32)


def test_scan_invalid_tree_zero_and_status():
    d = inputs.Dims(3, 32, 4, 64, 128, 1, "bf16")
    par = np.stack([trees.heap_kary(32, 2)] * 3)
    par[1, 9] = 20
    prob = inputs.make_problem(d, par, seed=5)
    t = api.upload(prob)
    st = dev_status()
    y = api.tree_scan(t, st)
    yy = y_of(y)
    assert int(st.item()) == 2
    assert not yy[1].any()
    ref, rst = oracle.scan_problem(prob)
    assert list(rst) == [0, 2, 0]
    assert_y_close(yy[[0, 2]], ref[[0, 2]], TOL_BF16)


def test_scan_head_shard_concat_bitexact():
    """Head-sharded then concatenated y == unsharded y, bit for bit (SURVEY §4 GPU properties)."""
    prob = inputs.config_problem("c4", batch=4)
    t = api.upload(prob)
    y = api.tree_scan(t)
    parts = []
    for h0_, h1_ in ((0, 40), (40, 80)):
        ts = dict(t)
        ts["x"] = t["x"][:, :, h0_:h1_].contiguous()
        ts["dt"] = t["dt"][:, :, h0_:h1_].contiguous()
        ts["A"] = t["A"][h0_:h1_].contiguous()
        ts["D"] = t["D"][h0_:h1_].contiguous()
        ts["h0"] = t["h0"][:, h0_:h1_].contiguous()
        parts.append(api.tree_scan(ts))
    assert torch.equal(torch.cat(parts, dim=2), y)


def test_scan_subtree_locality_bitexact():
    prob = inputs.config_problem("c3")
    t = api.upload(prob)
    y = api.tree_scan(t)
    t2 = dict(t)
    t2["x"] = t["x"].clone()
    j = 37
    t2["x"][0, j] += 1
    y2 = api.tree_scan(t2)
    rm, _, _ = oracle.build_mask(prob.parent)
    on_path = np.array([(rm[0, i, j // 32] >> (j % 32)) & 1 for i in range(64)], bool)
    diff = (y2 != y).flatten(2).any(-1)[0].cpu().numpy()
    assert not diff[~on_path].any() and diff[j]


# ---------------------------------------------------------------------------
# K3 accept
# ---------------------------------------------------------------------------
def test_accept_random_bitexact():
    rng = np.random.default_rng(3)
    for T in (1, 2, 7, 13, 32, 64, 100, 256):
        for p in (0.0, 0.5, 0.9, 1.0):
            B = 16
            par = np.stack([trees.random_recursive(T, int(rng.integers(1, 5)), rng) for _ in range(B)])
            tok, vt = inputs.make_accept_inputs(par, seed=int(rng.integers(1 << 30)), p_match=p,
                                                dup_siblings=(T % 2 == 0))
            tt = [torch.from_numpy(a).cuda() for a in (tok, par, vt)]
            path, plen, bonus = api.accept(*tt)
            rp, rl, rb, _ = oracle.accept(tok, par, vt)
            assert np.array_equal(path.cpu().numpy(), rp)
            assert np.array_equal(plen.cpu().numpy(), rl)
            assert np.array_equal(bonus.cpu().numpy(), rb)


def test_accept_chain_full_and_invalid():
    T = 256
    par = trees.chain(T)[None]
    tok = np.arange(1000, 1000 + T, dtype=np.int32)[None]
    vt = np.roll(tok, -1, axis=1)
    path, plen, bonus = api.accept(*[torch.from_numpy(a).cuda() for a in (tok, par, vt)])
    assert plen.item() == T and np.array_equal(path.cpu().numpy()[0], np.arange(T))
    bad = par.copy()
    bad[0, 0] = 3
    st = dev_status()
    path, plen, bonus = api.accept(*[torch.from_numpy(a).cuda() for a in (tok, bad, vt)], dev_status=st)
    assert st.item() == 1 and plen.item() == 0 and bonus.item() == -1 and (path == -1).all()


# ---------------------------------------------------------------------------
# K4 commit
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("cfg,io", [("c1", None), ("c2", "bf16"), ("c3", "bf16"), ("c3", "f32"), ("c4", "bf16")])
def test_commit_configs(cfg, io):
    prob = inputs.config_problem(cfg, io_dtype=io)
    tok, vt = inputs.make_accept_inputs(prob.parent, seed=17, p_match=0.9)
    rp, rl, _, _ = oracle.accept(tok, prob.parent, vt)
    t = api.upload(prob)
    st = dev_status()
    hn = api.commit(t, torch.from_numpy(rp).cuda(), torch.from_numpy(rl).cuda(), dev_status=st)
    ref, rst = oracle.commit_problem(prob, rp, rl)
    assert st.item() == 0 and not rst.any()
    assert_h_close(hn.cpu().numpy(), ref, TOL_F32)


def test_commit_inplace_long_chain_and_no_parent():
    T = 256
    d = inputs.Dims(2, T, 4, 64, 128, 1, "bf16")
    par = np.stack([trees.chain(T)] * 2)
    prob = inputs.make_problem(d, par, seed=8)
    path = np.stack([np.arange(T), np.arange(T)]).astype(np.int32)
    plen = np.array([T, 100], np.int32)
    path[1, 100:] = -1
    t = api.upload(prob)
    ref, _ = oracle.commit_problem(prob, path, plen)
    h = t["h0"]
    api.commit(t, torch.from_numpy(path).cuda(), torch.from_numpy(plen).cuda(), h_new=h, use_parent=False)
    assert_h_close(h.cpu().numpy(), ref, TOL_F32)


@pytest.mark.parametrize("shape", [(16, 64, 80, 64, 128, 1), (3, 37, 24, 64, 64, 2), (2, 200, 12, 64, 128, 3),
                                   (1, 1, 3, 64, 128, 1)])
def test_commit_pipeline_kernel(shape):
    """stree_commit on the TMA pipeline (replay warps of the tcgen05 kernel): oracle parity, equality with
    the CUDA-core ring kernel, distinct and in-place outputs."""
    B, T, H, P, N, G = shape
    rng = np.random.default_rng(T * 13 + H)
    par = np.stack([trees.random_recursive(T, 4, rng) for _ in range(B)])
    prob = inputs.make_problem(inputs.Dims(B, T, H, P, N, G, "bf16"), par, seed=T + N)
    tok, vt = inputs.make_accept_inputs(par, seed=T + 1, p_match=0.9)
    rp, rl, _, _ = oracle.accept(tok, par, vt)
    d = binding.stree_dims(B, T, H, P, N, G, 1)
    assert binding.stree_commit_kernel_for(d, True) == 2
    assert binding.stree_commit_kernel_for(d, False) == 1
    t = api.upload(prob)
    path, plen = torch.from_numpy(rp).cuda(), torch.from_numpy(rl).cuda()
    st = dev_status()
    hn = api.commit(t, path, plen, dev_status=st)
    ref, rst = oracle.commit_problem(prob, rp, rl)
    assert st.item() == 0 and not rst.any()
    assert_h_close(hn.cpu().numpy(), ref, TOL_F32)
    binding.stree_set_scan_impl(binding.STREE_SCAN_SIMT)
    try:
        hs = api.commit(t, path, plen)
    finally:
        binding.stree_set_scan_impl(binding.STREE_SCAN_AUTO)
    assert_h_close(hn.cpu().numpy(), hs.cpu().numpy(), 1e-5)
    h = t["h0"].clone()
    t2 = dict(t, h0=h)
    api.commit(t2, path, plen, h_new=h)
    assert torch.equal(h, hn)


def test_commit_invalid_paths():
    prob = inputs.config_problem("c2")
    T = prob.dims.n_nodes
    par = prob.parent[0]
    kids = trees.children_lists(par)
    bad_paths = [([1], 1), ([0, kids[0][0], kids[kids[0][1]][0]], 3), ([0], 0), ([0], T + 1)]
    for p, r in bad_paths:
        pa = np.full((1, T), -1, np.int32)
        pa[0, : len(p)] = p
        t = api.upload(prob)
        st = dev_status()
        hn = api.commit(t, torch.from_numpy(pa).cuda(), torch.tensor([r], dtype=torch.int32, device="cuda"),
                        dev_status=st)
        assert st.item() == 3
        assert torch.equal(hn, t["h0"])


def test_graft_invariant_two_iterations():
    """Alg. 1 losslessness on the GPU path: scan(tree2, h0=commit(tree1)) equals
    the oracle's scan of tree1 with tree2 grafted under the last accepted node."""
    rng = np.random.default_rng(4)
    T1 = T2 = 32
    p1 = trees.random_recursive(T1, 3, rng)
    p2 = trees.random_recursive(T2, 3, rng)
    d1 = inputs.Dims(1, T1, 8, 64, 128, 1, "f32")
    prob1 = inputs.make_problem(d1, p1[None], seed=1)
    tok, vt = inputs.make_accept_inputs(p1[None], seed=2, p_match=0.9)
    t1 = api.upload(prob1)
    path, plen, bonus = api.accept(*[torch.from_numpy(a).cuda() for a in (tok, p1[None], vt)])
    hk = api.commit(t1, path, plen)
    k = int(path[0, plen[0] - 1].item())
    prob2 = inputs.make_problem(inputs.Dims(1, T2, 8, 64, 128, 1, "f32"), p2[None], seed=3)
    prob2.A, prob2.D = prob1.A, prob1.D
    t2 = api.upload(prob2)
    t2["h0"] = hk
    y2 = y_of(api.tree_scan(t2))
    pg = np.concatenate([p1, [k], p2[1:] + T1]).astype(np.int32)[None]
    cat = lambda a, b: np.concatenate([a, b], axis=1)  # noqa: E731
    yg, _ = oracle.tree_scan(cat(prob1.x, prob2.x), cat(prob1.dt, prob2.dt), prob1.A, cat(prob1.Bm, prob2.Bm),
                             cat(prob1.Cm, prob2.Cm), prob1.D, prob1.h0, pg)
    assert_y_close(y2, yg[:, T1:], TOL_F32)


# ---------------------------------------------------------------------------
# tcgen05 kernel specifically (forced), incl. N=64, G>1, ragged T, NULL h0/D
# ---------------------------------------------------------------------------
def test_tc_kernel_selected_for_mamba2_shapes():
    # batch-1 layers (c2, c3: B·H <= #SMs) take the small-batch kernel, c4 the pipelined one
    for cfg, k in (("c2", 4), ("c3", 4), ("c4", 2)):
        d, _ = inputs.config_trees(cfg, 0)
        dims = binding.stree_dims(d.batch, d.n_nodes, d.n_heads, d.head_dim, d.d_state, d.n_groups, 1)
        assert binding.stree_scan_kernel_for(dims) == k, cfg
        binding.stree_set_scan_impl(binding.STREE_SCAN_TC_PIPELINE)
        try:
            assert binding.stree_scan_kernel_for(dims) == 2, cfg
        finally:
            binding.stree_set_scan_impl(binding.STREE_SCAN_AUTO)


# the forced tcgen05 tests run both the small-batch kernel (where B·H <= #SMs) and the pipelined one
TC_IMPLS = pytest.mark.parametrize("impl", ["tc", "pipeline"])


def _impl(name):
    return {"tc": binding.STREE_SCAN_TC, "pipeline": binding.STREE_SCAN_TC_PIPELINE}[name]


@pytest.mark.parametrize("shape", [(1, 64, 80, 64, 128, 1), (16, 64, 80, 64, 128, 1), (3, 1, 5, 64, 128, 1),
                                   (2, 13, 7, 64, 64, 1), (4, 50, 24, 64, 128, 2), (2, 33, 30, 64, 64, 3),
                                   (5, 17, 40, 64, 128, 1), (16, 50, 80, 64, 128, 1), (12, 37, 96, 64, 128, 1)])
@TC_IMPLS
def test_tc_forced_shapes(shape, impl):
    B, T, H, P, N, G = shape
    rng = np.random.default_rng(B * 1000 + T)
    par = np.stack([trees.random_recursive(T, 3, rng) for _ in range(B)])
    prob = inputs.make_problem(inputs.Dims(B, T, H, P, N, G, "bf16"), par, seed=T * 31 + H)
    y, ref, st, _ = scan_both(prob, _impl(impl))
    assert st == 0
    assert_y_close(y, ref, TOL_BF16)


@pytest.mark.parametrize("variant", ["stress_decay", "no_decay", "large_x", "h0_zero", "D_none"])
@TC_IMPLS
def test_tc_forced_stress(variant, impl):
    d = inputs.Dims(2, 64, 8, 64, 128, 1, "bf16")
    par = np.stack([trees.heap_kary(64, 2), trees.chain(64)])
    kw = dict(stress_decay=dict(dt_range=(0.5, 1.0), A_range=(16.0, 16.0)),
              no_decay=dict(dt_range=(1e-6, 1e-5)),
              large_x=dict(x_scale=100.0), h0_zero=dict(h0_zero=True), D_none=dict(D_none=True))[variant]
    prob = inputs.make_problem(d, par, seed=98, **kw)
    y, ref, st, _ = scan_both(prob, _impl(impl))
    assert_y_close(y, ref, TOL_BF16)


@pytest.mark.parametrize("with_h0", [True, False])
@pytest.mark.parametrize("B", [16, 2])
def test_tc_mixed_decay_modes(with_h0, B):
    """Heads of one CTA alternate between the factorised decay (Y' accumulated onto Y0) and the
    direct per-element decay (Y' in its own TMEM columns): A_h spans 1..16 over a chain, so
    min Λ crosses the -64 switch within the head range.  B = 2: the small-batch kernel (one head per
    CTA, the direct Y' in the G columns)."""
    d = inputs.Dims(B, 64, 48, 64, 128, 1, "bf16")      # 16 trees: several heads per CTA
    par = np.stack([trees.chain(64) if i % 2 == 0 else trees.heap_kary(64, 2) for i in range(B)])
    prob = inputs.make_problem(d, par, seed=77, dt_range=(0.05, 0.2), A_range=(1.0, 24.0))
    lam_min = (prob.dt[0] * prob.A[None, :]).sum(axis=0)
    assert (lam_min < -64).any() and (lam_min > -64).any()
    if not with_h0:
        binding.stree_set_scan_impl(binding.STREE_SCAN_TC)
        try:
            t = api.upload(prob)
            y = torch.empty_like(t["x"])
            binding.stree_tree_scan(t["x"], t["dt"], t["A"], t["Bm"], t["Cm"], t["D"], None, t["parent"], y)
            torch.cuda.synchronize()
        finally:
            binding.stree_set_scan_impl(binding.STREE_SCAN_AUTO)
        ref, _ = oracle.tree_scan(prob.io_as_f32("x"), prob.dt, prob.A, prob.io_as_f32("Bm"),
                                  prob.io_as_f32("Cm"), prob.D, None, prob.parent)
        assert_y_close(y_of(y), ref, TOL_BF16)
        return
    y, ref, st, _ = scan_both(prob, binding.STREE_SCAN_TC)
    assert st == 0
    assert_y_close(y, ref, TOL_BF16)


@TC_IMPLS
def test_tc_null_h0_D_and_invalid_tree(impl):
    prob = inputs.config_problem("c2")
    t = api.upload(prob)
    binding.stree_set_scan_impl(_impl(impl))
    try:
        y = torch.empty_like(t["x"])
        binding.stree_tree_scan(t["x"], t["dt"], t["A"], t["Bm"], t["Cm"], None, None, t["parent"], y)
        ref, _ = oracle.tree_scan(prob.io_as_f32("x"), prob.dt, prob.A, prob.io_as_f32("Bm"),
                                  prob.io_as_f32("Cm"), None, None, prob.parent)
        assert_y_close(y_of(y), ref, TOL_BF16)
        d = inputs.Dims(3, 32, 4, 64, 128, 1, "bf16")
        par = np.stack([trees.heap_kary(32, 2)] * 3)
        par[1, 9] = 20
        p2 = inputs.make_problem(d, par, seed=5)
        t2 = api.upload(p2)
        st = dev_status()
        y2 = y_of(api.tree_scan(t2, st))
        assert int(st.item()) == 2 and not y2[1].any()
        ref2, _ = oracle.scan_problem(p2)
        assert_y_close(y2[[0, 2]], ref2[[0, 2]], TOL_BF16)
    finally:
        binding.stree_set_scan_impl(binding.STREE_SCAN_AUTO)


def test_tc_matches_simt_closely():
    """Both kernels against each other on c4 (same tolerance class)."""
    prob = inputs.config_problem("c4", batch=4)
    ya, _, _, _ = scan_both(prob, binding.STREE_SCAN_TC)
    yb, ref, _, _ = scan_both(prob, binding.STREE_SCAN_SIMT)
    assert_y_close(ya, ref, TOL_BF16)
    assert_y_close(yb, ref, TOL_BF16)
