"""GPU parity of the scan options (include/stree.h stree_scan_opts; SURVEY §8(f) unranked variants): fused
dt bias + softplus and per-(head, channel) D, through stree_tree_scan_ex / stree_replay_scan_ex /
stree_commit_ex on every scan and commit kernel, against the oracle's tree_scan_ex / commit_ex; and
variable T per tree by padding leaves under the root."""
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
    binding.stree_set_scan_impl(binding.STREE_SCAN_AUTO)


def _raw_dt(prob, bias, rng, softplus):
    """Raw projection outputs whose effective dt is in the generator's range (softplus⁻¹(dt) - bias), plus
    N(0, 0.3) noise so the transform is exercised off the pre-image."""
    dt = prob.dt.astype(np.float64)
    base = np.log(np.expm1(dt)) if softplus else dt
    raw = base - (bias[None, None, :] if bias is not None else 0.0)
    if softplus:
        raw = raw + 0.3 * rng.standard_normal(raw.shape)
    return raw.astype(np.float32)


CASES = [  # B, T, H, P, N, io: kernel served
    (2, 40, 16, 64, 128, "bf16"),    # small-batch K2s
    (16, 64, 80, 64, 128, "bf16"),   # pipeline K2
    (2, 128, 8, 64, 128, "bf16"),    # 128-row K2b
    (2, 21, 3, 8, 16, "f32"),        # SIMT (fp32 path)
]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("bias,softplus,dpc", [(True, True, True), (False, True, False), (True, False, True)])
def test_tree_scan_ex_matches_oracle(case, bias, softplus, dpc):
    B, T, H, P, N, io = case
    rng = np.random.default_rng(T + H + 2 * bias + softplus)
    par = np.stack([trees.random_recursive(T, 3, rng) for _ in range(B)])
    prob = inputs.make_problem(inputs.Dims(B, T, H, P, N, 1, io), par, seed=T * 5 + H)
    b = rng.uniform(-1, 1, H).astype(np.float32) if bias else None
    raw = _raw_dt(prob, b, rng, softplus)
    Dhp = (1 + 0.1 * rng.standard_normal((H, P))).astype(np.float32) if dpc else prob.D
    t = api.upload(prob)
    t["dt"] = torch.from_numpy(raw).cuda()
    Dd = torch.from_numpy(np.ascontiguousarray(Dhp)).cuda()
    bd = torch.from_numpy(b).cuda() if b is not None else None
    opts = binding.make_opts(bd, softplus, dpc)
    y = torch.empty_like(t["x"])
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    binding.stree_tree_scan_ex(t["x"], t["dt"], t["A"], t["Bm"], t["Cm"], Dd, t["h0"], t["parent"], y, opts, st)
    torch.cuda.synchronize()
    ref, rst = oracle.tree_scan_ex(prob.io_as_f32("x"), raw, prob.A, prob.io_as_f32("Bm"), prob.io_as_f32("Cm"), Dhp,
                                   prob.h0, par, dt_bias=b, dt_softplus=softplus, d_per_channel=dpc)
    assert st.item() == 0 and not rst.any()
    assert_y_close(y.float().cpu().numpy(), ref, TOL_BF16 if io == "bf16" else TOL_F32)


@pytest.mark.parametrize("B,T,H,io,impl", [(2, 48, 16, "bf16", "auto"), (16, 64, 80, "bf16", "pipeline"),
                                           (3, 30, 4, "f32", "auto"), (2, 200, 8, "bf16", "auto")])
def test_replay_and_commit_ex_match_oracle(B, T, H, io, impl):
    """Fused replay+scan and the plain commit with the options: the committed state uses the effective dt of
    the cached tree (the same transform as the scan that verified it)."""
    rng = np.random.default_rng(B * T + H)
    P, N = (64, 128) if io == "bf16" else (8, 16)
    pp = np.stack([trees.random_recursive(T, 3, rng) for _ in range(B)])
    pn = np.stack([trees.random_recursive(min(T, 64), 4, rng) for _ in range(B)])
    prev = inputs.make_problem(inputs.Dims(B, T, H, P, N, 1, io), pp, seed=T + 1)
    new = inputs.make_problem(inputs.Dims(B, min(T, 64), H, P, N, 1, io), pn, seed=T + 2)
    new.A, new.D, new.h0 = prev.A, prev.D, prev.h0
    b = rng.uniform(-1, 1, H).astype(np.float32)
    raw_p, raw_n = _raw_dt(prev, b, rng, True), _raw_dt(new, b, rng, True)
    Dhp = (1 + 0.1 * rng.standard_normal((H, P))).astype(np.float32)
    tok, vt = inputs.make_accept_inputs(pp, seed=T + 3, p_match=0.9)
    path, plen, _, _ = oracle.accept(tok, pp, vt)
    binding.stree_set_scan_impl(binding.STREE_SCAN_TC_PIPELINE if impl == "pipeline" else binding.STREE_SCAN_AUTO)
    tp, tn = api.upload(prev), api.upload(new)
    tp["dt"], tn["dt"] = torch.from_numpy(raw_p).cuda(), torch.from_numpy(raw_n).cuda()
    bd, Dd = torch.from_numpy(b).cuda(), torch.from_numpy(Dhp).cuda()
    opts = binding.make_opts(bd, True, True)
    pd, ld = torch.from_numpy(path).cuda(), torch.from_numpy(plen).cuda()
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    hk_ref, _ = oracle.commit_ex(prev.io_as_f32("x"), raw_p, prev.A, prev.io_as_f32("Bm"), prev.h0, path, plen, pp,
                                 dt_bias=b, dt_softplus=True)
    # plain commit (ring / TMA pipeline kernels)
    hc = torch.empty_like(tp["h0"])
    binding.stree_commit_ex(tp["x"], tp["dt"], tp["A"], tp["Bm"], tp["h0"], tp["parent"], pd, ld, hc, opts, st)
    # fused replay + scan (K2s / K2; two launches for the shapes they do not serve)
    h = tp["h0"].clone()
    y = torch.empty_like(tn["x"])
    binding.stree_replay_scan_ex(tp["x"], tp["dt"], tp["Bm"], tp["parent"], pd, ld, tn["x"], tn["dt"], tn["A"],
                                 tn["Bm"], tn["Cm"], Dd, h, tn["parent"], y, opts, st)
    torch.cuda.synchronize()
    binding.stree_set_scan_impl(binding.STREE_SCAN_AUTO)
    yr, _ = oracle.tree_scan_ex(new.io_as_f32("x"), raw_n, new.A, new.io_as_f32("Bm"), new.io_as_f32("Cm"), Dhp,
                                hk_ref, pn, dt_bias=b, dt_softplus=True, d_per_channel=True)
    assert st.item() == 0
    assert_h_close(hc.cpu().numpy(), hk_ref, TOL_F32)
    assert_h_close(h.cpu().numpy(), hk_ref, TOL_F32)
    assert_y_close(y.float().cpu().numpy(), yr, TOL_BF16 if io == "bf16" else TOL_F32)


def test_opts_null_equals_plain_and_misaligned_bias():
    prob = inputs.config_problem("c2")
    t = api.upload(prob)
    y0 = api.tree_scan(t)
    y1 = torch.empty_like(t["x"])
    binding.stree_tree_scan_ex(t["x"], t["dt"], t["A"], t["Bm"], t["Cm"], t["D"], t["h0"], t["parent"], y1, None)
    torch.cuda.synchronize()
    assert torch.equal(y0.view(torch.int16), y1.view(torch.int16))
    bias = torch.zeros(prob.dims.n_heads + 1, device="cuda")[1:]
    bad = binding.stree_scan_opts(bias.data_ptr() + 2, 1, 0)
    with pytest.raises(binding.StreeError):
        binding.stree_tree_scan_ex(t["x"], t["dt"], t["A"], t["Bm"], t["Cm"], t["D"], t["h0"], t["parent"], y1, bad)


@pytest.mark.parametrize("n,T", [(9, 16), (40, 64), (100, 128)])
def test_variable_T_by_padding_leaves_gpu(n, T):
    """Trees of different sizes in one batch (beam trees): each padded to T with leaves under
    the root.  The real nodes' outputs match the oracle of the unpadded tree (the GPU path computes the padded
    batch in one call)."""
    rng = np.random.default_rng(n)
    B, H = 3, 16
    sizes = [n, T, max(1, n // 2)]
    real = [trees.random_recursive(k, 3, rng) for k in sizes]
    par = np.stack([np.concatenate([p, np.zeros(T - len(p), np.int32)]) for p in real])
    prob = inputs.make_problem(inputs.Dims(B, T, H, 64, 128, 1, "bf16"), par, seed=n + T)
    y = api.tree_scan(api.upload(prob)).float().cpu().numpy()
    for bi, k in enumerate(sizes):
        ref, _ = oracle.tree_scan(prob.io_as_f32("x")[bi:bi + 1, :k], prob.dt[bi:bi + 1, :k], prob.A,
                                  prob.io_as_f32("Bm")[bi:bi + 1, :k], prob.io_as_f32("Cm")[bi:bi + 1, :k], prob.D,
                                  prob.h0[bi:bi + 1], real[bi][None])
        assert_y_close(y[bi:bi + 1, :k], ref, TOL_BF16)
