"""GPU parity of tree attention and the KV-cache commit (reading R-attn)
against the fp64 oracle (oracle/attn.py), through the C ABI."""
import numpy as np
import pytest
import torch

from gen import trees
from gen.attn import AttnDims, attn_config, make_attn_problem
from oracle import attn as oattn
from tests.helpers import TOL_BF16, TOL_F32, _assert

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2505_14969_b200 import binding


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    binding.lib()
    yield
    binding.stree_set_scan_impl(binding.STREE_SCAN_AUTO)


def _dev(prob, name):
    a = getattr(prob, name)
    if prob.dims.io_dtype == "bf16":
        return torch.from_numpy(a.view(np.int16).copy()).view(torch.bfloat16).cuda()
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _f64(prob, name):
    return prob.as_f32(name).astype(np.float64)


def run_gpu(prob, impl=binding.STREE_SCAN_AUTO if torch.cuda.is_available() else 0, expect_kernel=None):
    binding.stree_set_scan_impl(impl)
    q, kn, vn, kc, vc = (_dev(prob, n) for n in ("q", "k_new", "v_new", "k_cache", "v_cache"))
    cl = torch.from_numpy(prob.cache_len.astype(np.int32)).cuda()
    par = torch.from_numpy(prob.parent.astype(np.int32)).cuda()
    o = torch.full_like(q, float("nan"))
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    d = binding.make_attn_dims(q, kn, kc)
    if expect_kernel is not None:
        assert binding.stree_attn_kernel_for(d) == expect_kernel
    binding.stree_tree_attn(q, kn, vn, kc, vc, cl, par, prob.scale, o, dev_status=st)
    torch.cuda.synchronize()
    binding.stree_set_scan_impl(binding.STREE_SCAN_AUTO)
    return o.float().cpu().numpy().astype(np.float64), int(st.item())


def run_oracle(prob):
    return oattn.tree_attn(_f64(prob, "q"), _f64(prob, "k_new"), _f64(prob, "v_new"), _f64(prob, "k_cache"),
                           _f64(prob, "v_cache"), prob.cache_len, prob.parent, prob.scale)


def check(o, ref, tol):
    """o [B][T][Hq][D]: blocks (tree, head), rows = nodes (tests/helpers.py checks)."""
    return _assert("attn", o, ref, tol, (1, 3), (3,))


def _tree(kind, T, rng):
    return {"random": lambda: trees.random_recursive(T, 4, rng), "chain": lambda: trees.chain(T),
            "heap": lambda: trees.heap_kary(T, 2), "star": lambda: trees.star(T),
            "wide": lambda: trees.heap_kary(T, 8)}[kind]()


def make_case(B, T, Hq, Hkv, D, S, io, seed, kind="random", cache_len=None):
    rng = np.random.default_rng(seed)
    par = np.stack([_tree(kind, T, rng) for _ in range(B)])
    return make_attn_problem(AttnDims(B, T, Hq, Hkv, D, S, io), par, seed, cache_len=cache_len,
                             len_range=(0, S))


def test_toy_fp32():
    prob = attn_config("toy", "f32")
    o, st = run_gpu(prob, expect_kernel=1)
    ref, _ = run_oracle(prob)
    assert st == 0
    check(o, ref, TOL_F32)


@pytest.mark.parametrize("kind", ["random", "chain", "heap"])
def test_fp32_simt_full_head_dim(kind):
    prob = make_case(3, 40, 8, 2, 128, 300, "f32", 5, kind, cache_len=[0, 129, 300])
    o, st = run_gpu(prob, expect_kernel=1)
    ref, _ = run_oracle(prob)
    assert st == 0
    check(o, ref, TOL_F32)


def test_hyb8b_full_size_tc():
    """The bench workload (MambaInLlama-8B attention shape, 16 trees of 64 nodes, ragged prefixes
    768..1280) in the launch configuration bench.py times."""
    prob = attn_config("hyb8b")
    o, st = run_gpu(prob, expect_kernel=2)
    ref, _ = run_oracle(prob)
    assert st == 0
    check(o, ref, TOL_BF16)


@pytest.mark.parametrize("T,Hq,Hkv,kind,lens", [
    (1, 32, 8, "random", [0, 1, 5]),             # single node, empty prefix
    (7, 4, 1, "heap", [127, 128, 129]),          # tile-boundary prefixes
    (33, 8, 8, "random", [0, 255, 256]),         # grp 1, ragged query tile
    (64, 16, 2, "wide", [1000, 17, 384]),        # grp 8: 4 query tiles = 2 CTA pairs
    (100, 12, 4, "star", [500, 0, 64]),          # grp 3 does not divide 128 -> SIMT kernel
    (130, 4, 4, "chain", [0, 130, 511]),         # two tree tiles
    (256, 8, 1, "random", [3, 700, 1024]),       # grp 8, 16 query tiles, T = 256
])
def test_bf16_ragged(T, Hq, Hkv, kind, lens):
    S = 1024
    prob = make_case(3, T, Hq, Hkv, 128, S, "bf16", 100 + T, kind, cache_len=lens)
    grp = Hq // Hkv
    o, st = run_gpu(prob, expect_kernel=2 if 128 % grp == 0 else 1)
    ref, _ = run_oracle(prob)
    assert st == 0
    check(o, ref, TOL_BF16)


def test_bf16_tc_equals_simt_kernel():
    prob = make_case(2, 48, 16, 4, 128, 600, "bf16", 77, cache_len=[599, 250])
    o_tc, _ = run_gpu(prob, expect_kernel=2)
    o_simt, _ = run_gpu(prob, impl=binding.STREE_SCAN_SIMT)
    ref, _ = run_oracle(prob)
    check(o_tc, ref, TOL_BF16)
    check(o_simt, ref, TOL_BF16)


def test_large_scores_lazy_rescale():
    """Peaky softmax (|s| up to ~40): exercises the running-max rescale path."""
    rng = np.random.default_rng(9)
    par = np.stack([trees.random_recursive(64, 3, rng) for _ in range(2)])
    prob = make_attn_problem(AttnDims(2, 64, 8, 2, 128, 512, "bf16"), par, 9, cache_len=[511, 300], q_scale=6.0)
    o, st = run_gpu(prob, expect_kernel=2)
    ref, _ = run_oracle(prob)
    check(o, ref, TOL_BF16)


@pytest.mark.parametrize("impl", ["tc", "simt"])
def test_invalid_tree_and_capacity(impl):
    prob = make_case(3, 16, 8, 2, 128, 256, "bf16", 31, cache_len=[10, 20, 30])
    prob.parent[1, 5] = 9          # forward reference -> status 2, o[1] = 0
    o, st = run_gpu(prob, impl=binding.STREE_SCAN_SIMT if impl == "simt" else binding.STREE_SCAN_AUTO)
    assert st == 2
    assert not o[1].any()
    ref, _ = run_oracle(prob)
    check(o[[0, 2]], ref[[0, 2]], TOL_BF16)
    prob2 = make_case(2, 16, 8, 2, 128, 256, "bf16", 32, cache_len=[10, 20])
    prob2.cache_len[0] = 257       # beyond the cache capacity -> status 5, o[0] = 0
    o2, st2 = run_gpu(prob2, impl=binding.STREE_SCAN_SIMT if impl == "simt" else binding.STREE_SCAN_AUTO)
    assert st2 == 5 and not o2[0].any()


# ---------------------------------------------------------------------------
# KV commit: bit-exact
# ---------------------------------------------------------------------------
def _accepted_paths(par_b, rng, T, deepest=()):
    B = par_b.shape[0]
    path = np.full((B, T), -1, np.int32)
    plen = np.zeros(B, np.int32)
    for b in range(B):
        node = int(rng.integers(0, T)) if b not in deepest else T - 1
        p = [node]
        while par_b[b][p[-1]] >= 0:
            p.append(int(par_b[b][p[-1]]))
        p = p[::-1]
        path[b, :len(p)] = p
        plen[b] = len(p)
    return path, plen


@pytest.mark.parametrize("io,D,Hkv", [("bf16", 128, 8), ("f32", 128, 2), ("bf16", 4, 1), ("f32", 4, 1)])
def test_kv_commit_bitexact(io, D, Hkv):
    rng = np.random.default_rng(41)
    T, S, B = 24, 64, 4
    prob = make_case(B, T, Hkv, Hkv, D, S, io, 41, cache_len=[0, 10, 50, 62])
    path, plen = _accepted_paths(prob.parent, rng, T, deepest=(3,))
    assert plen[3] >= 3              # 62 + path_len > 64: overflow -> status 5, tree 3 unchanged
    kn, vn, kc, vc = (_dev(prob, n) for n in ("k_new", "v_new", "k_cache", "v_cache"))
    cl = torch.from_numpy(prob.cache_len.astype(np.int32)).cuda()
    par = torch.from_numpy(prob.parent).cuda()
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    binding.stree_kv_commit(kn, vn, par, torch.from_numpy(path).cuda(), torch.from_numpy(plen).cuda(), kc, vc, cl,
                            dev_status=st)
    torch.cuda.synchronize()
    rk, rv, rcl, rst = oattn.kv_commit(_f64(prob, "k_new"), _f64(prob, "v_new"), _f64(prob, "k_cache"),
                                       _f64(prob, "v_cache"), prob.cache_len, path, plen, parent=prob.parent)
    assert int(st.item()) == int(rst.max())
    np.testing.assert_array_equal(cl.cpu().numpy(), rcl)
    np.testing.assert_array_equal(kc.float().cpu().numpy().astype(np.float64), rk)
    np.testing.assert_array_equal(vc.float().cpu().numpy().astype(np.float64), rv)


def test_kv_commit_invalid_path():
    prob = make_case(2, 8, 2, 2, 128, 32, "bf16", 43, kind="heap", cache_len=[3, 4])
    path = np.full((2, 8), -1, np.int32)
    path[0, :3] = [0, 2, 3]          # 3 is not a child of 2 -> status 3, tree 0 unchanged
    path[1, :2] = [0, 1]
    plen = np.array([3, 2], np.int32)
    kn, vn, kc, vc = (_dev(prob, n) for n in ("k_new", "v_new", "k_cache", "v_cache"))
    kc0 = kc.clone()
    cl = torch.from_numpy(prob.cache_len.astype(np.int32)).cuda()
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    binding.stree_kv_commit(kn, vn, torch.from_numpy(prob.parent).cuda(), torch.from_numpy(path).cuda(),
                            torch.from_numpy(plen).cuda(), kc, vc, cl, dev_status=st)
    torch.cuda.synchronize()
    assert int(st.item()) == 3
    assert cl.cpu().tolist() == [3, 6]
    assert torch.equal(kc[0], kc0[0])
    assert torch.equal(kc[1, 4], kn[1, 0]) and torch.equal(kc[1, 5], kn[1, 1])


def test_verify_commit_decode_matches_oracle():
    """tree attention -> commit of an accepted path -> one-node decode, all on the GPU, equals the oracle
    chain (which is itself pinned to decode-from-scratch)."""
    rng = np.random.default_rng(51)
    prob = make_case(4, 32, 32, 8, 128, 1024, "bf16", 51, cache_len=[900, 0, 128, 513])
    path, plen = _accepted_paths(prob.parent, rng, 32)
    q, kn, vn, kc, vc = (_dev(prob, n) for n in ("q", "k_new", "v_new", "k_cache", "v_cache"))
    cl = torch.from_numpy(prob.cache_len.astype(np.int32)).cuda()
    par = torch.from_numpy(prob.parent).cuda()
    binding.stree_kv_commit(kn, vn, par, torch.from_numpy(path).cuda(), torch.from_numpy(plen).cuda(), kc, vc, cl)
    nxt = make_case(4, 1, 32, 8, 128, 1024, "bf16", 52, cache_len=[0, 0, 0, 0])
    q2, kn2, vn2 = (_dev(nxt, n) for n in ("q", "k_new", "v_new"))
    o2 = torch.empty_like(q2)
    binding.stree_tree_attn(q2, kn2, vn2, kc, vc, cl, torch.from_numpy(nxt.parent).cuda(), nxt.scale, o2)
    torch.cuda.synchronize()
    rk, rv, rcl, _ = oattn.kv_commit(_f64(prob, "k_new"), _f64(prob, "v_new"), _f64(prob, "k_cache"),
                                     _f64(prob, "v_cache"), prob.cache_len, path, plen, parent=prob.parent)
    ref, _ = oattn.tree_attn(_f64(nxt, "q"), _f64(nxt, "k_new"), _f64(nxt, "v_new"), rk, rv, rcl, nxt.parent,
                             nxt.scale)
    check(o2.float().cpu().numpy().astype(np.float64), ref, TOL_BF16)


def test_early_kv_prefetch_flag():
    """STREE_LAUNCH_EARLY_STATE: the first K/V tiles stream before the PDL wait (decode-loop promise);
    results unchanged, and an invalid tree still drains its early loads and reports."""
    binding.stree_set_launch_flags(binding.STREE_LAUNCH_PDL | binding.STREE_LAUNCH_EARLY_STATE)
    try:
        prob = make_case(3, 64, 32, 8, 128, 1024, "bf16", 61, cache_len=[1000, 129, 0])
        o, st = run_gpu(prob, expect_kernel=2)
        ref, _ = run_oracle(prob)
        assert st == 0
        check(o, ref, TOL_BF16)
        prob.parent[0, 3] = 7
        o, st = run_gpu(prob, expect_kernel=2)
        assert st == 2 and not o[0].any()
        check(o[1:], ref[1:], TOL_BF16)
    finally:
        binding.stree_set_launch_flags(binding.STREE_LAUNCH_PDL)


def test_tc_128key_kernel_still_matches(tmp_path):
    """The default tcgen05 kernel is the 64-key double-buffered one (attn_db_kernel); the 128-key kernel stays
    selectable (STREE_ATTN_DB=0, read once per process), so check it in a child process."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, tests.test_attn_gpu as t\n"
        "from paper_2505_14969_b200 import binding\n"
        "binding.lib()\n"
        "for seed, (B, T, L) in enumerate([(2, 64, 900), (3, 37, 0), (1, 200, 300)]):\n"
        "    p = t.make_case(B, T, 32, 8, 128, 1280, 'bf16', 40 + seed, cache_len=[L] * B)\n"
        "    o, st = t.run_gpu(p)\n"
        "    ref, _ = t.run_oracle(p)\n"
        "    assert st == 0\n"
        "    t.check(o, ref, t.TOL_BF16)\n"
        "print('ok')\n")
    env = dict(os.environ, STREE_ATTN_DB="0")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("flags", [1 | 2, 1 | 2 | 8])
def test_attn_chain_under_launch_promises(flags):
    """A chain of dependent calls: each call's q is the previous call's output, written by the kernel right before
    it.  Under EARLY_STATE (K/V prefetch) + EARLY_TREE (tree validation before the dependency wait) q must still
    be read after the wait; parity with the oracle chain proves it."""
    binding.stree_set_launch_flags(flags)
    try:
        prob = make_case(3, 64, 32, 8, 128, 1024, "bf16", 71, cache_len=[900, 64, 0])
        q, kn, vn, kc, vc = (_dev(prob, n) for n in ("q", "k_new", "v_new", "k_cache", "v_cache"))
        cl = torch.from_numpy(prob.cache_len.astype(np.int32)).cuda()
        par = torch.from_numpy(prob.parent.astype(np.int32)).cuda()
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        outs = [q]
        for _ in range(3):
            o = torch.empty_like(q)
            binding.stree_tree_attn(outs[-1], kn, vn, kc, vc, cl, par, prob.scale, o, dev_status=st)
            outs.append(o)
        torch.cuda.synchronize()
        assert int(st.item()) == 0
        qi = _f64(prob, "q")
        for i in range(3):
            ref, _ = oattn.tree_attn(qi, _f64(prob, "k_new"), _f64(prob, "v_new"), _f64(prob, "k_cache"),
                                     _f64(prob, "v_cache"), prob.cache_len, prob.parent, prob.scale)
            got = outs[i + 1].float().cpu().numpy().astype(np.float64)
            check(got, ref, TOL_BF16)
            qi = got   # the next call reads exactly what this one wrote (bf16 values)
    finally:
        binding.stree_set_launch_flags(binding.STREE_LAUNCH_PDL)


@pytest.mark.parametrize("kernel_env", ["1", "0"])
def test_online_softmax_rescale_mid_stream(kernel_env):
    """Key tiles whose scores jump far above the running row max (x16 in the score scale, i.e. > 8 in log2
    units) after the first tiles: the lazy O rescale must run mid-stream — in K7b it first waits for the one
    P·V that can still be accumulating into O.  Run for both tcgen05 kernels (the 128-key one in a child
    process: the kernel choice is read once per process)."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, tests.test_attn_gpu as t\n"
        "from gen.attn import _io\n"
        "from paper_2505_14969_b200 import binding\n"
        "binding.lib()\n"
        "for seed, (T, L) in enumerate([(64, 700), (33, 130), (200, 90)]):\n"
        "    p = t.make_case(2, T, 32, 8, 128, 1280, 'bf16', 80 + seed, cache_len=[L, L // 2])\n"
        "    kc = p.as_f32('k_cache').copy()\n"
        "    for b in range(2):\n"
        "        hot = slice(int(p.cache_len[b]) // 2, int(p.cache_len[b]))\n"
        "        kc[b, hot] *= 16.0                    # later prefix keys: scores x16\n"
        "    p.k_cache = _io(kc, 'bf16')\n"
        "    o, st = t.run_gpu(p)\n"
        "    ref, _ = t.run_oracle(p)\n"
        "    assert st == 0 and np.isfinite(o).all()\n"
        "    t.check(o, ref, t.TOL_BF16)\n"
        "print('ok')\n")
    env = dict(os.environ, STREE_ATTN_DB=kernel_env)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
