"""GPU parity of the tree-causal depthwise conv1d and its conv-state commit (SURVEY §8(f) NEXT #2,
DESIGN.md reading R-conv) against the fp64 oracle, through the C ABI."""
import numpy as np
import pytest
import torch

import oracle
from gen import inputs, trees
from tests.helpers import TOL_BF16, TOL_F32, assert_conv_close

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2505_14969_b200 import binding


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    binding.lib()
    yield


MAMBA2_CONV = 80 * 64 + 2 * 128   # conv_dim of the 2.7B shape: H*P + 2*G*N = 5376


def make_conv(B, T, C, W, io, seed, kind="random", with_state=True, with_bias=True):
    """Seeded conv inputs: u ~ N(0,1) in the io dtype (bf16 = RNE), weight ~ U(-1/sqrt(W), 1/sqrt(W))
    (nn.Conv1d default init range), bias ~ same, state ~ N(0,1)."""
    rng = np.random.default_rng(seed)
    mk = {"random": lambda: trees.random_recursive(T, 4, rng), "chain": lambda: trees.chain(T),
          "heap": lambda: trees.heap_kary(T, 2)}[kind]
    par = np.stack([mk() for _ in range(B)]).astype(np.int32)
    lim = 1.0 / np.sqrt(W)
    u = rng.standard_normal((B, T, C)).astype(np.float32)
    weight = rng.uniform(-lim, lim, (C, W)).astype(np.float32)
    bias = rng.uniform(-lim, lim, C).astype(np.float32) if with_bias else None
    state = rng.standard_normal((B, W - 1, C)).astype(np.float32) if (with_state and W > 1) else None
    if io == "bf16":
        u = inputs.bf16_bits_to_f32(inputs.f32_to_bf16_bits(u))
        if state is not None:
            state = inputs.bf16_bits_to_f32(inputs.f32_to_bf16_bits(state))
    return par, u, weight, bias, state


def dev(a, io=None):
    if a is None:
        return None
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t.to(torch.bfloat16) if io == "bf16" else t


def run_conv(par, u, weight, bias, state, io, act=True):
    ud = dev(u, io)
    out = torch.empty_like(ud)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    binding.stree_tree_conv(ud, dev(weight), dev(bias), dev(state, io), dev(par), out, act=act, dev_status=st)
    torch.cuda.synchronize()
    return out.float().cpu().numpy(), int(st.item())


@pytest.mark.parametrize("shape", [(16, 64, MAMBA2_CONV, 4), (3, 37, 264, 4), (2, 256, 520, 3), (4, 1, 64, 2),
                                   (2, 19, 128, 1), (1, 200, 1024, 4)])
@pytest.mark.parametrize("io", ["bf16", "f32"])
def test_tree_conv_matches_oracle(shape, io):
    B, T, C, W = shape
    par, u, weight, bias, state = make_conv(B, T, C, W, io, seed=T * 3 + C + W)
    got, st = run_conv(par, u, weight, bias, state, io)
    ref, rst = oracle.tree_conv(u, weight, bias, state, par)
    assert st == 0 and not rst.any()
    assert_conv_close(got, ref, TOL_BF16 if io == "bf16" else TOL_F32)


@pytest.mark.parametrize("kind", ["chain", "heap"])
@pytest.mark.parametrize("act,with_state,with_bias", [(False, True, True), (True, False, False)])
def test_tree_conv_variants(kind, act, with_state, with_bias):
    B, T, C, W = 3, 64, 256, 4
    par, u, weight, bias, state = make_conv(B, T, C, W, "f32", seed=5, kind=kind, with_state=with_state,
                                            with_bias=with_bias)
    got, st = run_conv(par, u, weight, bias, state, "f32", act=act)
    ref, _ = oracle.tree_conv(u, weight, bias, state, par, act=act)
    assert_conv_close(got, ref, TOL_F32)


def test_tree_conv_invalid_tree_zero_and_status():
    B, T, C, W = 3, 32, 128, 4
    par, u, weight, bias, state = make_conv(B, T, C, W, "bf16", seed=7)
    par[1, 9] = 20
    got, st = run_conv(par, u, weight, bias, state, "bf16")
    assert st == 2 and not got[1].any()
    ref, rst = oracle.tree_conv(u, weight, bias, state, par)
    assert list(rst) == [0, 2, 0]
    assert_conv_close(got[[0, 2]], ref[[0, 2]], TOL_BF16)
    par[2, 0] = 3
    _, st = run_conv(par, u, weight, bias, state, "bf16")
    assert st in (1, 2)


def run_commit(u, state, par, path, plen, W, io, inplace=False, use_parent=True):
    ud, sd = dev(u, io), dev(state, io)
    new = sd if inplace else (torch.empty_like(sd) if sd is not None else
                              torch.empty((u.shape[0], W - 1, u.shape[2]), dtype=ud.dtype, device="cuda"))
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    binding.stree_conv_commit(ud, sd, dev(par) if use_parent else None, dev(path), dev(plen), new, W, dev_status=st)
    torch.cuda.synchronize()
    return new.float().cpu().numpy(), int(st.item())


@pytest.mark.parametrize("io", ["bf16", "f32"])
@pytest.mark.parametrize("inplace", [False, True])
def test_conv_commit_bit_exact(io, inplace):
    B, T, C, W = 16, 64, MAMBA2_CONV, 4
    par, u, weight, bias, state = make_conv(B, T, C, W, io, seed=11)
    tok, vt = inputs.make_accept_inputs(par, seed=12, p_match=0.7)
    path, plen, _, _ = oracle.accept(tok, par, vt)
    # the paths mix lengths shorter than, equal to and longer than the W - 1 state rows
    assert (plen < W - 1).any() and (plen >= W - 1).any()
    got, st = run_commit(u, state, par, path, plen, W, io, inplace=inplace)
    ref, rst = oracle.conv_commit(u, state, path, plen, W, parent=par)
    assert st == 0 and not rst.any()
    assert np.array_equal(got, ref.astype(np.float32))        # a copy: bit-exact


def test_conv_commit_short_paths_invalid_and_null_state():
    B, T, C, W = 4, 16, 64, 4
    par, u, weight, bias, state = make_conv(B, T, C, W, "bf16", seed=13, kind="chain")
    path = np.full((B, T), -1, np.int32)
    plen = np.array([1, 2, 16, 3], np.int32)
    for b in range(B):
        path[b, : plen[b]] = np.arange(plen[b])
    path[3, 2] = 5                                            # not parent-linked
    got, st = run_commit(u, state, par, path, plen, W, "bf16")
    ref, rst = oracle.conv_commit(u, state, path, plen, W, parent=par)
    assert st == 3 and list(rst) == [0, 0, 0, 3]
    assert np.array_equal(got, ref.astype(np.float32))
    got2, _ = run_commit(u, None, par, path, plen, W, "bf16", use_parent=False)
    ref2, _ = oracle.conv_commit(u, None, path, plen, W)
    assert np.array_equal(got2, ref2.astype(np.float32))


def test_conv_two_iterations_equal_grafted_tree():
    """conv(tree2, state = conv_commit(tree1)) on the GPU equals the oracle conv of tree2 grafted under
    the last accepted node of tree1 (the conv analogue of Alg. 1's losslessness)."""
    C, W = 256, 4
    par1, u1, weight, bias, state = make_conv(1, 24, C, W, "f32", seed=21)
    par2, u2, _, _, _ = make_conv(1, 20, C, W, "f32", seed=22)
    tok, vt = inputs.make_accept_inputs(par1, seed=23, p_match=0.9)
    path, plen, _, _ = oracle.accept(tok, par1, vt)
    s1, _ = run_commit(u1, state, par1, path, plen, W, "f32")
    got, _ = run_conv(par2, u2, weight, bias, s1, "f32")
    k = int(path[0, plen[0] - 1])
    pg = np.concatenate([par1[0], np.where(par2[0] < 0, k, par2[0] + 24)]).astype(np.int32)
    ref, _ = oracle.tree_conv(np.concatenate([u1, u2], 1), weight, bias, state, pg[None])
    assert_conv_close(got[0][None], ref[:, 24:], TOL_F32)


@pytest.mark.parametrize("flags", [1, 1 | 8, 1 | 2 | 8, 31])
@pytest.mark.parametrize("shape", [(16, 64, MAMBA2_CONV, 4), (2, 256, 520, 3), (3, 37, 264, 4), (2, 5, 64, 2)])
def test_tree_conv_launch_promises(flags, shape):
    """EARLY_TREE (weights, bias, parents and windows before the dependency wait) and EARLY_STATE (conv-state
    rows too), as a chain of dependent calls: each layer's input is the previous layer's output (written by the
    kernel immediately before it), so any read of u before the wait would see stale rows."""
    B, T, C, W = shape
    io = "bf16"
    par, u, weight, bias, state = make_conv(B, T, C, W, io, seed=T + C)
    binding.stree_set_launch_flags(flags)
    try:
        L = 4
        bufs = [dev(u, io)] + [torch.empty_like(dev(u, io)) for _ in range(L)]
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        for i in range(L):
            binding.stree_tree_conv(bufs[i], dev(weight), dev(bias), dev(state, io), dev(par), bufs[i + 1], act=True,
                                    dev_status=st)
        torch.cuda.synchronize()
        x = u
        for i in range(L):
            ref, _ = oracle.tree_conv(x, weight, bias, state, par)
            got = bufs[i + 1].float().cpu().numpy()
            assert_conv_close(got, ref, TOL_BF16)
            x = got   # the next layer reads exactly what the kernel wrote (bf16 values)
        assert int(st.item()) == 0
    finally:
        binding.stree_set_launch_flags(1)
