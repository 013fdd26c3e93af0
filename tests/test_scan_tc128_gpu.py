"""GPU parity of the 128-row-tile tcgen05 scan kernel (stree_scan_tc128.cu: 64 < T <= 256 — one tile up to
128 nodes, two row tiles above —, bf16, P = 64, N = 128; BASELINE configs[4] sweep range) against the fp64
oracle, through the C ABI."""
import numpy as np
import pytest
import torch

import oracle
from gen import inputs, trees
from tests.helpers import TOL_BF16, assert_y_close

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


def run(prob, h0=True):
    t = api.upload(prob)
    if not h0:
        t["h0"] = None
    dims = binding.make_dims(t["x"], t["Bm"])
    assert binding.stree_scan_kernel_for(dims) == 3
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    y = torch.full_like(t["x"], float("nan"))
    binding.stree_tree_scan(t["x"], t["dt"], t["A"], t["Bm"], t["Cm"], t["D"], t["h0"], t["parent"], y, st)
    torch.cuda.synchronize()
    return y.float().cpu().numpy(), int(st.item())


def _trees(kind, B, T, seed):
    rng = np.random.default_rng(seed)
    mk = {"random": lambda: trees.random_recursive(T, 4, rng), "heap2": lambda: trees.heap_kary(T, 2),
          "heap8": lambda: trees.heap_kary(T, 8), "chain": lambda: trees.chain(T), "star": lambda: trees.star(T)}[kind]
    return np.stack([mk() for _ in range(B)])


@pytest.mark.parametrize("B,T,H,G,kind", [(2, 65, 8, 1, "random"), (3, 80, 12, 1, "heap2"), (2, 100, 24, 2, "chain"),
                                          (1, 127, 80, 1, "heap8"), (4, 128, 16, 1, "random"), (2, 96, 30, 3, "star"),
                                          (16, 128, 80, 1, "heap2"), (2, 129, 8, 1, "random"),
                                          (3, 200, 12, 1, "heap2"), (2, 256, 16, 2, "chain"), (2, 256, 8, 1, "heap8"),
                                          (1, 170, 80, 1, "star"), (4, 256, 80, 1, "random")])
def test_tc128_matches_oracle(B, T, H, G, kind):
    prob = inputs.make_problem(inputs.Dims(B, T, H, 64, 128, G, "bf16"), _trees(kind, B, T, T + H), seed=T * 7 + H)
    y, st = run(prob)
    ref, _ = oracle.scan_problem(prob)
    assert st == 0
    assert_y_close(y, ref, TOL_BF16)


@pytest.mark.parametrize("variant", ["stress_decay", "mixed_decay", "no_decay", "large_x", "h0_none", "D_none"])
@pytest.mark.parametrize("T", [112, 240])
def test_tc128_stress(variant, T):
    d = inputs.Dims(2, T, 8, 64, 128, 1, "bf16")
    par = np.stack([trees.heap_kary(T, 2), trees.chain(T)])
    # mixed_decay: per-head A·dt spans factorised, chunk-rebased and direct-decay heads in one CTA
    kw = dict(stress_decay=dict(dt_range=(0.5, 1.0), A_range=(16.0, 16.0)),
              mixed_decay=dict(dt_range=(0.2, 1.0), A_range=(0.05, 16.0)), no_decay=dict(dt_range=(1e-6, 1e-5)),
              large_x=dict(x_scale=100.0), h0_none=dict(h0_zero=True), D_none=dict(D_none=True)).get(variant, {})
    prob = inputs.make_problem(d, par, seed=99, **kw)
    y, st = run(prob, h0=variant != "h0_none")
    ref, _ = oracle.scan_problem(prob)
    assert st == 0
    assert_y_close(y, ref, TOL_BF16)


@pytest.mark.parametrize("T,bad_node", [(90, 40), (220, 180)])
def test_tc128_invalid_tree_zero_and_status(T, bad_node):
    prob = inputs.make_problem(inputs.Dims(3, T, 8, 64, 128, 1, "bf16"), _trees("random", 3, T, 5), seed=5)
    prob.parent[1, bad_node] = bad_node + 5
    y, st = run(prob)
    assert st == 2
    assert not y[1].any()
    ref, _ = oracle.scan_problem(prob)
    assert_y_close(y[[0, 2]], ref[[0, 2]], TOL_BF16)
