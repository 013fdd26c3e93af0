"""Input generators: bf16 storage format and tree-shape contracts (CPU)."""
import numpy as np
import torch

from gen import inputs, trees


def test_bf16_rne_matches_torch():
    rng = np.random.default_rng(0)
    a = np.concatenate([rng.standard_normal(10000).astype(np.float32) * 10.0 ** rng.integers(-30, 30, 10000),
                        np.array([0.0, -0.0, 1.0, 65504.0, 3.0e38, 1e-40], np.float32)]).astype(np.float32)
    bits = inputs.f32_to_bf16_bits(a)
    ref = torch.from_numpy(a).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(bits, ref)
    back = inputs.bf16_bits_to_f32(bits)
    assert np.array_equal(back, torch.from_numpy(a).to(torch.bfloat16).float().numpy())


def test_tree_generators_topological():
    rng = np.random.default_rng(1)
    cases = [trees.heap_kary(64, 2), trees.heap_kary(256, 8), trees.chain(256), trees.star(9),
             trees.beam(5, 16, rng), trees.random_recursive(64, 4, rng)] + \
            [trees.static_tree(n) for n in "ABCDE"] + [p for _, p in inputs.sweep_cases()]
    for p in cases:
        assert p.dtype == np.int32 and p[0] == -1
        assert all(0 <= p[i] < i for i in range(1, len(p)))


def test_config_shapes():
    for cfg, shp in (("c1", (1, 7, 1, 4, 4)), ("c2", (1, 32, 24, 64, 128)),
                     ("c3", (1, 64, 80, 64, 128)), ("c4", (16, 64, 80, 64, 128))):
        d, par = inputs.config_trees(cfg, 0)
        assert (d.batch, d.n_nodes, d.n_heads, d.head_dim, d.d_state) == shp
        assert par.shape == (d.batch, d.n_nodes)
    p = inputs.config_problem("c1")
    assert p.x.dtype == np.float32 and p.dims.io_dtype == "f32"
    p = inputs.config_problem("c2")
    assert p.x.dtype == np.uint16 and p.x.shape == (1, 32, 24, 64) and p.h0.shape == (1, 24, 64, 128)
    assert (p.A < 0).all() and (p.dt > 0).all() and p.dt.max() <= 0.1
