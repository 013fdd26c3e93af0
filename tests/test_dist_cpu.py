"""Multi-process (gloo, world_size 2, CPU) tests of the sharding plumbing used by
bench.py --gpus N: shard plans, the head all-gather layout and max-over-ranks."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_14969_b200 import dist as sd


def test_shard_ranges_cover_exactly():
    for n in (0, 1, 7, 16, 80):
        for w in (1, 2, 3, 4, 8):
            spans = [sd.shard_range(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def test_shard_heads_groups():
    assert [sd.shard_heads(80, 1, 8, r) for r in range(8)] == [(10 * r, 10 * r + 10) for r in range(8)]
    assert [sd.shard_heads(24, 4, 2, r) for r in range(2)] == [(0, 12), (12, 24)]
    with pytest.raises(ValueError):
        sd.shard_heads(8, 2, 3, 1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, T, H, P = 3, 5, 8, 4
        full = torch.arange(B * T * H * P, dtype=torch.float32).reshape(B, T, H, P)
        lo, hi = sd.shard_heads(H, 1, world, rank)
        g = sd.gather_heads(full[:, :, lo:hi])
        recon = torch.cat(list(g), dim=2)
        ok_gather = torch.equal(recon, full) and torch.equal(sd.heads_to_layer(g), full)
        # the bench's head-sharded full-y plumbing, NCCL-fallback mode (gloo here): layer buffers filled by gather
        fy = sd.FullY(2, B, T, H, P, torch.float32, "cpu", prefer_p2p=False)
        for layer in range(2):
            fy.gather(layer, (full + layer)[:, :, lo:hi].contiguous())
        ok_gather = ok_gather and fy.mode == "nccl" and all(torch.equal(fy.buf[l], full + l) for l in range(2))
        ok_gather = ok_gather and fy.peers(1) == [fy.buf[1].data_ptr()]
        m = sd.max_over_ranks(1.5 + rank, "cpu")
        blo, bhi = sd.shard_range(16, world, rank)
        q.put((rank, ok_gather, m, (blo, bhi)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_and_max():
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [True, True]
    assert [r[2] for r in res] == [2.5, 2.5]
    assert [r[3] for r in res] == [(0, 8), (8, 16)]


def _scan_worker(rank, world, port, q):
    """Head-sharded layer on the CPU oracle: each rank scans its shard of heads (with its groups' B / C), the
    shards are all-gathered over gloo and re-laid out as [B][T][H][P] — must equal the unsharded scan."""
    import numpy as np

    import oracle
    from gen import inputs, trees
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)
        B, T, H, P, N, G = 2, 9, 8, 4, 8, 2
        par = np.stack([trees.random_recursive(T, 3, rng) for _ in range(B)])
        prob = inputs.make_problem(inputs.Dims(B, T, H, P, N, G, "f32"), par, seed=21)
        y_full, _ = oracle.tree_scan(prob.x, prob.dt, prob.A, prob.Bm, prob.Cm, prob.D, prob.h0, par, n_groups=G)
        lo, hi = sd.shard_heads(H, G, world, rank)
        hpg = H // G
        glo, ghi = lo // hpg, hi // hpg   # the shard's groups (heads of a group are contiguous, never split)
        y_sh, _ = oracle.tree_scan(prob.x[:, :, lo:hi], prob.dt[:, :, lo:hi], prob.A[lo:hi], prob.Bm[:, :, glo:ghi],
                                   prob.Cm[:, :, glo:ghi], prob.D[lo:hi], prob.h0[:, lo:hi], par, n_groups=ghi - glo)
        g = sd.gather_heads(torch.from_numpy(np.ascontiguousarray(y_sh)))
        y = sd.heads_to_layer(g).numpy()
        q.put((rank, bool(np.array_equal(y, y_full)), (lo, hi)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_head_sharded_scan_equals_unsharded():
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_scan_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [True, True]
    assert [r[2] for r in res] == [(0, 4), (4, 8)]
