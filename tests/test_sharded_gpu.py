"""Head-sharded layers on one GPU (BASELINE configs[3]: "heads sharded over 2/4/8 GPUs"):
stree_replay_scan_sharded / stree_tree_scan_sharded called once per head shard, every call writing its y
tiles into ALL of n "peer" buffers (here n distinct local buffers standing in for the ranks' full-y
buffers; across GPUs they are peer-mapped symmetric-memory buffers).  After every shard ran, every
buffer must hold the whole layer's y, identical to the unsharded call, and the shards' committed
states must equal the unsharded commit — the all-gather done by the scan epilogue, checked bit for bit
(the per-head arithmetic does not depend on the shard), and against the oracle."""
import numpy as np
import pytest
import torch

import oracle
from gen import inputs, trees
from paper_2505_14969_b200 import dist as sd
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


def _pair(B, Tp, T, H, seed):
    rng = np.random.default_rng(seed)
    pp = np.stack([trees.random_recursive(Tp, 3, rng) for _ in range(B)])
    pn = np.stack([trees.random_recursive(T, 4, rng) for _ in range(B)])
    prev = inputs.make_problem(inputs.Dims(B, Tp, H, 64, 128, 1, "bf16"), pp, seed=seed)
    new = inputs.make_problem(inputs.Dims(B, T, H, 64, 128, 1, "bf16"), pn, seed=seed + 1)
    new.A, new.D, new.h0 = prev.A, prev.D, prev.h0
    tok, vt = inputs.make_accept_inputs(pp, seed=seed + 2, p_match=0.9)
    path, plen, _, _ = oracle.accept(tok, pp, vt)
    return prev, new, path, plen


@pytest.mark.parametrize("B,Tp,T,H,world,impl", [
    (16, 64, 64, 80, 4, "pipeline"),   # BASELINE configs[3] at world 4: the tcgen05 pipeline kernel
    (16, 64, 64, 80, 2, "auto"),
    (1, 64, 64, 80, 2, "auto"),        # batch 1 (configs[2] shape): the small-batch kernel
    (2, 40, 24, 24, 3, "auto"),        # 130M-like head count, 3 shards, ragged trees
])
def test_replay_scan_sharded_equals_unsharded(B, Tp, T, H, world, impl):
    prev, new, path, plen = _pair(B, Tp, T, H, seed=100 + B + world)
    binding.stree_set_scan_impl(binding.STREE_SCAN_TC_PIPELINE if impl == "pipeline" else binding.STREE_SCAN_AUTO)
    tp, tn = api.upload(prev), api.upload(new)
    path_d, plen_d = torch.from_numpy(path).cuda(), torch.from_numpy(plen).cuda()
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    # unsharded reference call
    h_ref = tp["h0"].clone()
    y_ref = api.replay_scan(tp, path_d, plen_d, tn, h_ref, dev_status=st)
    # sharded: every shard writes into every peer buffer
    peers = [torch.full_like(tn["x"], float("nan")) for _ in range(world)]
    h_sh = tp["h0"].clone()
    for r in range(world):
        lo, hi = sd.shard_heads(H, 1, world, r)
        sl = lambda a, dim=2: a.narrow(dim, lo, hi - lo).contiguous()
        hs = h_sh[:, lo:hi].contiguous()
        yo = binding.make_yout(peers, heads_total=H, head_offset=lo)
        binding.stree_replay_scan_sharded(sl(tp["x"]), sl(tp["dt"]), tp["Bm"], tp["parent"], path_d, plen_d,
                                          sl(tn["x"]), sl(tn["dt"]), tn["A"][lo:hi].contiguous(), tn["Bm"], tn["Cm"],
                                          tn["D"][lo:hi].contiguous(), hs, tn["parent"], yo, st)
        h_sh[:, lo:hi] = hs
    torch.cuda.synchronize()
    assert st.item() == 0
    for p in peers:
        assert torch.equal(p.view(torch.int16), y_ref.view(torch.int16)), "peer y != unsharded y"
    assert torch.equal(h_sh, h_ref)
    # and against the oracle (commit then scan)
    hk, _ = oracle.commit_problem(prev, path, plen)
    ry, _ = oracle.tree_scan(new.io_as_f32("x"), new.dt, new.A, new.io_as_f32("Bm"), new.io_as_f32("Cm"), new.D, hk,
                             new.parent)
    assert_h_close(h_sh.cpu().numpy(), hk, TOL_F32)
    assert_y_close(peers[-1].float().cpu().numpy(), ry, TOL_BF16)


def test_tree_scan_sharded_single_peer_offset():
    """One peer, a shard in the middle of a wider layer: only that shard's heads are written."""
    B, T, H, Ht, off = 2, 33, 8, 24, 8
    rng = np.random.default_rng(3)
    prob = inputs.make_problem(inputs.Dims(B, T, H, 64, 128, 1, "bf16"),
                               np.stack([trees.random_recursive(T, 3, rng) for _ in range(B)]), seed=3)
    t = api.upload(prob)
    y_ref = api.tree_scan(t)
    full = torch.zeros((B, T, Ht, 64), dtype=torch.bfloat16, device="cuda")
    yo = binding.make_yout([full], heads_total=Ht, head_offset=off)
    binding.stree_tree_scan_sharded(t["x"], t["dt"], t["A"], t["Bm"], t["Cm"], t["D"], t["h0"], t["parent"], yo)
    torch.cuda.synchronize()
    assert torch.equal(full[:, :, off:off + H].view(torch.int16), y_ref.view(torch.int16))
    assert not full[:, :, :off].any() and not full[:, :, off + H:].any()


def test_full_y_symmetric_memory_one_rank():
    """The bench's P2P plumbing (paper_2505_14969_b200/dist.py FullY) on a one-rank NCCL group: torch
    symmetric memory, peer addresses into stree_replay_scan_sharded, the device barrier that publishes."""
    import os

    import torch.distributed as dist

    from paper_2505_14969_b200 import dist as sdist
    own = not dist.is_initialized()
    if own:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29541")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        B, Tp, T, H, L = 2, 32, 48, 16, 3
        fy = sdist.FullY(L, B, T, H, 64, torch.bfloat16, torch.device("cuda", 0), force_p2p=True)
        if fy.mode != "p2p":
            pytest.skip(f"symmetric memory unavailable: {fy.error}")
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        for layer in range(L):
            prev, new, path, plen = _pair(B, Tp, T, H, seed=40 + layer)
            tp, tn = api.upload(prev), api.upload(new)
            pd, ld = torch.from_numpy(path).cuda(), torch.from_numpy(plen).cuda()
            h_ref = tp["h0"].clone()
            y_ref = api.replay_scan(tp, pd, ld, tn, h_ref, dev_status=st)
            h = tp["h0"].clone()
            yo = binding.make_yout(fy.peers(layer), heads_total=H, head_offset=0)
            binding.stree_replay_scan_sharded(tp["x"], tp["dt"], tp["Bm"], tp["parent"], pd, ld, tn["x"], tn["dt"],
                                              tn["A"], tn["Bm"], tn["Cm"], tn["D"], h, tn["parent"], yo, st)
            fy.publish()
            torch.cuda.synchronize()
            assert torch.equal(fy.buf[layer].view(torch.int16), y_ref.view(torch.int16))
            assert torch.equal(h, h_ref)
        assert st.item() == 0
    finally:
        if own:
            dist.destroy_process_group()
