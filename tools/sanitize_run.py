"""Driver for compute-sanitizer (memcheck / racecheck / synccheck): one small call of every kernel family
on cuda:0, each checked against the oracle, so a sanitizer run also proves the results are right.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [--quick]

Kernels exercised (include/stree.h names): build_mask, accept, tree_scan (SIMT fp32 c1; small-batch c2;
tcgen05 pipeline K2 at B=16; 128-row K2b at T=256 chain), commit (TMA pipeline, ring), replay_scan (fused
small-batch and K2, with the EARLY launch promises), tree_conv + conv_commit, tree_attn (tcgen05) +
kv_commit, accept_mss."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from gen import inputs, trees  # noqa: E402
from paper_2505_14969_b200 import api, binding  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))


def check(name, err, tol):
    ok = err <= tol
    print(f"{name:34s} rel-err {err:.2e} (tol {tol:.0e}) {'ok' if ok else 'FAIL'}", flush=True)
    if not ok:
        raise SystemExit(f"{name}: rel-err {err} > {tol}")


def scan_case(name, prob, tol, impl=binding.STREE_SCAN_AUTO, flags=binding.STREE_LAUNCH_PDL, h0=True):
    binding.stree_set_scan_impl(impl)
    binding.stree_set_launch_flags(flags)
    try:
        t = api.upload(prob)
        if not h0:
            t["h0"] = None
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        y = api.tree_scan(t, st)
        torch.cuda.synchronize()
    finally:
        binding.stree_set_scan_impl(binding.STREE_SCAN_AUTO)
        binding.stree_set_launch_flags(binding.STREE_LAUNCH_PDL)
    ry, _ = oracle.scan_problem(prob)
    assert st.item() == 0
    check(name, rel(y.float().cpu().numpy(), ry), tol)
    return t


def replay_case(name, B, Tp, T, H, flags, impl=binding.STREE_SCAN_AUTO, seed=7):
    rng = np.random.default_rng(seed)
    pp = np.stack([trees.random_recursive(Tp, 3, rng) for _ in range(B)])
    pn = np.stack([trees.random_recursive(T, 4, rng) for _ in range(B)])
    prev = inputs.make_problem(inputs.Dims(B, Tp, H, 64, 128, 1, "bf16"), pp, seed=seed)
    new = inputs.make_problem(inputs.Dims(B, T, H, 64, 128, 1, "bf16"), pn, seed=seed + 1)
    new.A, new.D, new.h0 = prev.A, prev.D, prev.h0
    tok, vt = inputs.make_accept_inputs(pp, seed=seed + 2, p_match=0.9)
    path, plen, _, _ = oracle.accept(tok, pp, vt)
    binding.stree_set_scan_impl(impl)
    binding.stree_set_launch_flags(flags)
    try:
        tp, tn = api.upload(prev), api.upload(new)
        h = tp["h0"].clone()
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        y = api.replay_scan(tp, torch.from_numpy(path).cuda(), torch.from_numpy(plen).cuda(), tn, h, dev_status=st)
        torch.cuda.synchronize()
    finally:
        binding.stree_set_scan_impl(binding.STREE_SCAN_AUTO)
        binding.stree_set_launch_flags(binding.STREE_LAUNCH_PDL)
    hk, _ = oracle.commit_problem(prev, path, plen)
    ry, _ = oracle.tree_scan(new.io_as_f32("x"), new.dt, new.A, new.io_as_f32("Bm"), new.io_as_f32("Cm"), new.D, hk,
                             new.parent)
    assert st.item() == 0
    check(name + " h", rel(h.cpu().numpy(), hk), 1e-4)
    check(name + " y", rel(y.float().cpu().numpy(), ry), 2e-2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="scan kernels only")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    binding.lib()
    all_flags = (binding.STREE_LAUNCH_PDL | binding.STREE_LAUNCH_EARLY_STATE | binding.STREE_LAUNCH_EARLY_REPLAY |
                 binding.STREE_LAUNCH_EARLY_TREE | binding.STREE_LAUNCH_EARLY_DT)
    # c1 toy (SIMT fp32), c2 (small-batch tcgen05), mask + accept + commit on c2
    scan_case("scan c1 (simt fp32)", inputs.config_problem("c1"), 1e-4)
    p2 = inputs.config_problem("c2")
    t2 = scan_case("scan c2 (small-batch)", p2, 2e-2)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    mask, depth = api.build_mask(t2["parent"], st)
    rm, rd, _ = oracle.build_mask(p2.parent)
    assert np.array_equal(mask.cpu().numpy().view(np.uint32), rm) and np.array_equal(depth.cpu().numpy(), rd)
    print("mask c2                            bit-exact ok", flush=True)
    tok, vt = inputs.make_accept_inputs(p2.parent, seed=11, p_match=0.9)
    path, plen, bonus = api.accept(torch.from_numpy(tok).cuda(), t2["parent"], torch.from_numpy(vt).cuda(), st)
    rp, rl, rb, _ = oracle.accept(tok, p2.parent, vt)
    assert np.array_equal(path.cpu().numpy(), rp) and np.array_equal(plen.cpu().numpy(), rl)
    print("accept c2                          bit-exact ok", flush=True)
    h_new = api.commit(t2, path, plen, dev_status=st)
    torch.cuda.synchronize()
    rh, _ = oracle.commit_problem(p2, rp, rl)
    check("commit c2", rel(h_new.cpu().numpy(), rh), 1e-4)
    # K2 pipeline at B = 16, T = 64 (fewer heads than the bench, same kernel)
    d4 = inputs.Dims(16, 64, 16, 64, 128, 1, "bf16")
    rng = np.random.default_rng(5)
    p4 = inputs.make_problem(d4, np.stack([trees.random_recursive(64, 4, rng) for _ in range(16)]), seed=5)
    scan_case("scan B16 T64 (tcgen05 pipeline)", p4, 2e-2, binding.STREE_SCAN_TC_PIPELINE)
    # K2b: a 256-node chain (two 128-row tiles, direct decay)
    d5 = inputs.Dims(1, 256, 8, 64, 128, 1, "bf16")
    scan_case("scan T256 chain (tcgen05 128-row)", inputs.make_problem(d5, trees.chain(256)[None], seed=9), 2e-2)
    # K2b one tile (T <= 128): factorised, rebased and direct heads in one CTA; every EARLY promise; no h0
    d6 = inputs.Dims(2, 112, 12, 64, 128, 1, "bf16")
    p6 = inputs.make_problem(d6, np.stack([trees.heap_kary(112, 2), trees.chain(112)]), seed=13, dt_range=(0.2, 1.0),
                             A_range=(0.05, 16.0))
    scan_case("scan T112 mixed decay (128-row, early)", p6, 2e-2, flags=all_flags)
    p7 = inputs.make_problem(d6, p6.parent, seed=14, dt_range=(0.2, 1.0), A_range=(0.05, 16.0), h0_zero=True)
    scan_case("scan T112 mixed decay (128-row, no h0)", p7, 2e-2, h0=False)
    # fused replay + scan: small-batch and pipeline kernels, every EARLY promise
    replay_case("replay_scan B2 H16 (small-batch)", 2, 48, 40, 16, all_flags)
    replay_case("replay_scan B2 H16 (small-batch, PDL only)", 2, 48, 40, 16, binding.STREE_LAUNCH_PDL)
    replay_case("replay_scan B1 H80 (small-batch, c3)", 1, 64, 64, 80, all_flags)
    replay_case("replay_scan B16 H8 (pipeline)", 16, 64, 64, 8, all_flags, binding.STREE_SCAN_TC_PIPELINE)
    if args.quick:
        return
    # tree conv + conv commit, tree attention + KV commit, MSS (the §8(f) rows), via their own test helpers
    import pytest
    rc = pytest.main(["-q", "-x", "-p", "no:cacheprovider", "-m", "gpu",
                      "tests/test_conv_gpu.py", "tests/test_attn_gpu.py", "tests/test_mss_gpu.py", "-k",
                      "(conv_matches_oracle and 264) or conv_commit_bit_exact or bf16_ragged or "
                      "kv_commit_bitexact or (random_trees and 1000) or (launch_promises and 37)"])
    if rc != 0:
        raise SystemExit(f"§8(f) tests failed under the sanitizer (pytest rc {rc})")


if __name__ == "__main__":
    main()
