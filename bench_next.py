"""Measurement of the SURVEY §8(f) rows beyond the SSM step (imported by bench.py; also runnable alone:
``python bench_next.py`` prints one JSON object).

Each row is timed the way the main step is: L back-to-back calls on distinct per-layer buffers
(inputs larger than L2), captured in one CUDA graph, CUDA events on the launching stream, W warm-up
replays, median over K replays; algorithmic bytes per call / time against the measured HBM copy peak.

  tree_attn  stree_tree_attn on the hybrid MambaInLlama-8B attention shape (gen.attn 'hyb8b':
             16 trees x 64 nodes, Hq=32, Hkv=8, D=128, bf16, committed prefixes 768..1280), 32 layers
             (the 50%-attention hybrid of PAPER.md:318 has 32 attention layers)
  kv_commit  stree_kv_commit of the accepted paths of those trees into each layer's cache
  tree_conv  stree_tree_conv on the Mamba-2 2.7B conv (conv_dim 5376 = H*P + 2*G*N, W = 4), c4 trees
  conv_commit stree_conv_commit along the accepted paths
  accept_mss stree_accept_mss (multi-step speculative sampling) on the c4 trees, V = 50,280
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from gen import inputs  # noqa: E402
from gen.attn import attn_config  # noqa: E402


def _graph_time_us(fn, calls, stream, warmup=3, reps=9):
    import torch
    with torch.cuda.stream(stream):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        fn()
    for _ in range(warmup):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        with torch.cuda.stream(stream):
            g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / calls)
    return float(np.median(ts))


def _accepted(parent, seed):
    """Deterministic accepted paths (root to a random node) for each tree."""
    rng = np.random.default_rng(seed)
    B, T = parent.shape
    path = np.full((B, T), -1, np.int32)
    plen = np.zeros(B, np.int32)
    for b in range(B):
        p = [int(rng.integers(0, T))]
        while parent[b][p[-1]] >= 0:
            p.append(int(parent[b][p[-1]]))
        p = p[::-1]
        path[b, :len(p)] = p
        plen[b] = len(p)
    return path, plen


def measure(dev, hbm_peak, bf16_peak, layers_attn=32, layers_ssm=64):
    import torch
    from paper_2505_14969_b200 import binding

    stream = torch.cuda.Stream(device=dev)
    out = {}
    # decode-loop launch promises: a layer's KV cache / conv state and the iteration's tree are not written by the
    # kernel right before it
    binding.stree_set_launch_flags(binding.STREE_LAUNCH_PDL | binding.STREE_LAUNCH_EARLY_STATE |
                                   binding.STREE_LAUNCH_EARLY_TREE)

    # ---------------- tree attention + KV commit ----------------
    prob = attn_config("hyb8b")
    d = prob.dims
    B, T, Hq, Hkv, D, S = d.batch, d.n_nodes, d.n_q_heads, d.n_kv_heads, d.head_dim, d.cache_cap
    gen = torch.Generator(device=dev)
    gen.manual_seed(inputs.BASE_SEED + 500)
    par = torch.from_numpy(prob.parent).to(dev)
    cl0 = torch.from_numpy(prob.cache_len).to(dev)
    bf = torch.bfloat16
    lay = []
    for _ in range(layers_attn):
        lay.append({
            "q": torch.randn((B, T, Hq, D), generator=gen, device=dev).to(bf),
            "kn": torch.randn((B, T, Hkv, D), generator=gen, device=dev).to(bf),
            "vn": torch.randn((B, T, Hkv, D), generator=gen, device=dev).to(bf),
            "kc": torch.randn((B, S, Hkv, D), generator=gen, device=dev).to(bf),
            "vc": torch.randn((B, S, Hkv, D), generator=gen, device=dev).to(bf),
            "o": torch.empty((B, T, Hq, D), dtype=bf, device=dev),
            "cl": cl0.clone(),
        })
    dims = binding.make_attn_dims(lay[0]["q"], lay[0]["kn"], lay[0]["kc"])
    status = torch.zeros(1, dtype=torch.int32, device=dev)

    def attn_all():
        for t in lay:
            binding.stree_tree_attn(t["q"], t["kn"], t["vn"], t["kc"], t["vc"], t["cl"], par, prob.scale, t["o"],
                                    status, dims=dims)

    us = _graph_time_us(attn_all, layers_attn, stream)
    depth = np.zeros((B, T), np.int64)
    for b in range(B):
        for i in range(1, T):
            depth[b, i] = depth[b, prob.parent[b, i]] + 1
    Lsum = int(prob.cache_len.sum())
    abytes = (2 * B * T * Hq * D * 2 + Lsum * Hkv * D * 2 * 2 + B * T * Hkv * D * 2 * 2 + B * T * 4 + B * 4)
    aflops = 4 * D * Hq * int(sum(int(prob.cache_len[b]) * T + int((depth[b] + 1).sum()) for b in range(B)))
    gbs = abytes / (us * 1e-6) / 1e9
    tfs = aflops / (us * 1e-6) / 1e12
    out["tree_attn"] = {"us": us, "bytes": abytes, "GB/s": gbs, "frac": gbs / hbm_peak, "bound": "hbm",
                        "flops": aflops, "TFLOP/s": tfs, "tensor_frac": tfs / bf16_peak,
                        "impl": {1: "simt", 2: "tcgen05"}.get(binding.stree_attn_kernel_for(dims)),
                        "layers": layers_attn,
                        "workload": "hyb8b: 16 trees x 64 nodes, Hq=32 Hkv=8 D=128 bf16, prefix 768..1280"}
    # KV commit (each replay re-commits from the same cache_len: the kernel sees cache_len advance, so reset it
    # inside the graph with a device copy — counted separately, tiny)
    path, plen = _accepted(prob.parent, inputs.BASE_SEED + 501)
    path_d, plen_d = torch.from_numpy(path).to(dev), torch.from_numpy(plen).to(dev)

    def commit_all():
        for t in lay:
            t["cl"].copy_(cl0)
            binding.stree_kv_commit(t["kn"], t["vn"], par, path_d, plen_d, t["kc"], t["vc"], t["cl"], status,
                                    dims=dims)

    us_c = _graph_time_us(commit_all, layers_attn, stream)
    cbytes = int(plen.sum()) * Hkv * D * 2 * 2 * 2
    out["kv_commit"] = {"us": us_c, "bytes": cbytes, "GB/s": cbytes / (us_c * 1e-6) / 1e9,
                        "frac": cbytes / (us_c * 1e-6) / 1e9 / hbm_peak, "bound": "latency",
                        "mean_path_len": float(plen.mean()), "note": "includes a 64-byte cache_len reset copy"}
    del lay
    torch.cuda.empty_cache()

    # ---------------- tree conv + conv commit ----------------
    dd, par_np = inputs.config_trees("c4", inputs.BASE_SEED + 3)
    B, T = par_np.shape
    C, W = 80 * 64 + 2 * 128, 4
    parc = torch.from_numpy(par_np.astype(np.int32)).to(dev)
    cl = []
    for _ in range(layers_ssm):
        cl.append({"u": torch.randn((B, T, C), generator=gen, device=dev).to(bf),
                   "w": torch.rand((C, W), generator=gen, device=dev) - 0.5,
                   "bias": torch.rand((C,), generator=gen, device=dev) - 0.5,
                   "st": torch.randn((B, W - 1, C), generator=gen, device=dev).to(bf),
                   "out": torch.empty((B, T, C), dtype=bf, device=dev)})
    cdims = binding.make_conv_dims(cl[0]["u"], cl[0]["w"])
    # decode-loop promises for the conv (as the scan bench uses them): the tree, the conv weights / bias and the
    # conv state are not written by the kernel right before a layer's conv (EARLY_TREE + EARLY_STATE)
    binding.stree_set_launch_flags(binding.STREE_LAUNCH_PDL | binding.STREE_LAUNCH_EARLY_STATE |
                                   binding.STREE_LAUNCH_EARLY_TREE)

    def conv_all():
        for t in cl:
            binding.stree_tree_conv(t["u"], t["w"], t["bias"], t["st"], parc, t["out"], True, status, dims=cdims)

    us_v = _graph_time_us(conv_all, layers_ssm, stream)
    vbytes = 2 * B * T * C * 2 + B * (W - 1) * C * 2 + C * W * 4 + C * 4 + B * T * 4
    out["tree_conv"] = {"us": us_v, "bytes": vbytes, "GB/s": vbytes / (us_v * 1e-6) / 1e9,
                        "frac": vbytes / (us_v * 1e-6) / 1e9 / hbm_peak, "bound": "hbm", "layers": layers_ssm,
                        "workload": "c4 trees (16 x 64 nodes), conv_dim 5376, W=4, bf16"}
    path, plen = _accepted(par_np, inputs.BASE_SEED + 502)
    path_d, plen_d = torch.from_numpy(path).to(dev), torch.from_numpy(plen).to(dev)
    for t in cl:
        t["st2"] = torch.empty_like(t["st"])

    def conv_commit_all():
        for t in cl:
            binding.stree_conv_commit(t["u"], t["st"], parc, path_d, plen_d, t["st2"], W, status, dims=cdims)

    us_cc = _graph_time_us(conv_commit_all, layers_ssm, stream)
    ccbytes = B * (W - 1) * C * 2 * 2
    out["conv_commit"] = {"us": us_cc, "bytes": ccbytes, "GB/s": ccbytes / (us_cc * 1e-6) / 1e9,
                          "frac": ccbytes / (us_cc * 1e-6) / 1e9 / hbm_peak, "bound": "latency"}
    del cl
    torch.cuda.empty_cache()

    # ---------------- MSS verification (once per iteration) ----------------
    from gen.mss import mss_config
    mp = mss_config("c4")
    md = {k: torch.from_numpy(getattr(mp, k)).to(dev) for k in ("tokens", "parent", "p_target", "q_draft",
                                                                  "u_accept", "u_bonus")}
    B, T = mp.parent.shape
    mpath = torch.empty((B, T), dtype=torch.int32, device=dev)
    mplen = torch.empty((B,), dtype=torch.int32, device=dev)
    mbonus = torch.empty((B,), dtype=torch.int32, device=dev)

    def mss_calls():   # 16 back-to-back calls per graph (idempotent) so the graph launch is amortised
        for _ in range(16):
            binding.stree_accept_mss(md["tokens"], md["parent"], md["p_target"], md["q_draft"], md["u_accept"],
                                     md["u_bonus"], mpath, mplen, mbonus, status)

    us_m = _graph_time_us(mss_calls, 16, stream)
    out["accept_mss"] = {"us": us_m, "bound": "latency", "mean_path_len": float(mplen.float().mean().item()),
                         "workload": "c4 trees (16 x 64 nodes), V=50280, target sigma=3, draft noise 1",
                         "note": "one call per verify iteration; vocab rows touched depend on the rejections"}
    torch.cuda.synchronize()
    assert status.item() == 0, f"device status {status.item()}"
    out["c5_sweep"] = measure_c5()
    k2b = out["c5_sweep"]["k2b_B16_T128"]
    k2b["frac"] = k2b["GB/s"] / hbm_peak
    return out


def measure_c5():
    """BASELINE configs[4] headline shapes (full sweep: tools/sweep_c5.py): packed tree vs the unrolled
    baseline (every root-to-leaf path its own sequence from the same h0), batch 1, us per layer."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import sweep_c5
    from gen import trees
    from paper_2505_14969_b200 import binding
    # a stack of scan layers: no layer writes the next one's tree, dt, parameters or state (as sweep_c5.py)
    binding.stree_set_launch_flags(binding.STREE_LAUNCH_PDL | binding.STREE_LAUNCH_EARLY_STATE |
                                   binding.STREE_LAUNCH_EARLY_TREE | binding.STREE_LAUNCH_EARLY_DT)
    res = {}
    for T in (64, 128, 256):
        par = trees.heap_kary(T, 2)
        paths = sweep_c5.leaf_paths(par)
        maxlen = max(len(p) for p in paths)
        t_p, k_p = sweep_c5.time_scan(par[None], L=16)
        t_u, _ = sweep_c5.time_scan(np.stack([trees.chain(maxlen)] * len(paths)), L=16)
        res[f"heap2_T{T}"] = {"packed_us": t_p, "unrolled_us": t_u, "speedup_vs_unrolled": t_u / t_p,
                              "kernel": {1: "simt", 2: "tcgen05", 3: "tcgen05-128"}.get(k_p)}
    # the 128-row kernel (K2b) at batch 16: HBM roofline of one scan call (state read once, x read, y written,
    # B and C once per tree, dt, parent; 2.7B shape H=80 P=64 N=128 G=1)
    B, T, H, P, N = 16, 128, 80, 64, 128
    t16, k16 = sweep_c5.time_scan(np.stack([trees.heap_kary(T, 2)] * B), L=16)
    nbytes = B * H * P * N * 4 + 2 * B * T * H * P * 2 + 2 * B * T * N * 2 + B * T * H * 4 + B * T * 4 + 2 * H * 4
    res["k2b_B16_T128"] = {"us": t16, "bytes": nbytes, "GB/s": nbytes / t16 * 1e-3, "nodes_per_s": B * T / (t16 * 1e-6),
                           "kernel": {1: "simt", 2: "tcgen05", 3: "tcgen05-128"}.get(k16), "bound": "hbm"}
    return res


if __name__ == "__main__":
    import torch
    sys.path.insert(0, ROOT)
    from bench import load_peaks
    hbm, bf16, _ = load_peaks()
    print(json.dumps(measure(torch.device("cuda", 0), hbm, bf16)))
