"""BASELINE configs[4] / SURVEY c5: tree-shape sweep on the Mamba-2 2.7B layer shape (H=80, P=64, N=128,
bf16), packed tree scan vs the paper's two baselines (Fig. 3):

  packed    stree_tree_scan of the packed tree (this work)
  chain     the same number of nodes as one chain through the same call (the cost of tree-ness)
  unrolled  every root-to-leaf path as its own sequence (batch = #leaves, each from the same h0, padded to
            the longest path) — the unrolled baseline; useful work counted = the T packed nodes only

Each variant: L = 32 distinct layers back-to-back in one CUDA graph (inputs > L2), median of 7 replays,
device time per layer; batch = 1 tree (latency, the paper's setting) and, for packed, 16 trees
(throughput).  Prints one JSON object per case.

    python tools/sweep_c5.py [--quick]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gen import inputs, trees  # noqa: E402
from paper_2505_14969_b200 import binding  # noqa: E402

H, P, N, G = 80, 64, 128, 1
LAYERS = 32
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(inputs.BASE_SEED + 900)


def make_layers(B, T, L):
    out = []
    for _ in range(L):
        out.append({
            "x": torch.randn((B, T, H, P), generator=gen, device=dev).to(torch.bfloat16),
            "dt": torch.exp(torch.empty((B, T, H), device=dev).uniform_(np.log(1e-3), np.log(1e-1), generator=gen)),
            "A": -torch.empty((H,), device=dev).uniform_(1.0, 16.0, generator=gen),
            "Bm": torch.randn((B, T, G, N), generator=gen, device=dev).to(torch.bfloat16),
            "Cm": torch.randn((B, T, G, N), generator=gen, device=dev).to(torch.bfloat16),
            "D": 1 + 0.1 * torch.randn((H,), generator=gen, device=dev),
            "h0": torch.randn((B, H, P, N), generator=gen, device=dev),
            "y": torch.empty((B, T, H, P), dtype=torch.bfloat16, device=dev),
        })
    return out


def time_scan(par_b, L=LAYERS):
    par_b = np.asarray(par_b, np.int32)
    B, T = par_b.shape
    lay = make_layers(B, T, L)
    par = torch.from_numpy(par_b).to(dev)
    dims = binding.make_dims(lay[0]["x"], lay[0]["Bm"])
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.Stream(device=dev)

    def run():
        for t in lay:
            binding.stree_tree_scan(t["x"], t["dt"], t["A"], t["Bm"], t["Cm"], t["D"], t["h0"], par, t["y"], st,
                                    dims=dims)

    with torch.cuda.stream(stream):
        run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        run()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        with torch.cuda.stream(stream):
            g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / L)
    assert st.item() == 0
    kern = binding.stree_scan_kernel_for(dims)
    del lay, g
    torch.cuda.empty_cache()
    return float(np.median(ts)), kern


def leaf_paths(par):
    kids = trees.children_lists(par)
    out = []
    for leaf in [i for i in range(len(par)) if not kids[i]]:
        p = [leaf]
        while par[p[-1]] >= 0:
            p.append(int(par[p[-1]]))
        out.append(p[::-1])
    return out


def main():
    quick = "--quick" in sys.argv
    # a stack of scan-only layers: the preceding kernel (the previous layer) writes none of a layer's state, tree,
    # dt or parameters, so the EARLY promises hold (as in bench.py)
    binding.stree_set_launch_flags(binding.STREE_LAUNCH_PDL | binding.STREE_LAUNCH_EARLY_STATE |
                                   binding.STREE_LAUNCH_EARLY_TREE | binding.STREE_LAUNCH_EARLY_DT)
    cases = inputs.sweep_cases()
    if quick:
        cases = [c for c in cases if c[0] in ("heap2_T16", "heap2_T64", "heap4_T64", "chain_T64", "fullbin_L5",
                                              "heap2_T256")]
    for name, par in cases:
        par = np.asarray(par, np.int32)
        T = len(par)
        paths = leaf_paths(par)
        maxlen = max(len(p) for p in paths)
        t_packed, k_packed = time_scan(par[None])
        t_chain, _ = time_scan(trees.chain(T)[None])
        # unrolled: batch of #leaves chains of the longest path length
        t_unr, _ = time_scan(np.stack([trees.chain(maxlen)] * len(paths)))
        t_p16, _ = time_scan(np.stack([par] * 16)) if T <= 128 else (None, None)
        rec = {"case": name, "T": T, "leaves": len(paths), "unrolled_tokens": int(sum(len(p) for p in paths)),
               "kernel": {1: "simt", 2: "tcgen05", 3: "tcgen05-128"}.get(k_packed),
               "packed_us": t_packed, "chain_us": t_chain, "unrolled_us": t_unr,
               "packed_nodes_per_s": T / (t_packed * 1e-6), "unrolled_nodes_per_s": T / (t_unr * 1e-6),
               "speedup_vs_unrolled": t_unr / t_packed, "tree_over_chain": t_packed / t_chain}
        if t_p16 is not None:
            rec["packed_b16_us"] = t_p16
            rec["packed_b16_nodes_per_s"] = 16 * T / (t_p16 * 1e-6)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
