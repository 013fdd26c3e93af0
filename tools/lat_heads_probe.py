"""Batch-1 fused replay+scan per-layer time vs the number of heads (CTAs per layer) at the c3 tree and layer shape
(T = 64, P = 64, N = 128): 64 distinct layers in one CUDA graph under the bench's launch promises.  With at most
#SMs/2 CTAs the kernel takes one SM per CTA (consecutive layers on different SMs); above that, two CTAs share an
SM and a layer's CTAs sit beside the next layer's pre-wait work.  The per-CTA work is the same for every H, so
the curve separates per-CTA latency from SM sharing.

    python tools/lat_heads_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from gen import inputs  # noqa: E402
from paper_2505_14969_b200 import api, binding  # noqa: E402

binding.stree_set_launch_flags(int(os.environ.get("FLAGS", "31")))
FUSED = os.environ.get("FUSED", "1") == "1"   # 0: stree_tree_scan only
base = inputs.config_problem("c3")
tok, vt = inputs.make_accept_inputs(base.parent, seed=3, p_match=0.9)
L = 64
for H in [int(x) for x in os.environ.get("HEADS", "8,24,40,64,74,80,96,128").split(",")]:
    d = inputs.Dims(1, base.dims.n_nodes, H, 64, 128, 1, "bf16")
    lay = [api.upload(inputs.make_problem(d, base.parent, seed=inputs.BASE_SEED + 50 + i)) for i in range(L)]
    par = lay[0]["parent"]
    path, plen, _ = api.accept(torch.from_numpy(tok).cuda(), par, torch.from_numpy(vt).cuda())
    ys = [torch.empty_like(t["x"]) for t in lay]
    s = torch.cuda.Stream()

    def run():
        for t, y in zip(lay, ys):
            if FUSED:
                api.replay_scan(t, path, plen, t, t["h0"], y=y)
            else:
                api.tree_scan(t, y=y)

    with torch.cuda.stream(s):
        run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        run()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"H = {H:3d} ({H} CTAs per layer): {e0.elapsed_time(e1) / 10 / L * 1e3:6.2f} us per layer", flush=True)
    del lay, ys, g
