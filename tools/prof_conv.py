"""Tree conv at the bench shape (c4 trees, conv_dim 5376, W = 4, bf16, 64 layers in one CUDA graph): time
per call under the launch flags PDL / + EARLY_TREE / all promises, or a few eager calls for ncu (--ncu)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from gen import inputs  # noqa: E402
from paper_2505_14969_b200 import binding  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ncu", action="store_true")
ap.add_argument("--layers", type=int, default=64)
args = ap.parse_args()
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(1)
dd, par_np = inputs.config_trees("c4", inputs.BASE_SEED + 3)
B, T = par_np.shape
C, W = 80 * 64 + 2 * 128, 4
parc = torch.from_numpy(par_np.astype(np.int32)).to(dev)
bf = torch.bfloat16
cl = [{"u": torch.randn((B, T, C), generator=gen, device=dev).to(bf),
       "w": torch.rand((C, W), generator=gen, device=dev) - 0.5,
       "bias": torch.rand((C,), generator=gen, device=dev) - 0.5,
       "st": torch.randn((B, W - 1, C), generator=gen, device=dev).to(bf),
       "out": torch.empty((B, T, C), dtype=bf, device=dev)} for _ in range(args.layers)]
cdims = binding.make_conv_dims(cl[0]["u"], cl[0]["w"])
st = torch.zeros(1, dtype=torch.int32, device=dev)


def run():
    for t in cl:
        binding.stree_tree_conv(t["u"], t["w"], t["bias"], t["st"], parc, t["out"], True, st, dims=cdims)


vbytes = 2 * B * T * C * 2 + B * (W - 1) * C * 2 + C * W * 4 + C * 4 + B * T * 4
for flags in (1, 1 | 8, 31):
    binding.stree_set_launch_flags(flags)
    if args.ncu:
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        continue
    s = torch.cuda.Stream()
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
    us = e0.elapsed_time(e1) * 1e3 / (10 * len(cl))
    print(f"flags={flags}: {us:.2f} us per call, {vbytes / us / 1e3:.0f} GB/s")
