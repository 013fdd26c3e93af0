"""Eager driver for ncu: runs the hot-path kernels of one config a few times on
distinct layer buffers (no graphs), so `ncu -k regex:<kernel>` can capture them.

    python tools/prof_kernels.py [--config c4] [--layers 4] [--iters 3] [--scan-impl auto|simt|tc]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from gen import inputs  # noqa: E402
from paper_2505_14969_b200 import api, binding  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--layers", type=int, default=8)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--scan-impl", default="auto")
ap.add_argument("--fused", action="store_true")
args = ap.parse_args()
binding.stree_set_scan_impl({"auto": 0, "simt": 1, "tc": 2}[args.scan_impl])
prob = inputs.config_problem(args.config)
layers = [api.upload(inputs.make_problem(prob.dims, prob.parent, seed=inputs.BASE_SEED + 3 + li))
          for li in range(args.layers)]
tok, vt = inputs.make_accept_inputs(prob.parent, seed=5, p_match=0.9)
tok, vt = torch.from_numpy(tok).cuda(), torch.from_numpy(vt).cuda()
path, plen, bonus = api.accept(tok, layers[0]["parent"], vt)
for it in range(args.iters):
    mask, depth = api.build_mask(layers[0]["parent"])
    if args.fused:   # replay of the previous acceptance fused with the scan (state in place)
        ys = [api.replay_scan(t, path, plen, t, t["h0"]) for t in layers]
    else:
        ys = [api.tree_scan(t) for t in layers]
    path, plen, bonus = api.accept(tok, layers[0]["parent"], vt)
    if not args.fused:
        for t in layers:
            api.commit(t, path, plen, h_new=t["h0"])
torch.cuda.synchronize()
print("ok")
