"""Per-CTA phase timeline of the tcgen05 scan kernel (globaltimer stamps).

    python tools/trace_tc.py [--config c4]
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from gen import inputs  # noqa: E402
from paper_2505_14969_b200 import api, binding  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--flags", type=int, default=0)
args = ap.parse_args()
binding.stree_set_launch_flags(args.flags)
prob = inputs.config_problem(args.config)
layers = [api.upload(inputs.make_problem(prob.dims, prob.parent, seed=inputs.BASE_SEED + 50 + i)) for i in range(8)]
t = layers[-1]
L = binding.lib()
L.stree_debug_tc_trace.argtypes = [ctypes.c_void_p]
buf = torch.zeros((1024, 256), dtype=torch.int64, device="cuda")
ys = [torch.empty_like(l["x"]) for l in layers]
for _ in range(3):
    for l, y in zip(layers, ys):
        api.tree_scan(l, y=y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    for l, y in zip(layers, ys):
        api.tree_scan(l, y=y)
e1.record()
torch.cuda.synchronize()
print(f"eager back-to-back over 8 layers: {e0.elapsed_time(e1) / 40 * 1e3:.2f} us per scan")
for l, y in zip(layers[:-1], ys):
    api.tree_scan(l, y=y)
L.stree_debug_tc_trace(ctypes.c_void_p(buf.data_ptr()))
api.tree_scan(t, y=ys[-1])
torch.cuda.synchronize()
L.stree_debug_tc_trace(None)
tr = buf.cpu().numpy().astype(np.int64)
n = int((tr[:, 0] > 0).sum())
tr = tr[:n]
t0 = tr[:, 0].min()
rel = np.where(tr > 0, tr - t0, -1) / 1000.0  # us
print(f"{n} CTAs; kernel span {rel[:, 45].max():.2f} us")
names = {0: "start", 1: "epi start", 2: "C landed", 3: "G in regs", 45: "end", 46: "ctf32 done", 47: "mask done", 48: "dt stored", 49: "lam done", 50: "coefs done", 51: "BAR_G passed"}
for k in range(12):
    names[4 + 2 * k] = f"acc{k}"
    names[5 + 2 * k] = f"out{k}"
    names[30 + k] = f"mma_full{k}"
for k in range(16):
    names[128 + k] = f"state_issue{k}"
for k in range(9):
    names[100 + k] = f"mma_y0issued{k}"
    names[109 + k] = f"mma_x+m_ready{k}"
    names[118 + k] = f"mma_accempty{k}"
    names[91 + k] = f"built_m{k}"
names[170] = "epi_dry_start"
names[171] = "epi_dry_end"
for k in range(6):
    names[52 + 2 * k] = f"epi_go{k}"
    names[53 + 2 * k] = f"epi_done{k}"
cols = sorted(names)
for c in cols:
    v = rel[:, c]
    v = v[v >= 0]
    if len(v):
        print(f"{names[c]:>20s}: min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f} us")
for cta in (0, n // 2, n - 1):
    print(f"cta {cta}: " + " ".join(f"{names[c]}={rel[cta, c]:.2f}" for c in cols if rel[cta, c] >= 0))
