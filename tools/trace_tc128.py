"""Per-CTA timeline of the 128-row scan kernel K2b (stree_scan_tc128.cu) across back-to-back layers in one
CUDA graph with PDL (needs a STREE_TRACE=1 build):

    STREE_TRACE=1 python -m paper_2505_14969_b200.build && python tools/trace_tc128.py [--B 16] [--T 128]
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from gen import inputs, trees  # noqa: E402
from paper_2505_14969_b200 import api, binding  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=16)
ap.add_argument("--T", type=int, default=128)
ap.add_argument("--H", type=int, default=80)
ap.add_argument("--layers", type=int, default=8)
ap.add_argument("--flags", type=int, default=31)
args = ap.parse_args()
binding.stree_set_launch_flags(args.flags)
par = np.stack([trees.heap_kary(args.T, 2) for _ in range(args.B)])
d = inputs.Dims(args.B, args.T, args.H, 64, 128, 1, "bf16")
lay = [api.upload(inputs.make_problem(d, par, seed=100 + i)) for i in range(args.layers)]
ys = [torch.empty_like(t["x"]) for t in lay]
lib = binding.lib()
lib.stree_debug_tc128_trace.argtypes = [ctypes.c_void_p]
W = 64
buf = torch.zeros((16, 1024, W), dtype=torch.int64, device="cuda")
s = torch.cuda.Stream()


def run():
    for t, y in zip(lay, ys):
        api.tree_scan(t, y=y)


with torch.cuda.stream(s):
    run()
torch.cuda.synchronize()
lib.stree_debug_tc128_trace(ctypes.c_void_p(buf.data_ptr()))
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    run()
lib.stree_debug_tc128_trace(None)
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    g.replay()
e1.record()
torch.cuda.synchronize()
L = args.layers
print(f"B={args.B} T={args.T} H={args.H}: graph of {L} layers: {e0.elapsed_time(e1) / 10 / L * 1e3:.2f} us per layer")
tr = buf.cpu().numpy().astype(np.int64)[:L]
ncta = int((tr[0, :, 0] > 0).sum())
tr = tr[:, :ncta]
names = {0: "start", 1: "pdl wait passed", 14: "math: prologue loads landed", 15: "math: pointer jumping done",
         16: "math: modes + coefficients done", 2: "iss: C,B landed", 3: "math: tree prologue done", 4: "math: C->tf32 done",
         5: "math: G ready", 63: "end"}
for k in range(8):
    names[6 + k] = f"bld: X' (M') head {k} ready"
    names[20 + 2 * k] = f"iss: Y0 head {k} issued"
    names[21 + 2 * k] = f"iss: M'+x head {k} ready"
    names[40 + 2 * k] = f"epi: acc head {k} ready"
    names[41 + 2 * k] = f"epi: head {k} done"
li = L // 2
base = tr[li, :, 1][tr[li, :, 1] > 0].min()
print(f"{ncta} CTAs per launch; layer {li} phases relative to its first dependency-wait release (us):")
for k in sorted(names):
    v = tr[li, :, k]
    v = v[v > 0]
    if len(v):
        v = (v - base) / 1000.0
        print(f"  {names[k]:>26s}: min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f}")
for l in range(L):
    st, wt, en = tr[l, :, 0], tr[l, :, 1], tr[l, :, 63]
    print(f"layer {l}: start {(st.min() - base) / 1e3:7.2f}  wait {(wt.min() - base) / 1e3:7.2f}..{(wt.max() - base) / 1e3:7.2f}"
          f"  end {(en.min() - base) / 1e3:7.2f}..{(en.max() - base) / 1e3:7.2f}")
