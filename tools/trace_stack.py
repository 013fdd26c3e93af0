"""Per-CTA timeline of the fused replay+scan kernel K2 (stree_scan_tc.cu) across back-to-back layers in one
CUDA graph with PDL, as bench.py runs it (STREE_TRACE=1 build):

    STREE_TRACE=1 python -m paper_2505_14969_b200.build && python tools/trace_stack.py [--config c4] [--flags 31]

Times are relative to the end of the previous layer's last CTA (≈ when this layer's dependency wait can
release)."""
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
ap.add_argument("--flags", type=int, default=31)
ap.add_argument("--layers", type=int, default=8)
args = ap.parse_args()
binding.stree_set_launch_flags(args.flags)
prob = inputs.config_problem(args.config)
L = args.layers
lay = [api.upload(inputs.make_problem(prob.dims, prob.parent, seed=inputs.BASE_SEED + 50 + i)) for i in range(L)]
tok, vt = inputs.make_accept_inputs(prob.parent, seed=5, p_match=0.9)
path, plen, _ = api.accept(torch.from_numpy(tok).cuda(), lay[0]["parent"], torch.from_numpy(vt).cuda())
ys = [torch.empty_like(t["x"]) for t in lay]
lib = binding.lib()
lib.stree_debug_tc_trace_ring.argtypes = [ctypes.c_void_p, ctypes.c_int]
W = 256
buf = torch.zeros((16, 1024, W), dtype=torch.int64, device="cuda")
s = torch.cuda.Stream()


def run():
    for t, y in zip(lay, ys):
        api.replay_scan(t, path, plen, t, t["h0"], y=y)


with torch.cuda.stream(s):
    run()
torch.cuda.synchronize()
lib.stree_debug_tc_trace_ring(ctypes.c_void_p(buf.data_ptr()), 16)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    run()
lib.stree_debug_tc_trace_ring(None, 0)
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    g.replay()
e1.record()
torch.cuda.synchronize()
print(f"{args.config} fused replay+scan, graph of {L} layers, flags {args.flags}: "
      f"{e0.elapsed_time(e1) / 10 / L * 1e3:.2f} us per layer")
tr = buf.cpu().numpy().astype(np.int64)[:L]
ncta = int((tr[0, :, 0] > 0).sum())
tr = tr[:, :ncta]
names = {0: "start", 2: "C landed", 46: "ctf32", 50: "coefs done", 51: "BAR_G", 3: "G ready", 45: "end"}
for k in range(9):
    names[4 + 2 * k] = f"acc{k}"
    names[5 + 2 * k] = f"out{k}"
    names[64 + 3 * k] = f"upd_full{k}"
    names[65 + 3 * k] = f"upd_done{k}"
    names[66 + 3 * k] = f"upd_store{k}"
    names[100 + k] = f"mma_y0issued{k}"
    names[109 + k] = f"mma_x+m_ready{k}"
    names[91 + k] = f"built_m{k}"
    names[128 + k] = f"state_issue{k}"
    names[30 + k] = f"mma_full{k}"
    names[118 + k] = f"mma_accempty{k}"
li = L // 2
base = tr[li - 1, :, 45].max()
print(f"{ncta} CTAs per launch; layer {li} relative to layer {li - 1}'s last CTA end (us):")
for c in sorted(names):
    v = tr[li, :, c]
    v = v[v > 0]
    if len(v):
        v = (v - base) / 1000.0
        print(f"  {names[c]:>14s}: min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f}")
for l in range(1, L):
    st, en = tr[l, :, 0], tr[l, :, 45]
    b0 = tr[l - 1, :, 45].max()
    print(f"layer {l}: start {(st.min() - b0) / 1e3:7.2f}..{(st.max() - b0) / 1e3:7.2f}"
          f"  end {(en.min() - b0) / 1e3:7.2f}..{(en.max() - b0) / 1e3:7.2f}  (period {(en.max() - b0) / 1e3:.2f})")
