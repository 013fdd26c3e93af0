"""Per-CTA timeline of the small-batch scan kernel (stree_scan_lat.cu) across back-to-back layers in one
CUDA graph with PDL (needs a STREE_TRACE=1 build):

    STREE_TRACE=1 python -m paper_2505_14969_b200.build && python tools/trace_lat.py [--config c3] [--flags 7]
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
ap.add_argument("--config", default="c3")
ap.add_argument("--flags", type=int, default=7)
ap.add_argument("--layers", type=int, default=12)
ap.add_argument("--fused", type=int, default=1)
args = ap.parse_args()
binding.stree_set_launch_flags(args.flags)
prob = inputs.config_problem(args.config)
L = args.layers
lay = [api.upload(inputs.make_problem(prob.dims, prob.parent, seed=inputs.BASE_SEED + 50 + i)) for i in range(L)]
tok, vt = inputs.make_accept_inputs(prob.parent, seed=3, p_match=0.9)
par = lay[0]["parent"]
path, plen, bonus = api.accept(torch.from_numpy(tok).cuda(), par, torch.from_numpy(vt).cuda())
ys = [torch.empty_like(t["x"]) for t in lay]
lib = binding.lib()
lib.stree_debug_lat_trace.argtypes = [ctypes.c_void_p]
W = 32
buf = torch.zeros((16, 1024, W), dtype=torch.int64, device="cuda")
s = torch.cuda.Stream()


def run():
    for t, y in zip(lay, ys):
        if args.fused:
            api.replay_scan(t, path, plen, t, t["h0"], y=y)
        else:
            api.tree_scan(t, y=y)


with torch.cuda.stream(s):
    run()
torch.cuda.synchronize()
lib.stree_debug_lat_trace(ctypes.c_void_p(buf.data_ptr()))
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    run()
lib.stree_debug_lat_trace(None)
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    g.replay()
e1.record()
torch.cuda.synchronize()
print(f"graph of {L} layers: {e0.elapsed_time(e1) / 10 / L * 1e3:.2f} us per layer")
tr = buf.cpu().numpy().astype(np.int64)[:L]
ncta = int((tr[0, :, 0] > 0).sum())
tr = tr[:, :ncta]
t0 = tr[:, :, 0][tr[:, :, 0] > 0].min()
names = {0: "start", 1: "setup done", 2: "pdl wait passed", 3: "iss: C,B landed", 4: "iss: split ready",
         5: "iss: Y0 issued", 6: "iss: M' ready", 7: "iss: x ready", 8: "iss: Y' issued", 10: "row: tree done",
         11: "row: lambda done", 12: "row: G ready", 13: "row: M' done", 14: "epi: acc ready", 15: "epi: stored",
         16: "aux: split done", 17: "epi: tmem loaded", 18: "epi: computed", 25: "bld: G loaded",
         26: "bld: computed", 27: "bld: stored", 28: "upd half0", 29: "split half0", 19: "upd half1", 20: "rep: prologue", 21: "rep: state landed", 22: "state: upd+split",
         23: "rep: wait passed", 24: "rep: stored", 30: "end"}
rel = np.where(tr > 0, tr - t0, -1) / 1000.0
print(f"{ncta} CTAs per launch")
for li in range(L):
    st = rel[li, :, 0]
    en = rel[li, :, 30]
    print(f"layer {li:2d}: start {st.min():7.2f}..{st.max():7.2f}  wait {rel[li, :, 2].min():7.2f}..{rel[li, :, 2].max():7.2f}"
          f"  end {en.min():7.2f}..{en.max():7.2f}")
for li in (L // 2, L // 2 + 1):
    base = rel[li, :, 2].min()
    print(f"layer {li} phases relative to its first dependency-wait release:")
    for k in sorted(names):
        v = rel[li, :, k]
        v = v[v >= 0]
        if len(v):
            print(f"  {names[k]:>20s}: min {v.min() - base:7.2f}  med {np.median(v) - base:7.2f}  max {v.max() - base:7.2f}")
# per layer: body (wait -> last end), gap (last end -> next wait), pre-wait window (first start -> wait), median of
# the key phases relative to the wait, and how many CTAs share an SM with a CTA of the previous layer
sm = tr[:, :, 31]
keys = [(1, "setup"), (21, "st.land"), (22, "upd+spl"), (16, "split"), (3, "CB"), (12, "G"), (13, "M'"), (14, "acc"),
        (15, "stored")]
print("layer  window  body   gap   " + " ".join(f"{n:>7s}" for _, n in keys) + "  shareSM")
for li in range(1, L - 1):
    w = rel[li, :, 2].min()
    body = rel[li, :, 30].max() - w
    gap = rel[li + 1, :, 2].min() - rel[li, :, 30].max()
    win = w - rel[li, :, 0].min()
    cols = []
    for k, _ in keys:
        v = rel[li, :, k]
        v = v[v >= 0]
        cols.append(f"{np.median(v) - w:7.2f}" if len(v) else "      -")
    share = len(set(sm[li].tolist()) & set(sm[li - 1].tolist()))
    print(f"{li:5d} {win:6.2f} {body:6.2f} {gap:5.2f}   " + " ".join(cols) + f"  {share:5d}")
# stragglers of one layer: the CTAs that end last, with their SM and phases (relative to the layer's wait)
li = L // 2
w = rel[li, :, 2].min()
order = np.argsort(rel[li, :, 30])[::-1]
print(f"layer {li}: slowest / fastest CTAs (block, sm, start, setup, prologue, upd+split, CB, G, M', acc, end)")
for c in list(order[:6]) + list(order[-3:]):
    v = [rel[li, c, k] - w if rel[li, c, k] >= 0 else float("nan") for k in (0, 1, 20, 22, 3, 12, 13, 14, 30)]
    print(f"  cta {c:3d} sm {int(sm[li, c]):3d}  " + " ".join(f"{x:6.2f}" for x in v))
