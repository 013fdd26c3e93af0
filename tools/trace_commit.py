"""Per-CTA timeline of the commit ring kernel (globaltimer stamps)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from gen import inputs  # noqa: E402
from paper_2505_14969_b200 import api, binding  # noqa: E402

prob = inputs.config_problem("c4")
t = api.upload(prob)
tok, vt = inputs.make_accept_inputs(prob.parent, seed=5, p_match=0.9)
path, plen, bonus = api.accept(torch.from_numpy(tok).cuda(), t["parent"], torch.from_numpy(vt).cuda())
L = binding.lib()
L.stree_debug_commit_trace.argtypes = [ctypes.c_void_p]
buf = torch.zeros((1024, 64), dtype=torch.int64, device="cuda")
h = t["h0"]
for _ in range(3):
    api.commit(t, path, plen, h_new=h)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    api.commit(t, path, plen, h_new=h)
e1.record()
torch.cuda.synchronize()
print(f"commit eager avg {e0.elapsed_time(e1) / 10 * 1e3:.2f} us")
L.stree_debug_commit_trace(ctypes.c_void_p(buf.data_ptr()))
api.commit(t, path, plen, h_new=h)
torch.cuda.synchronize()
L.stree_debug_commit_trace(None)
tr = buf.cpu().numpy()
n = int((tr[:, 0] > 0).sum())
tr = tr[:n].astype(np.int64)
t0 = tr[:, 0].min()
rel = np.where(tr > 0, tr - t0, -1) / 1000.0
names = {0: "start", 1: "validated", 2: "coefs staged", 3: "end"}
for k in range(16):
    names[4 + 2 * k] = f"full{k}"
    names[5 + 2 * k] = f"stored{k}"
for c in sorted(names):
    v = rel[:, c]
    v = v[v >= 0]
    if len(v):
        print(f"{names[c]:>14s}: min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f}")
