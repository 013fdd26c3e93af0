"""Do consecutive scan launches overlap under PDL?  Traces 4 back-to-back scans
(distinct layers) into separate buffers and prints each kernel's CTA start/end span."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from gen import inputs  # noqa: E402
from paper_2505_14969_b200 import api, binding  # noqa: E402

flags = int(sys.argv[1]) if len(sys.argv) > 1 else 3
binding.stree_set_launch_flags(flags)
prob = inputs.config_problem("c4")
layers = [api.upload(inputs.make_problem(prob.dims, prob.parent, seed=inputs.BASE_SEED + 50 + i)) for i in range(8)]
ys = [torch.empty_like(l["x"]) for l in layers]
L = binding.lib()
L.stree_debug_tc_trace.argtypes = [ctypes.c_void_p]
bufs = [torch.zeros((1024, 256), dtype=torch.int64, device="cuda") for _ in range(4)]
for _ in range(2):
    for l, y in zip(layers, ys):
        api.tree_scan(l, y=y)
torch.cuda.synchronize()
for i in range(4):   # scans of layers 4..7, traced
    api.tree_scan(layers[i], y=ys[i])
for i in range(4):
    L.stree_debug_tc_trace(ctypes.c_void_p(bufs[i].data_ptr()))
    api.tree_scan(layers[4 + i], y=ys[4 + i])
L.stree_debug_tc_trace(None)
torch.cuda.synchronize()
trs = [b.cpu().numpy().astype(np.int64) for b in bufs]
t0 = min(int(t[t[:, 0] > 0, 0].min()) for t in trs)
for i, t in enumerate(trs):
    t = t[t[:, 0] > 0]
    last_out = np.max(t[:, 4:28], axis=1)   # latest acc/out stamp per CTA
    print(f"kernel {i}: CTAs {len(t)}  start {(t[:, 0].min() - t0) / 1e3:7.2f}..{(t[:, 0].max() - t0) / 1e3:7.2f} us"
          f"  last-out {(last_out.min() - t0) / 1e3:7.2f}..{(last_out.max() - t0) / 1e3:7.2f} us"
          f"  G-ready med {(np.median(t[:, 3]) - t0) / 1e3:7.2f}  first-acc med {(np.median(t[:, 4]) - t0) / 1e3:7.2f}")
