"""Timeline of tree 7 / rank 0 of the MSS kernel (build with STREE_TRACE=1)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gen.mss import mss_config  # noqa: E402
from paper_2505_14969_b200 import binding  # noqa: E402

mp = mss_config("c4")
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
args = [d(getattr(mp, k)) for k in ("tokens", "parent", "p_target", "q_draft", "u_accept", "u_bonus")]
B, T = mp.parent.shape
path = torch.empty((B, T), dtype=torch.int32, device="cuda")
plen = torch.empty(B, dtype=torch.int32, device="cuda")
bon = torch.empty(B, dtype=torch.int32, device="cuda")
L = binding.lib()
L.stree_debug_mss_trace.argtypes = [ctypes.c_void_p]
for _ in range(3):
    binding.stree_accept_mss(*args, path, plen, bon)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
binding.stree_accept_mss(*args, path, plen, bon)
e1.record()
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 64)()
L.stree_debug_mss_trace(buf)
t = np.array([buf[i] for i in range(64)], dtype=np.int64)
t = t[t > 0]
print("kernel (events) us:", e0.elapsed_time(e1) * 1e3)
print("stamps (us from first):", np.round((t - t[0]) / 1e3, 2).tolist())
