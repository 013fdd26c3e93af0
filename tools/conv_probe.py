"""Probe: stree_tree_conv timing on one buffer set (L2-resident), with / without PDL, eager launches."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gen import inputs  # noqa: E402
from paper_2505_14969_b200 import binding  # noqa: E402

dev = torch.device("cuda", 0)
_, par_np = inputs.config_trees("c4", inputs.BASE_SEED + 3)
B, T = par_np.shape
for C in (5376, 1024, 16384):
    W = 4
    par = torch.from_numpy(par_np.astype(np.int32)).to(dev)
    u = torch.randn((B, T, C), device=dev).to(torch.bfloat16)
    w = torch.rand((C, W), device=dev)
    bias = torch.rand((C,), device=dev)
    st = torch.randn((B, W - 1, C), device=dev).to(torch.bfloat16)
    out = torch.empty_like(u)
    d = binding.make_conv_dims(u, w)
    for flags in (1, 0):
        binding.stree_set_launch_flags(flags)
        for _ in range(5):
            binding.stree_tree_conv(u, w, bias, st, par, out, True, dims=d)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(100):
            binding.stree_tree_conv(u, w, bias, st, par, out, True, dims=d)
        e1.record()
        torch.cuda.synchronize()
        print(f"C={C} pdl={flags}: {e0.elapsed_time(e1) * 10:.2f} us/call (same buffers, eager)")
    binding.stree_set_launch_flags(1)
    x = torch.empty(1 << 28, dtype=torch.uint8, device=dev)
    e0.record(); x.zero_(); e1.record(); torch.cuda.synchronize()
    print("memset 256MB", e0.elapsed_time(e1) * 1e3, "us")

import ctypes
L = binding.lib()
L.stree_debug_conv_trace.argtypes = [ctypes.c_void_p]
C = 5376
u = torch.randn((B, T, C), device=dev).to(torch.bfloat16)
w = torch.rand((C, 4), device=dev)
bias = torch.rand((C,), device=dev)
st = torch.randn((B, 3, C), device=dev).to(torch.bfloat16)
out = torch.empty_like(u)
par = torch.from_numpy(par_np.astype(np.int32)).to(dev)
binding.stree_set_launch_flags(0)
for it in range(4):
    binding.stree_tree_conv(u, w, bias, st, par, out, it < 2)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 8)()
    L.stree_debug_conv_trace(buf)
    t = [buf[i] for i in range(6)]
    print("phases (us): weights %.2f  pdl %.2f  staging %.2f  validate %.2f  compute+store %.2f" % tuple(
        (t[i + 1] - t[i]) / 1e3 for i in range(5)))
