"""Eager K2b driver for ncu: B trees of T nodes (heap-2), H=80 heads, distinct layer buffers."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from gen import inputs, trees
from paper_2505_14969_b200 import api, binding
B, T = int(sys.argv[1]), int(sys.argv[2])
binding.stree_set_launch_flags(31)
par = np.stack([trees.heap_kary(T, 2) for _ in range(B)])
d = inputs.Dims(B, T, 80, 64, 128, 1, "bf16")
lay = [api.upload(inputs.make_problem(d, par, seed=100 + i)) for i in range(4)]
for it in range(4):
    for t in lay:
        api.tree_scan(t)
torch.cuda.synchronize(); print("ok")
