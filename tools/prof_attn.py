"""ncu target: a few stree_tree_attn / stree_kv_commit calls on the bench workload (hyb8b)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_next  # noqa: E402

if __name__ == "__main__":
    bench_next.measure(torch.device("cuda", 0), 6546.9, 1651.3, layers_attn=4, layers_ssm=4)
