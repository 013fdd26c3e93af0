"""Timeline of CTA 0 of the 128-key tcgen05 tree-attention kernel K7 (globaltimer stamps; debug hook
stree_debug_attn_trace).  Prints per-KV-tile event times relative to the first stamp (us).  The default kernel
is K7b (attn_db_kernel), which has no trace hook: run with STREE_ATTN_DB=0."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gen.attn import attn_config  # noqa: E402
from paper_2505_14969_b200 import binding  # noqa: E402


def main():
    prob = attn_config("hyb8b")
    if "--one-tile" in sys.argv:   # T = 32 nodes x 4 heads = 128 rows: one query tile per CTA (no ping-pong)
        from gen.attn import AttnDims, make_attn_problem
        prob = make_attn_problem(AttnDims(16, 32), prob.parent[:, :32], 7, cache_len=[1280] * 16)
    dev = torch.device("cuda", 0)

    def t(a):
        return torch.from_numpy(a.view(np.int16).copy()).view(torch.bfloat16).to(dev)
    q, kn, vn, kc, vc = (t(getattr(prob, n)) for n in ("q", "k_new", "v_new", "k_cache", "v_cache"))
    cl = torch.from_numpy(prob.cache_len).to(dev)
    par = torch.from_numpy(prob.parent).to(dev)
    o = torch.empty_like(q)
    buf = torch.zeros(1024, dtype=torch.int64, device=dev)
    L = binding.lib()
    L.stree_debug_attn_trace.argtypes = [ctypes.c_void_p]
    for it in range(3):
        binding.stree_tree_attn(q, kn, vn, kc, vc, cl, par, prob.scale, o)
    torch.cuda.synchronize()
    buf.zero_()
    L.stree_debug_attn_trace(ctypes.c_void_p(buf.data_ptr()))
    binding.stree_tree_attn(q, kn, vn, kc, vc, cl, par, prob.scale, o)
    torch.cuda.synchronize()
    L.stree_debug_attn_trace(None)
    a = buf.cpu().numpy().astype(np.int64)
    nz = a[a > 0]
    t0 = nz.min()
    f = lambda v: f"{(v - t0) / 1e3:7.2f}" if v > 0 else "    -  "
    print("cache_len[0] =", prob.cache_len[0])
    print(" j | kempty  vempty | kfull  | pfull0  pfull1 | sfull0  sfull1 | parr0   parr1")
    for j in range(64):
        row = [a[j], a[64 + j], a[256 + j], a[128 + 2 * j], a[129 + 2 * j], a[384 + 2 * j], a[385 + 2 * j],
               a[512 + 2 * j], a[513 + 2 * j]]
        if not any(row):
            continue
        sm = [a[640 + 4 * j + k] for k in range(4)]
        print(f"{j:2d} | {f(row[0])} {f(row[1])} | {f(row[2])} | {f(row[3])} {f(row[4])} | {f(row[5])} {f(row[6])} | "
              f"{f(row[7])} {f(row[8])} | softmax0: ld {f(sm[0])} max {f(sm[1])} exp {f(sm[2])} st {f(sm[3])}")


if __name__ == "__main__":
    main()
