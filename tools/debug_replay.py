import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from tests.test_replay_gpu import make_pair, run_fused, oracle_pair
from paper_2505_14969_b200 import binding
binding.lib()
B, Tp, T, H, P, N, G = 16, 64, 64, 80, 64, 128, 1
prev, new, path, plen = make_pair(B, Tp, T, H, P, N, G, "bf16", seed=Tp * 7 + T)
y, h, st = run_fused(prev, new, path, plen)
yr, hr, _, _ = oracle_pair(prev, new, path, plen)
err = np.abs(h - hr).max(axis=(2, 3)) / np.abs(hr).max(axis=(2, 3))
bad = np.argwhere(err > 1e-4)
print("status", st, "bad blocks", len(bad), "of", B * H)
print("bad (b,h) sample", bad[:20].tolist())
print("plen", plen.tolist())
cnt = np.zeros(H, int)
for b_, h_ in bad:
    cnt[h_] += 1
print("bad per head", cnt.tolist())
if len(bad):
    b_, h_ = bad[0]
    d = np.abs(h[b_, h_] - hr[b_, h_])
    print("bad rows", np.argwhere(d.max(1) > 1e-3).ravel().tolist()[:70])
    print("bad cols", np.argwhere(d.max(0) > 1e-3).ravel().tolist()[:130])
    # compare with h0 (unchanged?)
    print("equal to h0?", np.abs(h[b_, h_] - prev.h0[b_, h_]).max())
