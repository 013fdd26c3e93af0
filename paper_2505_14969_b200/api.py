"""Allocation helpers around the binding: allocate outputs with torch, call the
C ABI, return tensors.  Still no computation outside the CUDA kernels."""
from __future__ import annotations

import numpy as np
import torch

from . import binding as _b


def bf16_from_bits(bits: np.ndarray, device) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).to(device)


def upload(prob, device="cuda", pin=False) -> dict:
    """gen.inputs.Problem -> dict of device tensors in the ABI layouts."""
    def io(a):
        if prob.dims.io_dtype == "bf16":
            t = torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16)
        else:
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
        return t.pin_memory().to(device, non_blocking=True) if pin else t.to(device)

    def f32(a):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
        return t.to(device)

    return dict(x=io(prob.x), dt=f32(prob.dt), A=f32(prob.A), Bm=io(prob.Bm), Cm=io(prob.Cm), D=f32(prob.D),
                h0=f32(prob.h0), parent=torch.from_numpy(np.ascontiguousarray(prob.parent, np.int32)).to(device))


def build_mask(parent: torch.Tensor, dev_status=None):
    B, T = parent.shape
    W = (T + 31) // 32
    mask = torch.empty((B, T, W), dtype=torch.int32, device=parent.device)
    depth = torch.empty((B, T), dtype=torch.int32, device=parent.device)
    _b.stree_build_mask(parent, mask, depth, dev_status)
    return mask, depth


def tree_scan(t: dict, dev_status=None, y=None, h0="h0"):
    x = t["x"]
    if y is None:
        y = torch.empty_like(x)
    _b.stree_tree_scan(x, t["dt"], t["A"], t["Bm"], t["Cm"], t.get("D"), t.get(h0) if h0 else None,
                       t["parent"], y, dev_status)
    return y


def accept(tokens, parent, vtok, dev_status=None):
    B, T = parent.shape
    path = torch.empty((B, T), dtype=torch.int32, device=parent.device)
    plen = torch.empty((B,), dtype=torch.int32, device=parent.device)
    bonus = torch.empty((B,), dtype=torch.int32, device=parent.device)
    _b.stree_accept(tokens, parent, vtok, path, plen, bonus, dev_status)
    return path, plen, bonus


def commit(t: dict, path, path_len, h_new=None, dev_status=None, use_parent=True):
    if h_new is None:
        h_new = torch.empty_like(t["h0"])
    _b.stree_commit(t["x"], t["dt"], t["A"], t["Bm"], t["h0"], t["parent"] if use_parent else None, path,
                    path_len, h_new, dev_status)
    return h_new


def replay_scan(prev: dict, path, path_len, t: dict, h, dev_status=None, y=None, use_parent=True):
    """Fused commit of the previous tree (cache `prev`, accepted `path`) into the state `h` (in place)
    and scan of the new tree `t` from the committed state; returns y."""
    if y is None:
        y = torch.empty_like(t["x"])
    _b.stree_replay_scan(prev["x"], prev["dt"], prev["Bm"], prev["parent"] if use_parent else None, path, path_len,
                         t["x"], t["dt"], t["A"], t["Bm"], t["Cm"], t.get("D"), h, t["parent"], y, dev_status)
    return y
