"""Thin Python binding of the C ABI in include/stree.h (argument marshalling only).

Every function has the name of the C entry point, takes torch CUDA tensors
(caller-allocated outputs, exactly like the C call), passes raw device
pointers and the current torch stream to libstree.so, and raises
``StreeError`` on a non-zero status.  All computation happens in the CUDA
kernels of ``csrc/``; there is no CPU or PyTorch fallback: if the library is
missing or fails to load, import/usage fails loudly.
"""
from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libstree.so")

STREE_F32, STREE_BF16 = 0, 1
STREE_SCAN_AUTO, STREE_SCAN_SIMT, STREE_SCAN_TC, STREE_SCAN_TC_PIPELINE = 0, 1, 2, 3
DEV_BAD_ROOT, DEV_BAD_PARENT, DEV_BAD_PATH, DEV_CAPACITY = 1, 2, 3, 5
MAX_NODES = 256


class StreeError(RuntimeError):
    def __init__(self, fn, status):
        super().__init__(f"{fn}: status {status} ({status_string(status)})")
        self.status = status


class stree_dims(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("n_nodes", ctypes.c_int32), ("n_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("d_state", ctypes.c_int32), ("n_groups", ctypes.c_int32),
                ("io_dtype", ctypes.c_int32)]


STREE_MAX_Y_PEERS = 8


class stree_yout(ctypes.Structure):
    _fields_ = [("n_peers", ctypes.c_int32), ("heads_total", ctypes.c_int32), ("head_offset", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("peers", ctypes.c_void_p * STREE_MAX_Y_PEERS)]


def make_yout(peers, heads_total: int, head_offset: int) -> stree_yout:
    """peers: tensors or raw device addresses (ints) of the [B][T][heads_total][P] y buffers."""
    yo = stree_yout()
    if not 1 <= len(peers) <= STREE_MAX_Y_PEERS:
        raise ValueError(f"1..{STREE_MAX_Y_PEERS} y peers, got {len(peers)}")
    yo.n_peers, yo.heads_total, yo.head_offset = len(peers), int(heads_total), int(head_offset)
    for i, p in enumerate(peers):
        yo.peers[i] = p if isinstance(p, int) else p.data_ptr()
    return yo


class stree_scan_opts(ctypes.Structure):
    _fields_ = [("dt_bias", ctypes.c_void_p), ("dt_softplus", ctypes.c_int32), ("d_per_channel", ctypes.c_int32)]


def make_opts(dt_bias=None, dt_softplus=False, d_per_channel=False) -> stree_scan_opts:
    """Scan options (include/stree.h): dt_bias [H] f32 tensor or None, softplus of dt, D of shape [H][P]."""
    return stree_scan_opts(_ptr(dt_bias), int(bool(dt_softplus)), int(bool(d_per_channel)))


class stree_attn_dims(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("n_nodes", ctypes.c_int32), ("n_q_heads", ctypes.c_int32),
                ("n_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32), ("cache_cap", ctypes.c_int32),
                ("io_dtype", ctypes.c_int32)]


class stree_conv_dims(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("n_nodes", ctypes.c_int32), ("channels", ctypes.c_int32),
                ("width", ctypes.c_int32), ("io_dtype", ctypes.c_int32)]


_lib = None


def lib():
    """Load libstree.so (built in-tree by __graft_entry__.build()).  No fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32 = ctypes.c_void_p, ctypes.c_int32
        sig = {
            "stree_build_mask": [vp, i32, i32, vp, vp, vp, vp],
            "stree_tree_scan": [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp],
            "stree_accept": [vp, vp, vp, i32, i32, vp, vp, vp, vp, vp],
            "stree_commit": [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp],
            "stree_set_scan_impl": [ctypes.c_int],
            "stree_set_launch_flags": [ctypes.c_uint32],
            "stree_replay_scan": [vp] * 19,
            "stree_tree_scan_sharded": [vp] * 12,
            "stree_tree_scan_ex": [vp] * 13,
            "stree_commit_ex": [vp] * 13,
            "stree_replay_scan_ex": [vp] * 20,
            "stree_replay_scan_sharded": [vp] * 19,
            "stree_scan_kernel_for": [vp],
            "stree_commit_kernel_for": [vp, i32],
            "stree_tree_conv": [vp, vp, vp, vp, vp, vp, i32, vp, vp, vp],
            "stree_conv_commit": [vp, vp, vp, vp, vp, vp, vp, vp, vp],
            "stree_tree_attn": [vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_float, vp, vp, vp],
            "stree_kv_commit": [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp],
            "stree_attn_kernel_for": [vp],
            "stree_accept_mss": [vp, vp, vp, vp, vp, vp, i32, i32, i32, vp, vp, vp, vp, vp],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.stree_status_string.argtypes = [ctypes.c_int]
        L.stree_status_string.restype = ctypes.c_char_p
        L.stree_version.argtypes = []
        L.stree_version.restype = ctypes.c_char_p
        _lib = L
    return _lib


(STREE_LAUNCH_PDL, STREE_LAUNCH_EARLY_STATE, STREE_LAUNCH_EARLY_REPLAY, STREE_LAUNCH_EARLY_TREE,
 STREE_LAUNCH_EARLY_DT) = 1, 2, 4, 8, 16

EXPORTED_SYMBOLS = ("stree_build_mask", "stree_tree_scan", "stree_accept", "stree_commit",
                    "stree_status_string", "stree_set_scan_impl", "stree_set_launch_flags", "stree_scan_kernel_for", "stree_version",
                    "stree_replay_scan", "stree_commit_kernel_for", "stree_tree_conv", "stree_conv_commit",
                    "stree_tree_attn", "stree_kv_commit", "stree_attn_kernel_for", "stree_accept_mss")


def status_string(s: int) -> str:
    return lib().stree_status_string(int(s)).decode()


def version() -> str:
    return lib().stree_version().decode()


def _ptr(t):
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        raise TypeError("expected a torch.Tensor")
    if not t.is_cuda:
        raise ValueError("stree: tensors must live on a CUDA device")
    if not t.is_contiguous():
        raise ValueError("stree: tensors must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _check(fn, st):
    if st != 0:
        raise StreeError(fn, st)


def io_code(dtype) -> int:
    if dtype == torch.bfloat16:
        return STREE_BF16
    if dtype == torch.float32:
        return STREE_F32
    raise TypeError(f"stree: unsupported io dtype {dtype}")


def make_dims(x: torch.Tensor, Bm: torch.Tensor) -> stree_dims:
    B, T, H, P = x.shape
    G, N = Bm.shape[2], Bm.shape[3]
    return stree_dims(B, T, H, P, N, G, io_code(x.dtype))


def stree_build_mask(parent, mask, depth=None, dev_status=None, stream=None):
    B, T = parent.shape
    _check("stree_build_mask", lib().stree_build_mask(_ptr(parent), B, T, _ptr(mask), _ptr(depth),
                                                      _ptr(dev_status), _stream(stream)))


def stree_tree_scan(x, dt, A, Bm, Cm, D, h0, parent, y, dev_status=None, stream=None, dims=None):
    d = dims if dims is not None else make_dims(x, Bm)
    _check("stree_tree_scan", lib().stree_tree_scan(ctypes.byref(d), _ptr(x), _ptr(dt), _ptr(A), _ptr(Bm),
                                                    _ptr(Cm), _ptr(D), _ptr(h0), _ptr(parent), _ptr(y),
                                                    _ptr(dev_status), _stream(stream)))


def stree_accept(tokens, parent, vtok, path, path_len, bonus, dev_status=None, stream=None):
    B, T = parent.shape
    _check("stree_accept", lib().stree_accept(_ptr(tokens), _ptr(parent), _ptr(vtok), B, T, _ptr(path),
                                              _ptr(path_len), _ptr(bonus), _ptr(dev_status), _stream(stream)))


def stree_commit(x, dt, A, Bm, h0, parent, path, path_len, h_new, dev_status=None, stream=None, dims=None):
    d = dims if dims is not None else make_dims(x, Bm)
    _check("stree_commit", lib().stree_commit(ctypes.byref(d), _ptr(x), _ptr(dt), _ptr(A), _ptr(Bm), _ptr(h0),
                                              _ptr(parent), _ptr(path), _ptr(path_len), _ptr(h_new),
                                              _ptr(dev_status), _stream(stream)))


def stree_replay_scan(x_prev, dt_prev, Bm_prev, parent_prev, path, path_len, x, dt, A, Bm, Cm, D, h, parent, y,
                      dev_status=None, stream=None, dims_prev=None, dims=None):
    dp = dims_prev if dims_prev is not None else make_dims(x_prev, Bm_prev)
    d = dims if dims is not None else make_dims(x, Bm)
    _check("stree_replay_scan", lib().stree_replay_scan(
        ctypes.byref(dp), _ptr(x_prev), _ptr(dt_prev), _ptr(Bm_prev), _ptr(parent_prev), _ptr(path),
        _ptr(path_len), ctypes.byref(d), _ptr(x), _ptr(dt), _ptr(A), _ptr(Bm), _ptr(Cm), _ptr(D), _ptr(h),
        _ptr(parent), _ptr(y), _ptr(dev_status), _stream(stream)))


def stree_tree_scan_sharded(x, dt, A, Bm, Cm, D, h0, parent, yout, dev_status=None, stream=None, dims=None):
    d = dims if dims is not None else make_dims(x, Bm)
    _check("stree_tree_scan_sharded", lib().stree_tree_scan_sharded(
        ctypes.byref(d), _ptr(x), _ptr(dt), _ptr(A), _ptr(Bm), _ptr(Cm), _ptr(D), _ptr(h0), _ptr(parent),
        ctypes.byref(yout), _ptr(dev_status), _stream(stream)))


def stree_replay_scan_sharded(x_prev, dt_prev, Bm_prev, parent_prev, path, path_len, x, dt, A, Bm, Cm, D, h, parent,
                              yout, dev_status=None, stream=None, dims_prev=None, dims=None):
    dp = dims_prev if dims_prev is not None else make_dims(x_prev, Bm_prev)
    d = dims if dims is not None else make_dims(x, Bm)
    _check("stree_replay_scan_sharded", lib().stree_replay_scan_sharded(
        ctypes.byref(dp), _ptr(x_prev), _ptr(dt_prev), _ptr(Bm_prev), _ptr(parent_prev), _ptr(path),
        _ptr(path_len), ctypes.byref(d), _ptr(x), _ptr(dt), _ptr(A), _ptr(Bm), _ptr(Cm), _ptr(D), _ptr(h),
        _ptr(parent), ctypes.byref(yout), _ptr(dev_status), _stream(stream)))


def stree_tree_scan_ex(x, dt, A, Bm, Cm, D, h0, parent, y, opts, dev_status=None, stream=None, dims=None):
    d = dims if dims is not None else make_dims(x, Bm)
    _check("stree_tree_scan_ex", lib().stree_tree_scan_ex(
        ctypes.byref(d), _ptr(x), _ptr(dt), _ptr(A), _ptr(Bm), _ptr(Cm), _ptr(D), _ptr(h0), _ptr(parent), _ptr(y),
        ctypes.byref(opts) if opts is not None else None, _ptr(dev_status), _stream(stream)))


def stree_commit_ex(x, dt, A, Bm, h0, parent, path, path_len, h_new, opts, dev_status=None, stream=None, dims=None):
    d = dims if dims is not None else make_dims(x, Bm)
    _check("stree_commit_ex", lib().stree_commit_ex(
        ctypes.byref(d), _ptr(x), _ptr(dt), _ptr(A), _ptr(Bm), _ptr(h0), _ptr(parent), _ptr(path), _ptr(path_len),
        _ptr(h_new), ctypes.byref(opts) if opts is not None else None, _ptr(dev_status), _stream(stream)))


def stree_replay_scan_ex(x_prev, dt_prev, Bm_prev, parent_prev, path, path_len, x, dt, A, Bm, Cm, D, h, parent, y,
                         opts, dev_status=None, stream=None, dims_prev=None, dims=None):
    dp = dims_prev if dims_prev is not None else make_dims(x_prev, Bm_prev)
    d = dims if dims is not None else make_dims(x, Bm)
    _check("stree_replay_scan_ex", lib().stree_replay_scan_ex(
        ctypes.byref(dp), _ptr(x_prev), _ptr(dt_prev), _ptr(Bm_prev), _ptr(parent_prev), _ptr(path),
        _ptr(path_len), ctypes.byref(d), _ptr(x), _ptr(dt), _ptr(A), _ptr(Bm), _ptr(Cm), _ptr(D), _ptr(h),
        _ptr(parent), _ptr(y), ctypes.byref(opts) if opts is not None else None, _ptr(dev_status), _stream(stream)))


def stree_set_scan_impl(impl: int):
    _check("stree_set_scan_impl", lib().stree_set_scan_impl(int(impl)))


def stree_set_launch_flags(flags: int):
    _check("stree_set_launch_flags", lib().stree_set_launch_flags(int(flags)))


def stree_scan_kernel_for(dims: stree_dims) -> int:
    return lib().stree_scan_kernel_for(ctypes.byref(dims))


def stree_commit_kernel_for(dims: stree_dims, has_h0: bool = True) -> int:
    return lib().stree_commit_kernel_for(ctypes.byref(dims), int(bool(has_h0)))


def make_conv_dims(u: torch.Tensor, weight: torch.Tensor) -> stree_conv_dims:
    B, T, C = u.shape
    return stree_conv_dims(B, T, C, weight.shape[1], io_code(u.dtype))


def stree_tree_conv(u, weight, bias, conv_state, parent, out, act=True, dev_status=None, stream=None, dims=None):
    d = dims if dims is not None else make_conv_dims(u, weight)
    _check("stree_tree_conv", lib().stree_tree_conv(ctypes.byref(d), _ptr(u), _ptr(weight), _ptr(bias),
                                                    _ptr(conv_state), _ptr(parent), int(bool(act)), _ptr(out),
                                                    _ptr(dev_status), _stream(stream)))


def stree_conv_commit(u, conv_state, parent, path, path_len, conv_state_new, width, dev_status=None, stream=None,
                      dims=None):
    B, T, C = u.shape
    d = dims if dims is not None else stree_conv_dims(B, T, C, int(width), io_code(u.dtype))
    _check("stree_conv_commit", lib().stree_conv_commit(ctypes.byref(d), _ptr(u), _ptr(conv_state), _ptr(parent),
                                                        _ptr(path), _ptr(path_len), _ptr(conv_state_new),
                                                        _ptr(dev_status), _stream(stream)))



def make_attn_dims(q: torch.Tensor, k_new: torch.Tensor, k_cache: torch.Tensor) -> stree_attn_dims:
    B, T, Hq, D = q.shape
    return stree_attn_dims(B, T, Hq, k_new.shape[2], D, k_cache.shape[1], io_code(q.dtype))


def stree_tree_attn(q, k_new, v_new, k_cache, v_cache, cache_len, parent, scale, o, dev_status=None, stream=None,
                    dims=None):
    d = dims if dims is not None else make_attn_dims(q, k_new, k_cache)
    _check("stree_tree_attn", lib().stree_tree_attn(ctypes.byref(d), _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(k_cache),
                                                    _ptr(v_cache), _ptr(cache_len), _ptr(parent), float(scale),
                                                    _ptr(o), _ptr(dev_status), _stream(stream)))


def stree_kv_commit(k_new, v_new, parent, path, path_len, k_cache, v_cache, cache_len, dev_status=None, stream=None,
                    dims=None):
    d = dims if dims is not None else make_attn_dims(k_new, k_new, k_cache)
    if dims is None:
        d.n_q_heads = k_new.shape[2]
    _check("stree_kv_commit", lib().stree_kv_commit(ctypes.byref(d), _ptr(k_new), _ptr(v_new), _ptr(parent),
                                                    _ptr(path), _ptr(path_len), _ptr(k_cache), _ptr(v_cache),
                                                    _ptr(cache_len), _ptr(dev_status), _stream(stream)))


def stree_attn_kernel_for(dims: stree_attn_dims) -> int:
    return lib().stree_attn_kernel_for(ctypes.byref(dims))


def stree_accept_mss(tokens, parent, p_target, q_draft, u_accept, u_bonus, path, path_len, bonus, dev_status=None,
                     stream=None):
    B, T = parent.shape
    V = p_target.shape[-1]
    _check("stree_accept_mss", lib().stree_accept_mss(_ptr(tokens), _ptr(parent), _ptr(p_target), _ptr(q_draft),
                                                      _ptr(u_accept), _ptr(u_bonus), B, T, V, _ptr(path),
                                                      _ptr(path_len), _ptr(bonus), _ptr(dev_status),
                                                      _stream(stream)))
