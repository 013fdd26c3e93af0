"""CPU oracle for the STree tree-verify hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It shares no code with
``paper_2505_14969_b200`` and the product path never imports it.

The arithmetic lives in ``stree_oracle.c`` (fp64, plain definition, see its
header for the paper passages).  This wrapper only widens inputs to float64
and marshals arrays.  Pins: tests/test_oracle_pins.py (closed forms, the
hand-worked example in tests/golden/, the paper's matrix form re-derived
independently in numpy, the textbook Mamba-2 chain scan, brute force over
all small trees).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "stree_oracle.c")
_lib = None


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _host_key() -> str:
    """-march=native code is specific to the host's ISA: the library name carries a hash of the CPU
    model and flags, so a build made on one host (the CPU container) is never executed on another
    (the GPU box), where it is rebuilt on first use (gcc is in both images)."""
    import hashlib
    flags = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    flags = line
                    break
    except OSError:
        pass
    return hashlib.sha1((cpu_model() + flags).encode()).hexdigest()[:10]


_LIB = os.path.join(_HERE, f"libstree_oracle.{_host_key()}.so")


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc -O3 -march=native -fopenmp).  No -ffast-math: fp64 semantics kept
    (gcc does not contract a*b+c into an FMA across statements without -ffp-contract=fast in ISO C mode)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-march=native", "-ffp-contract=off", "-fopenmp", "-fPIC",
                               "-shared", "-std=c11", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i = ctypes.c_int
        lib.oracle_build_mask.argtypes = [P, i, i, P, P, P]
        lib.oracle_tree_scan.argtypes = [i, i, i, i, i, i, P, P, P, P, P, P, P, P, P, P]
        lib.oracle_accept.argtypes = [P, P, P, i, i, P, P, P, P]
        lib.oracle_commit.argtypes = [i, i, i, i, i, i, P, P, P, P, P, P, P, P, P, P]
        lib.oracle_num_threads.argtypes = []
        lib.oracle_set_threads.argtypes = [i]
        lib.oracle_tree_conv.argtypes = [i, i, i, i, P, P, P, P, P, i, P, P]
        lib.oracle_conv_commit.argtypes = [i, i, i, i, P, P, P, P, P, P, P]
        for f in (lib.oracle_build_mask, lib.oracle_tree_scan, lib.oracle_accept,
                  lib.oracle_commit, lib.oracle_num_threads, lib.oracle_tree_conv, lib.oracle_conv_commit):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def num_threads() -> int:
    return _load().oracle_num_threads()


def set_threads(n: int) -> None:
    """OpenMP thread count of later oracle calls (n <= 0: the runtime default)."""
    _load().oracle_set_threads(int(n))


def build_mask(parent):
    """parent [B][T] -> (mask uint32 [B][T][ceil(T/32)], depth int32 [B][T], status [B])."""
    parent = _i32(parent)
    B, T = parent.shape
    W = (T + 31) // 32
    mask = np.zeros((B, T, W), np.uint32)
    depth = np.zeros((B, T), np.int32)
    st = np.zeros(B, np.int32)
    _load().oracle_build_mask(_p(parent), B, T, _p(mask), _p(depth), _p(st))
    return mask, depth, st


def tree_scan(x, dt, A, Bm, Cm, D, h0, parent, n_groups=1):
    """Float inputs (any float dtype, widened exactly to fp64).
    x[B][T][H][P], dt[B][T][H], A[H], Bm/Cm[B][T][G][N], D[H] or None,
    h0[B][H][P][N] or None, parent[B][T] -> (y fp64 [B][T][H][P], status[B])."""
    x, dt, A, Bm, Cm = map(_f64, (x, dt, A, Bm, Cm))
    D, h0 = _f64(D), _f64(h0)
    parent = _i32(parent)
    B, T, H, P = x.shape
    N = Bm.shape[-1]
    y = np.zeros((B, T, H, P), np.float64)
    st = np.zeros(B, np.int32)
    rc = _load().oracle_tree_scan(B, T, H, P, N, n_groups, _p(x), _p(dt), _p(A), _p(Bm), _p(Cm),
                                  _p(D), _p(h0), _p(parent), _p(y), _p(st))
    if rc:
        raise RuntimeError(f"oracle internal inconsistency rc={rc}")
    return y, st


def accept(tokens, parent, vtok):
    """-> (path int32 [B][T] (-1 padded), path_len [B], bonus [B], status [B])."""
    tokens, parent, vtok = _i32(tokens), _i32(parent), _i32(vtok)
    B, T = parent.shape
    path = np.full((B, T), -1, np.int32)
    plen = np.zeros(B, np.int32)
    bonus = np.zeros(B, np.int32)
    st = np.zeros(B, np.int32)
    _load().oracle_accept(_p(tokens), _p(parent), _p(vtok), B, T, _p(path), _p(plen), _p(bonus), _p(st))
    return path, plen, bonus, st


def commit(x, dt, A, Bm, h0, path, path_len, parent=None, n_groups=1):
    """-> (h_new fp64 [B][H][P][N], status [B])."""
    x, dt, A, Bm, h0 = map(_f64, (x, dt, A, Bm, h0))
    path, path_len = _i32(path), _i32(path_len)
    parent = None if parent is None else _i32(parent)
    B, T, H, P = x.shape
    N = Bm.shape[-1]
    h_new = np.zeros((B, H, P, N), np.float64)
    st = np.zeros(B, np.int32)
    _load().oracle_commit(B, T, H, P, N, n_groups, _p(x), _p(dt), _p(A), _p(Bm), _p(h0), _p(parent),
                          _p(path), _p(path_len), _p(h_new), _p(st))
    return h_new, st


def scan_problem(prob):
    """Convenience: run tree_scan on a gen.inputs.Problem (bf16 widened exactly)."""
    return tree_scan(prob.io_as_f32("x"), prob.dt, prob.A, prob.io_as_f32("Bm"), prob.io_as_f32("Cm"),
                     prob.D, prob.h0, prob.parent, n_groups=prob.dims.n_groups)


def commit_problem(prob, path, path_len, use_parent=True):
    return commit(prob.io_as_f32("x"), prob.dt, prob.A, prob.io_as_f32("Bm"), prob.h0, path, path_len,
                  parent=prob.parent if use_parent else None, n_groups=prob.dims.n_groups)


def effective_dt(dt, dt_bias=None, dt_softplus=False):
    """The scan options' discretisation (include/stree.h stree_scan_opts; Mamba-2, reading R9 with the raw
    projection as input): dt <- dt + dt_bias[h], then softplus(v) = log(1 + e^v), in fp64."""
    v = _f64(dt)
    if dt_bias is not None:
        v = v + _f64(dt_bias)[None, None, :]
    return np.logaddexp(0.0, v) if dt_softplus else v


def tree_scan_ex(x, dt, A, Bm, Cm, D, h0, parent, n_groups=1, dt_bias=None, dt_softplus=False,
                 d_per_channel=False):
    """tree_scan with the scan options: the effective dt above, and D of shape [H][P] when d_per_channel
    (y_i += D[h][p] x_i[p], P:45 with a skip weight per channel) — the recurrence itself is unchanged."""
    dte = effective_dt(dt, dt_bias, dt_softplus)
    if not d_per_channel:
        return tree_scan(x, dte, A, Bm, Cm, D, h0, parent, n_groups=n_groups)
    y, st = tree_scan(x, dte, A, Bm, Cm, None, h0, parent, n_groups=n_groups)
    if D is not None:
        y = y + _f64(D)[None, None, :, :] * _f64(x)
        y[st != 0] = 0.0   # invalid trees stay zero-filled
    return y, st


def commit_ex(x, dt, A, Bm, h0, path, path_len, parent=None, n_groups=1, dt_bias=None, dt_softplus=False):
    """commit along the accepted path with the effective dt (the same transform as the scan that verified it)."""
    return commit(x, effective_dt(dt, dt_bias, dt_softplus), A, Bm, h0, path, path_len, parent=parent,
                  n_groups=n_groups)


def tree_conv(u, weight, bias, state, parent, act=True):
    """Tree-causal depthwise conv1d (stree_oracle.c, reading R-conv).
    u [B][T][C], weight [C][W], bias [C] or None, state [B][W-1][C] or None, parent [B][T]
    -> (out fp64 [B][T][C], status [B])."""
    u, weight = _f64(u), _f64(weight)
    bias = None if bias is None else _f64(bias)
    state = None if state is None else _f64(state)
    parent = _i32(parent)
    B, T, C = u.shape
    W = weight.shape[1]
    out = np.zeros((B, T, C), np.float64)
    st = np.zeros(B, np.int32)
    _load().oracle_tree_conv(B, T, C, W, _p(u), _p(weight), _p(bias), _p(state), _p(parent), int(bool(act)),
                             _p(out), _p(st))
    return out, st


def conv_commit(u, state, path, path_len, W, parent=None):
    """Conv-state commit: last W-1 inputs of state ++ u[path] -> (state_new fp64 [B][W-1][C], status [B])."""
    u = _f64(u)
    state = None if state is None else _f64(state)
    path, path_len = _i32(path), _i32(path_len)
    parent = None if parent is None else _i32(parent)
    B, T, C = u.shape
    out = np.zeros((B, W - 1, C), np.float64)
    st = np.zeros(B, np.int32)
    _load().oracle_conv_commit(B, T, C, W, _p(u), _p(state), _p(parent), _p(path), _p(path_len), _p(out), _p(st))
    return out, st

