"""Comparison helpers for parity tests (tolerances: BASELINE north_star;
metric: SURVEY.md §8(c) C20)."""
import numpy as np

TOL_F32 = 1e-4   # fp32 path
TOL_BF16 = 2e-2  # bf16 inputs, fp32 accumulation


def blockwise_relerr(got, ref, block_axes):
    """Normwise rel-err per block (blocks = all indices except block_axes reduced).
    Returns (max normwise rel err, max of max|a-b|/max|b|)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    diff = got - ref
    num = np.sqrt((diff ** 2).sum(axis=block_axes))
    den = np.sqrt((ref ** 2).sum(axis=block_axes))
    mx = np.abs(diff).max(axis=block_axes)
    mref = np.abs(ref).max(axis=block_axes)
    ok = den > 0
    r1 = float((num[ok] / den[ok]).max()) if ok.any() else float(num.max())
    r2 = float((mx[ok] / mref[ok]).max()) if ok.any() else float(mx.max())
    return r1, r2


def assert_y_close(y_gpu, y_ref, tol):
    """y [B][T][H][P]: blocks are (tree, head)."""
    r1, r2 = blockwise_relerr(y_gpu, y_ref, (1, 3))
    assert r1 <= tol and r2 <= tol, f"y rel-err normwise {r1:.3e} max {r2:.3e} > tol {tol:.0e}"
    return r1, r2


def assert_h_close(h_gpu, h_ref, tol):
    """h [B][H][P][N]: blocks are (tree, head)."""
    r1, r2 = blockwise_relerr(h_gpu, h_ref, (2, 3))
    assert r1 <= tol and r2 <= tol, f"h rel-err normwise {r1:.3e} max {r2:.3e} > tol {tol:.0e}"
    return r1, r2


def assert_conv_close(o_gpu, o_ref, tol):
    """tree conv output [B][T][C]: blocks are (tree, channel)."""
    r1, r2 = blockwise_relerr(o_gpu, o_ref, (1,))
    assert r1 <= tol and r2 <= tol, f"conv rel-err normwise {r1:.3e} max {r2:.3e} > tol {tol:.0e}"
    return r1, r2
