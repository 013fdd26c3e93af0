"""C-ABI library: loads, exports every symbol include/stree.h declares, and the
host-side validation returns the documented status codes (no GPU needed:
these calls are rejected before any CUDA work)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2505_14969_b200 import build as bld
    bld.build()
    from paper_2505_14969_b200 import binding
    return binding.lib()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "stree.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(stree_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    syms = declared_symbols()
    assert {"stree_build_mask", "stree_tree_scan", "stree_accept", "stree_commit"} <= set(syms)
    for s in syms:
        assert hasattr(L, s), s


def test_status_strings_and_version(L):
    from paper_2505_14969_b200 import binding
    assert binding.status_string(0) == "ok"
    assert binding.status_string(2) == "bad shape"
    assert "sm_100a" in binding.version()


def test_host_validation_codes(L):
    from paper_2505_14969_b200 import binding as b
    vp = ctypes.c_void_p
    fake = vp(0x10000)  # never dereferenced: every call below fails validation first
    # empty problems are successful no-ops
    assert L.stree_build_mask(None, 0, 5, None, None, None, None) == 0
    assert L.stree_build_mask(None, 3, 0, None, None, None, None) == 0
    # NULL / shape errors
    assert L.stree_build_mask(None, 1, 5, None, None, None, None) == 1
    assert L.stree_build_mask(fake, 1, 257, fake, None, None, None) == 2
    assert L.stree_accept(fake, fake, None, 1, 4, fake, fake, fake, None, None) == 1
    d = b.stree_dims(1, 4, 2, 8, 8, 1, b.STREE_F32)
    assert L.stree_tree_scan(None, fake, fake, fake, fake, fake, None, None, fake, fake, None, None) == 1
    assert L.stree_tree_scan(ctypes.byref(d), None, fake, fake, fake, fake, None, None, fake, fake, None, None) == 1
    bad = b.stree_dims(1, 4, 3, 8, 8, 2, b.STREE_F32)  # H % G != 0
    assert L.stree_tree_scan(ctypes.byref(bad), fake, fake, fake, fake, fake, None, None, fake, fake, None, None) == 2
    big = b.stree_dims(1, 300, 2, 8, 8, 1, b.STREE_F32)
    assert L.stree_tree_scan(ctypes.byref(big), fake, fake, fake, fake, fake, None, None, fake, fake, None, None) == 2
    dt_bad = b.stree_dims(1, 4, 2, 8, 8, 1, 7)
    assert L.stree_tree_scan(ctypes.byref(dt_bad), fake, fake, fake, fake, fake, None, None, fake, fake, None,
                             None) == 3
    mis = vp(0x10004)
    assert L.stree_tree_scan(ctypes.byref(d), mis, fake, fake, fake, fake, None, None, fake, fake, None, None) == 4
    assert L.stree_commit(ctypes.byref(d), fake, fake, fake, fake, fake, None, fake, fake, mis, None, None) == 4
    # partial overlap of h0 / h_new rejected (in-place allowed)
    assert L.stree_commit(ctypes.byref(d), fake, fake, fake, fake, vp(0x10000), None, fake, fake, vp(0x10010),
                          None, None) == 2


def test_scan_kernel_selection(L):
    from paper_2505_14969_b200 import binding as b
    d = b.stree_dims(1, 7, 1, 4, 4, 1, b.STREE_F32)
    assert b.stree_scan_kernel_for(d) == 1          # fp32 toy -> SIMT
    b.stree_set_scan_impl(b.STREE_SCAN_SIMT)
    big = b.stree_dims(16, 64, 80, 64, 128, 1, b.STREE_BF16)
    assert b.stree_scan_kernel_for(big) == 1
    b.stree_set_scan_impl(b.STREE_SCAN_AUTO)
    assert b.stree_scan_kernel_for(big) in (1, 2)
    t100 = b.stree_dims(4, 100, 80, 64, 128, 1, b.STREE_BF16)
    assert b.stree_scan_kernel_for(t100) == 3       # 128-node tcgen05 kernel
    t200 = b.stree_dims(4, 200, 80, 64, 128, 1, b.STREE_BF16)
    assert b.stree_scan_kernel_for(t200) == 3       # two 128-row tiles
    assert b.stree_scan_kernel_for(b.stree_dims(4, 200, 80, 64, 64, 1, b.STREE_BF16)) == 1   # N = 64: SIMT
    with pytest.raises(b.StreeError):
        b.stree_set_scan_impl(9)


def test_host_validation_next_rows(L):
    """§8(f) calls: tree attention, KV commit, MSS verification, tree conv — host-side codes."""
    from paper_2505_14969_b200 import binding as b
    vp = ctypes.c_void_p
    fake, mis = vp(0x10000), vp(0x10004)
    f = ctypes.c_float(0.125)
    d = b.stree_attn_dims(2, 16, 32, 8, 128, 1024, b.STREE_BF16)
    z = b.stree_attn_dims(0, 16, 32, 8, 128, 1024, b.STREE_BF16)
    assert L.stree_tree_attn(ctypes.byref(z), None, None, None, None, None, None, None, f, None, None, None) == 0
    assert L.stree_tree_attn(None, fake, fake, fake, fake, fake, fake, fake, f, fake, None, None) == 1
    assert L.stree_tree_attn(ctypes.byref(d), fake, fake, fake, fake, fake, None, fake, f, fake, None, None) == 1
    gqa = b.stree_attn_dims(2, 16, 30, 8, 128, 1024, b.STREE_BF16)      # Hq % Hkv != 0
    assert L.stree_tree_attn(ctypes.byref(gqa), fake, fake, fake, fake, fake, fake, fake, f, fake, None, None) == 2
    wide = b.stree_attn_dims(2, 16, 32, 8, 512, 1024, b.STREE_BF16)     # D > 256
    assert L.stree_tree_attn(ctypes.byref(wide), fake, fake, fake, fake, fake, fake, fake, f, fake, None, None) == 2
    dtb = b.stree_attn_dims(2, 16, 32, 8, 128, 1024, 9)
    assert L.stree_tree_attn(ctypes.byref(dtb), fake, fake, fake, fake, fake, fake, fake, f, fake, None, None) == 3
    assert L.stree_tree_attn(ctypes.byref(d), mis, fake, fake, fake, fake, fake, fake, f, fake, None, None) == 4
    # kernel selection: bf16 D=128 with (Hq/Hkv) | 128 -> tcgen05; fp32 or grp=3 -> SIMT
    assert b.stree_attn_kernel_for(d) == 2
    assert b.stree_attn_kernel_for(b.stree_attn_dims(2, 16, 32, 8, 128, 1024, b.STREE_F32)) == 1
    assert b.stree_attn_kernel_for(b.stree_attn_dims(2, 16, 12, 4, 128, 1024, b.STREE_BF16)) == 1
    # KV commit: NULL / row size not a multiple of 4 bytes / alignment
    assert L.stree_kv_commit(ctypes.byref(d), fake, fake, None, fake, fake, fake, fake, None, None, None) == 1
    odd = b.stree_attn_dims(2, 16, 1, 1, 1, 64, b.STREE_BF16)             # 2-byte rows
    assert L.stree_kv_commit(ctypes.byref(odd), fake, fake, None, fake, fake, fake, fake, fake, None, None) == 2
    assert L.stree_kv_commit(ctypes.byref(d), mis, fake, None, fake, fake, fake, fake, fake, None, None) == 4
    # MSS: vocabulary bound, NULLs, empty
    i32 = ctypes.c_int32
    assert L.stree_accept_mss(fake, fake, fake, fake, fake, fake, i32(2), i32(8), i32(200000), fake, fake, fake,
                              None, None) == 2
    assert L.stree_accept_mss(fake, fake, None, fake, fake, fake, i32(2), i32(8), i32(1000), fake, fake, fake,
                              None, None) == 1
    assert L.stree_accept_mss(None, None, None, None, None, None, i32(0), i32(8), i32(1000), None, None, None,
                              None, None) == 0
    # tree conv: width out of range, channels not a multiple of the vector width, misaligned weight
    cd = b.stree_conv_dims(2, 16, 5376, 4, b.STREE_BF16)
    w5 = b.stree_conv_dims(2, 16, 5376, 5, b.STREE_BF16)
    assert L.stree_tree_conv(ctypes.byref(w5), fake, fake, None, None, fake, 1, fake, None, None) == 2
    c7 = b.stree_conv_dims(2, 16, 5377, 4, b.STREE_BF16)
    assert L.stree_tree_conv(ctypes.byref(c7), fake, fake, None, None, fake, 1, fake, None, None) == 2
    assert L.stree_tree_conv(ctypes.byref(cd), fake, mis, None, None, fake, 1, fake, None, None) == 4


def test_sharded_yout_validation(L):
    """stree_*_sharded (include/stree.h, head-sharded layers): the stree_yout descriptor is validated before
    any CUDA work; shapes the tcgen05 kernels do not serve are STREE_ERR_UNSUPPORTED (no silent fallback)."""
    from paper_2505_14969_b200 import binding as b
    vp = ctypes.c_void_p
    fake = vp(0x10000)
    d = b.stree_dims(1, 16, 8, 64, 128, 1, b.STREE_BF16)
    good = b.make_yout([0x20000, 0x30000], heads_total=16, head_offset=8)
    args = (ctypes.byref(d), fake, fake, fake, fake, fake, None, fake, fake)
    assert L.stree_tree_scan_sharded(*args, None, None, None) == 1                       # NULL yout
    zero = b.stree_yout()
    assert L.stree_tree_scan_sharded(*args, ctypes.byref(zero), None, None) == 2         # n_peers = 0
    over = b.make_yout([0x20000], heads_total=15, head_offset=8)
    assert L.stree_tree_scan_sharded(*args, ctypes.byref(over), None, None) == 2         # shard past heads_total
    nullp = b.make_yout([0x20000, 0], heads_total=16, head_offset=8)
    assert L.stree_tree_scan_sharded(*args, ctypes.byref(nullp), None, None) == 1        # NULL peer
    mis = b.make_yout([0x20008], heads_total=16, head_offset=8)
    assert L.stree_tree_scan_sharded(*args, ctypes.byref(mis), None, None) == 4          # misaligned peer
    f32 = b.stree_dims(1, 16, 8, 64, 128, 1, b.STREE_F32)
    assert L.stree_tree_scan_sharded(ctypes.byref(f32), fake, fake, fake, fake, fake, None, fake, fake,
                                     ctypes.byref(good), None, None) == 5                 # SIMT shape: unsupported
    with pytest.raises(ValueError):
        b.make_yout([0x20000] * 9, heads_total=16, head_offset=0)
    dp = b.stree_dims(1, 16, 8, 64, 128, 1, b.STREE_BF16)
    rargs = (ctypes.byref(dp), fake, fake, fake, None, fake, fake, ctypes.byref(d), fake, fake, fake, fake, fake,
             None, fake, fake)
    assert L.stree_replay_scan_sharded(*rargs, None, None, None) == 1
    assert L.stree_replay_scan_sharded(*rargs, ctypes.byref(over), None, None) == 2
