"""stree-b200: B200-native (sm_100a) tree-verify hot path of STree (arXiv 2505.14969).

The product is the C-ABI library ``libstree.so`` (include/stree.h); this
package is its thin Python binding (``binding``) plus allocation helpers
(``api``).  See DESIGN.md.
"""
from .binding import (  # noqa: F401
    StreeError, stree_accept, stree_replay_scan, stree_set_launch_flags, stree_build_mask, stree_commit, stree_dims, stree_set_scan_impl,
    stree_scan_kernel_for, stree_tree_scan, status_string, version,
    STREE_SCAN_AUTO, STREE_SCAN_SIMT, STREE_SCAN_TC, STREE_BF16, STREE_F32,
)
