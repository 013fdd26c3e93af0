// K2 stree_tree_scan on tcgen05 tensor cores (placeholder until the kernel lands).
#include "stree_common.cuh"

extern "C" int stree_tc_supports(const stree_dims* d) { (void)d; return 0; }

extern "C" int stree_launch_scan_tc(const stree_dims*, const void*, const float*, const float*, const void*,
                                    const void*, const float*, const float*, const int32_t*, void*, int32_t*,
                                    cudaStream_t) {
    return (int)cudaErrorNotSupported;
}
