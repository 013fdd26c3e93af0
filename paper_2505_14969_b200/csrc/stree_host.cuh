// stree_host.cuh — host-side helpers shared by the launchers (not device code):
//  * TMA tensor-map encoding with a per-process cache keyed by (pointer, shape, box): an eager call
//    re-uses the descriptors of an earlier call on the same buffers instead of re-encoding them
//    (cuTensorMapEncodeTiled costs ~1-2 us of host time per map);
//  * the SM count and a once-per-(kernel, device) dynamic shared-memory attribute.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace stree {
namespace host {

// 2-D tiled map: dims (inner, outer), row pitch row_bytes, box (box_inner, box_outer), SWIZZLE_128B
// (or no swizzle: the box lands row after row, box_inner elements each).
bool tmap_2d(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t inner, uint64_t outer,
             uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer, bool swizzle128 = true);
// 4-D bf16 map (d0 contiguous), box (64, b1, b2, 1), SWIZZLE_128B (tree attention).
bool tmap_4d_bf16(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t d3, uint32_t b1,
                  uint32_t b2);
// number of cached maps (tests / debugging)
size_t tmap_cache_size();
void tmap_cache_clear();

int num_sms();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (function, device, size)
cudaError_t smem_attr(const void* func, int bytes);

}  // namespace host
}  // namespace stree
