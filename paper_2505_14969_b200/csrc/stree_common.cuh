// stree_common.cuh — device helpers shared by the STree kernels (CUDA path only).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "../../include/stree.h"

namespace stree {

constexpr int kMaxNodes = STREE_MAX_NODES;          // T <= 256
constexpr int kMaxWords = (kMaxNodes + 31) / 32;    // mask words per row

// ---- Programmatic dependent launch (PDL) ----
// Every kernel calls pdl_wait() before its first global read or write of call arguments (setup that
// touches no argument memory — barrier init, TMEM allocation, descriptor prefetch — runs before it).
// The wait is followed by griddepcontrol.launch_dependents: the next grid in the stream may be
// scheduled only once every CTA of this grid has passed its own dependency wait (or exited), i.e. once
// the grid before this one has completed.  So a kernel launched by this library can overlap only the
// kernel immediately preceding it in the stream, never an older one — the scope of the
// STREE_LAUNCH_EARLY_* promises (include/stree.h).
__device__ __forceinline__ void pdl_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// effective dt of the *_ex options (include/stree.h): dt + dt_bias[h], then softplus (PyTorch's threshold 20)
struct DtX {
    const float* bias;   // [H] or NULL
    int softplus;
    __host__ static DtX from(const stree_scan_opts* o) {
        DtX x;
        x.bias = o ? o->dt_bias : nullptr;
        x.softplus = (o && o->dt_softplus) ? 1 : 0;
        return x;
    }
};
// softplus out of line: log1pf inlined at every dt_eff call site was ≈ 450 SASS instructions of the small-batch
// scan kernel's 4100 (instruction-fetch bound at batch 1), for an option the common path never takes
static __device__ __noinline__ float softplus_f(float v) { return v > 20.f ? v : log1pf(__expf(v)); }
__device__ __forceinline__ float dt_eff(const DtX& x, float raw, int h) {
    const float v = x.bias ? raw + x.bias[h] : raw;
    return x.softplus ? softplus_f(v) : v;
}

__device__ __forceinline__ void report(int32_t* dev_status, int code) {
    if (dev_status) atomicCAS(dev_status, 0, code);
}

template <typename T> __device__ __forceinline__ float to_f32(T v);
template <> __device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// Validates one tree (PAPER.md:90 precondition: parent[0] = -1, 0 <= parent[i] < i)
// and builds its ancestor-mask rows L[i] in shared memory by
// pointer jumping: after round k, row(i) holds the ancestors at distance < 2^k
// and jmp(i) is the 2^k-th ancestor, so ceil(log2 T) rounds give the full
// root-to-i path.  All threads of the block must call this.
//   sp    : parent[T] already in smem (int)
//   rows  : [T][W] uint32 output; rows2: [T][W] scratch; jmp/jmp2: [T] int scratch
// Returns 0 or the device status code (1 bad root / 2 bad parent); rows are
// zero for an invalid tree.
__device__ __forceinline__ int build_tree_rows(const int* sp, int T, int W, uint32_t* rows,
                                               uint32_t* rows2, int* jmp, int* jmp2) {
    const int tid = threadIdx.x, nt = blockDim.x;
    int bad = 0;
    for (int i = tid; i < T; i += nt) {
        int p = sp[i];
        if (i == 0) { if (p != -1) bad = max(bad, 1); }
        else if (p < 0 || p >= i) bad = max(bad, 2);
    }
    // block-wide max of the error code
    int any1 = __syncthreads_or(bad == 1);
    int any2 = __syncthreads_or(bad == 2);
    int code = any1 ? 1 : (any2 ? 2 : 0);
    if (code) {
        for (int k = tid; k < T * W; k += nt) rows[k] = 0u;
        __syncthreads();
        return code;
    }
    for (int i = tid; i < T; i += nt) {
        for (int w = 0; w < W; ++w) rows[i * W + w] = (w == (i >> 5)) ? (1u << (i & 31)) : 0u;
        jmp[i] = sp[i];
    }
    __syncthreads();
    uint32_t* ra = rows; uint32_t* rb = rows2;
    int* ja = jmp; int* jb = jmp2;
    int rounds = 0;
    while ((1 << rounds) < T) ++rounds;
    for (int r = 0; r < rounds; ++r) {
        for (int i = tid; i < T; i += nt) {
            int j = ja[i];
            for (int w = 0; w < W; ++w) rb[i * W + w] = ra[i * W + w] | (j >= 0 ? ra[j * W + w] : 0u);
            jb[i] = j >= 0 ? ja[j] : -1;
        }
        __syncthreads();
        uint32_t* t = ra; ra = rb; rb = t;
        int* tj = ja; ja = jb; jb = tj;
    }
    if (ra != rows) {
        for (int k = tid; k < T * W; k += nt) rows[k] = ra[k];
        __syncthreads();
    }
    return 0;
}

__device__ __forceinline__ bool mask_bit(const uint32_t* rows, int W, int i, int j) {
    return (rows[i * W + (j >> 5)] >> (j & 31)) & 1u;
}

}  // namespace stree

// launch options (stree_set_launch_flags), read by every launcher
extern "C" uint32_t stree_launch_flags_get();
// scan options of the *_ex call in progress on this thread (NULL: plain call), read by the scan / commit launchers
extern "C" const stree_scan_opts* stree_scan_opts_get();

namespace stree {
// cudaLaunchKernelEx with the programmatic-stream-serialization attribute when PDL is enabled
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (stree_launch_flags_get() & STREE_LAUNCH_PDL) ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
}  // namespace stree
