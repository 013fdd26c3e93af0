// K5 stree_tree_conv / K6 stree_conv_commit: tree-causal depthwise conv1d over the xBC channels
// and its conv-state commit (reading R-conv).
//
//   seq_i        = conv_state[b] (W-1 rows, oldest first) ++ u[b][root .. i]
//   out[b][i][c] = act( bias[c] + sum_{w<W} weight[c][w] * seq_i[len - W + w][c] )
//
// HBM-bound (intensity ~W FLOP per 4 bytes).  One CTA per (tree, block of 16 16-byte channel
// chunks): the tree's rows of that channel block (and the conv state) are read once (cp.async),
// into shared memory; every node then reads its W-1 ancestors from there (the ancestor chain is
// walked in shared memory, stepping into the state rows above the root), and the output row is
// written once, coalesced.
#include "stree_common.cuh"
#include "stree_host.cuh"

namespace stree {
namespace conv {

constexpr int kChunks = 32;     // 16-byte channel chunks per conv-commit warp (lane = chunk)
#ifndef STREE_CONV_KC
#define STREE_CONV_KC 8
#endif
constexpr int kConvKC = STREE_CONV_KC;     // chunks per tree-conv CTA (tree_conv_kernel)
#ifndef STREE_CONV_MINB
#define STREE_CONV_MINB 10   // min CTAs per SM at KC = 8 (register cap; 13 / 16, which would let two layers be resident, measured 9.3 / 9.4 vs 6.5 us)
#endif
#ifndef STREE_CONV_GROUPS
#define STREE_CONV_GROUPS 4
#endif
constexpr int kConvGroups = STREE_CONV_GROUPS;   // cp.async node groups per tree-conv CTA

template <typename IO>
struct Pack;
template <>
struct Pack<__nv_bfloat16> {
    static constexpr int V = 8;
    __device__ static void unpack(const uint4& v, float* f) {
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            f[2 * q] = __uint_as_float(w[q] << 16);
            f[2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
        }
    }
    __device__ static uint4 pack(const float* f) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * q], f[2 * q + 1]);
            w[q] = *reinterpret_cast<uint32_t*>(&h);
        }
        return make_uint4(w[0], w[1], w[2], w[3]);
    }
};
template <>
struct Pack<float> {
    static constexpr int V = 4;
    __device__ static void unpack(const uint4& v, float* f) {
        f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y);
        f[2] = __uint_as_float(v.z); f[3] = __uint_as_float(v.w);
    }
    __device__ static uint4 pack(const float* f) {
        return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
    }
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
// packed fp32 pairs (FFMA2: two fused multiply-adds per instruction on sm_100a)
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void f2unpack(uint64_t r, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
// the 16-byte chunk as V/2 packed fp32 pairs (bf16: w << 16 is the low element, w & 0xffff0000 the high one)
template <typename IO>
__device__ __forceinline__ void unpack2(const uint4& v, uint64_t* p);
template <>
__device__ __forceinline__ void unpack2<__nv_bfloat16>(const uint4& v, uint64_t* p) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) p[q] = f2pack(__uint_as_float(w[q] << 16), __uint_as_float(w[q] & 0xFFFF0000u));
}
template <>
__device__ __forceinline__ void unpack2<float>(const uint4& v, uint64_t* p) {
    p[0] = f2pack(__uint_as_float(v.x), __uint_as_float(v.y));
    p[1] = f2pack(__uint_as_float(v.z), __uint_as_float(v.w));
}

__host__ __device__ constexpr size_t tree_conv_smem(int T, int W, int KC) {
    return (size_t)kMaxNodes * 4 + (size_t)((W - 1) + T) * KC * 16;
}

// SiLU from h = z/2 (the kernel folds the exact factor 1/2 into the weights and bias): silu(z) = z·σ(z) =
// h + h·tanh(h).  bf16 outputs: one MUFU op and one FMA (tanh.approx's 2^-11 error is far below the bf16
// rounding of the output); fp32 outputs keep the exp + division form (the 1e-4 path)
template <typename IO>
__device__ __forceinline__ float silu_h(float h);
template <>
__device__ __forceinline__ float silu_h<__nv_bfloat16>(float h) {
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(h));
    return fmaf(h, t, h);
}
template <>
__device__ __forceinline__ float silu_h<float>(float h) { return __fdividef(2.f * h, 1.f + __expf(-2.f * h)); }

// One CTA per (tree, block of KC 16-byte channel chunks), 8·KC threads: thread = (chunk ch = tid % KC, node
// slot ns = tid / KC); slot ns computes nodes ns, ns + 8, ...  KC = 8 (64 threads, 1344 CTAs at the 2.7B
// shape, all resident): tools/conv_sweep.sh measured KC = 8 / 16 / 32 at 6.5 / 6.7 / 8.3 µs per call (4 groups).
// Under STREE_LAUNCH_EARLY_TREE the weights, bias and parents are read, and every node's window tabulated,
// before the dependency wait (EARLY_STATE: the conv-state rows too), so only the tree's rows remain after it.
// The rows arrive in kGroups cp.async groups of consecutive nodes; group k is computed and stored while the
// later groups are still in flight (topological order: a node's window only reaches back to earlier groups),
// so the reads and writes of the layer overlap in HBM instead of running as two bursts.
__device__ __forceinline__ void cp_async_wait_n(int n) {   // n is a compile-time constant after unrolling
    switch (n) {
        case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
        case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
        case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
        case 3: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
        case 4: asm volatile("cp.async.wait_group 4;" ::: "memory"); break;
        case 5: asm volatile("cp.async.wait_group 5;" ::: "memory"); break;
        case 6: asm volatile("cp.async.wait_group 6;" ::: "memory"); break;
        default: asm volatile("cp.async.wait_group 7;" ::: "memory"); break;
    }
}
template <typename IO, int W, int KC, bool ACT, int kGroups>
__global__ void __launch_bounds__(8 * KC, KC <= 8 ? STREE_CONV_MINB : KC <= 16 ? 5 : 3) tree_conv_kernel(const IO* __restrict__ u, const float* __restrict__ weight,
                                                                 const float* __restrict__ bias, const IO* __restrict__ state,
                                                                 const int32_t* __restrict__ parent,
                                                                 IO* __restrict__ out, int T, int C, int32_t* dev_status,
                                                                 int early_tree, int early_state) {
    constexpr int V = Pack<IO>::V, NT = 8 * KC, kSlots = 8;
    static_assert(W <= 4, "window");
    extern __shared__ __align__(16) unsigned char sm[];
    int* sp = reinterpret_cast<int*>(sm);                                   // parent[T]
    unsigned char* rows = sm + kMaxNodes * 4;                               // [(W-1) + T][KC] 16-byte chunks
    __shared__ int s_bad;
    const int b = blockIdx.y, c0 = blockIdx.x * KC * V;
    const int tid = threadIdx.x, ch = tid % KC, ns = tid / KC;
    const bool cv = c0 + ch * V < C;                                       // this thread's chunk exists
    if (tid == 0) s_bad = 0;
    // the block's weights and bias (with ACT pre-scaled by the 1/2 of silu_h; zero for absent channels):
    // coalesced loads issued together with the parent and staging loads below (one memory latency for all
    // of them), then through shared memory, [w][v][chunk] so the per-thread reads are conflict-free
    __shared__ float s_w[4 * 8 * KC];
    __shared__ float s_b[8 * KC];
    __shared__ __align__(16) int s_win[kMaxNodes * 4];   // per node: byte offsets of its W window rows
    constexpr float hs = ACT ? 0.5f : 1.f;
    if (!early_tree) pdl_wait();
    const int nc = min(KC * V, C - c0);   // channels of this block (nc * W <= 4 * NT)
    float wv[4], bv;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int k = tid + q * NT;
        wv[q] = k < nc * W ? hs * __ldg(weight + (size_t)c0 * W + k) : 0.f;
    }
    bv = (tid < nc && bias) ? hs * __ldg(bias + c0 + tid) : 0.f;
    for (int i = tid; i < T; i += NT) sp[i] = parent[(size_t)b * T + i];
    // stage the state rows and the tree's rows of this channel block with cp.async (global -> shared, no
    // register round trip); missing state rows and absent chunks are zero-filled (source size 0)
    const uint32_t cbytes = cv ? 16u : 0u;
    const size_t cofs = (size_t)c0 + (cv ? ch * V : 0);
    const uint32_t rbase = (uint32_t)__cvta_generic_to_shared(rows) + ch * 16;
    auto stage_state = [&]() {
        if (ns < W - 1)
            cp_async16(rbase + ns * KC * 16, (state ? state + ((size_t)b * (W - 1) + ns) * C : u) + cofs,
                       state ? cbytes : 0u);
    };
    const int gs = ((T + 8 * kGroups - 1) / (8 * kGroups)) * 8;   // nodes per group (a multiple of the 8 slots)
    auto stage_rows = [&]() {
#pragma unroll
        for (int k = 0; k < kGroups; ++k) {
            const int n1 = min((k + 1) * gs, T);
            for (int n = k * gs + ns; n < n1; n += kSlots)
                cp_async16(rbase + ((W - 1) + n) * KC * 16, u + ((size_t)b * T + n) * C + cofs, cbytes);
            cp_async_commit();
        }
    };
    if (early_tree && early_state) stage_state();   // caller's promise: conv_state not written by the preceding kernel
    if (!early_tree) {
        stage_state();
        stage_rows();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int k = tid + q * NT;
        if (k < KC * V * W) {
            const int cl = k / W, w = k % W;
            s_w[(w * V + cl % V) * KC + cl / V] = wv[q];
        }
    }
    if (tid < KC * V) s_b[(tid % V) * KC + tid / V] = bv;
    // PAPER.md:90 precondition: parent[0] = -1, 0 <= parent[i] < i (root error takes precedence); the same
    // pass tabulates every node's window rows as byte offsets (oldest first: ancestors at distance W-1 .. 1,
    // then the node; above the root the chain continues into the state rows W-2, W-3, ...) so the main
    // loop's shared-memory loads are independent
    __syncthreads();
    for (int i = tid; i < T; i += NT) {
        const int p = sp[i];
        if (i == 0 ? p != -1 : (p < 0 || p >= i)) atomicMax(&s_bad, i == 0 ? 2 : 1);
        int v = i, srow = W - 1;
        s_win[i * 4 + W - 1] = ((W - 1) + i) * KC * 16;
#pragma unroll
        for (int k = 1; k < W; ++k) {
            if (v >= 0) {
                const int pv = sp[v];
                v = (pv >= 0 && pv < v) ? pv : -1;
            }
            s_win[i * 4 + W - 1 - k] = (v >= 0 ? (W - 1) + v : --srow) * KC * 16;
        }
    }
    uint64_t wt2[W][V / 2], bs2[V / 2];
#pragma unroll
    for (int q = 0; q < V / 2; ++q) {
#pragma unroll
        for (int w = 0; w < W; ++w) wt2[w][q] = f2pack(s_w[(w * V + 2 * q) * KC + ch], s_w[(w * V + 2 * q + 1) * KC + ch]);
        bs2[q] = f2pack(s_b[2 * q * KC + ch], s_b[(2 * q + 1) * KC + ch]);
    }
    if (early_tree) {   // the dependency wait: only the tree's rows (and, without EARLY_STATE, the state) remain
        pdl_wait();
        if (!early_state) stage_state();
        stage_rows();
    }
    __syncthreads();
    const int bad = s_bad;
    if (bad && tid == 0 && blockIdx.x == 0) report(dev_status, bad == 2 ? 1 : 2);
    const unsigned char* rl = rows + ch * 16;   // this thread's chunk of every row
#pragma unroll
    for (int k = 0; k < kGroups; ++k) {
        // group k (and the state rows, in group 0) landed for every thread of the CTA
        cp_async_wait_n(kGroups - 1 - k);
        __syncthreads();
        const int n1 = min((k + 1) * gs, T);
        IO* op = out + ((size_t)b * T + k * gs + ns) * C + c0 + ch * V;
#pragma unroll 2
        for (int i = k * gs + ns; i < n1; i += kSlots, op += (size_t)kSlots * C) {
            const int4 ro = *reinterpret_cast<const int4*>(s_win + i * 4);
            const int rw[4] = {ro.x, ro.y, ro.z, ro.w};
            uint64_t z2[V / 2];
#pragma unroll
            for (int q = 0; q < V / 2; ++q) z2[q] = bs2[q];
#pragma unroll
            for (int w = 0; w < W; ++w) {
                uint64_t f2[V / 2];
                unpack2<IO>(*reinterpret_cast<const uint4*>(rl + rw[w]), f2);
#pragma unroll
                for (int q = 0; q < V / 2; ++q) z2[q] = ffma2(wt2[w][q], f2[q], z2[q]);
            }
            float z[V];
#pragma unroll
            for (int q = 0; q < V / 2; ++q) f2unpack(z2[q], z[2 * q], z[2 * q + 1]);
            if (ACT) {
#pragma unroll
                for (int q = 0; q < V; ++q) z[q] = silu_h<IO>(z[q]);
            }
            if (bad) {
#pragma unroll
                for (int q = 0; q < V; ++q) z[q] = 0.f;
            }
            if (cv) *reinterpret_cast<uint4*>(op) = Pack<IO>::pack(z);
        }
    }
}

// Conv-state commit: new[b][j] = (state[b] ++ u[b][path])[L - (W-1) + j], L = W-1 + r.  One warp per
// (tree, channel block); all sources are read before any store (in place is allowed).
template <typename IO, int W>
__global__ void __launch_bounds__(32) conv_commit_kernel(const IO* __restrict__ u, const IO* state,
                                                         const int32_t* __restrict__ parent,
                                                         const int32_t* __restrict__ path,
                                                         const int32_t* __restrict__ path_len, IO* state_new, int T,
                                                         int C, int32_t* dev_status) {
    constexpr int V = Pack<IO>::V;
    const int b = blockIdx.y, c0 = blockIdx.x * kChunks * V, lane = threadIdx.x;
    const bool cv = c0 + lane * V < C;
    pdl_wait();
    const int r = path_len[b];
    const int32_t* pa = path + (size_t)b * T;
    // root-anchored, increasing, parent-linked (as stree_commit)
    int ok = (r >= 1 && r <= T);
    if (ok) {
        for (int m = lane; m < r; m += 32) {
            const int v = pa[m];
            bool good = v >= 0 && v < T;
            if (m == 0) good = good && v == 0;
            else {
                const int pu = pa[m - 1];
                good = good && v > pu;
                if (parent && good) good = parent[(size_t)b * T + v] == pu;
            }
            if (!good) ok = 0;
        }
    }
    ok = __all_sync(0xffffffffu, ok);
    if (!ok && lane == 0 && blockIdx.x == 0) report(dev_status, STREE_DEV_BAD_PATH);
    const int L = (W - 1) + (ok ? r : 0);
    uint4 v[W > 1 ? W - 1 : 1];
#pragma unroll
    for (int j = 0; j < W - 1; ++j) {
        const int q = L - (W - 1) + j;
        v[j] = make_uint4(0, 0, 0, 0);
        if (cv) {
            if (q < W - 1) {
                if (state) v[j] = *reinterpret_cast<const uint4*>(state + ((size_t)b * (W - 1) + q) * C + c0 + lane * V);
            } else {
                v[j] = *reinterpret_cast<const uint4*>(u + ((size_t)b * T + pa[q - (W - 1)]) * C + c0 + lane * V);
            }
        }
    }
#pragma unroll
    for (int j = 0; j < W - 1; ++j)
        if (cv) *reinterpret_cast<uint4*>(state_new + ((size_t)b * (W - 1) + j) * C + c0 + lane * V) = v[j];
}

template <typename IO, int W>
cudaError_t launch_conv(const stree_conv_dims* d, const void* u, const float* weight, const float* bias,
                        const void* state, const int32_t* parent, int act, void* out, int32_t* dev_status,
                        cudaStream_t s) {
    constexpr int V = Pack<IO>::V, KC = kConvKC;
    const int C = d->channels, T = d->n_nodes;
    dim3 grid((C / V + KC - 1) / KC, d->batch);
    const size_t smem = tree_conv_smem(T, W, KC);
    // row groups per CTA (8 groups measured slower at the 2.7B shape: 7.1 vs 6.8 µs per call)
    auto k = act ? tree_conv_kernel<IO, W, KC, true, kConvGroups> : tree_conv_kernel<IO, W, KC, false, kConvGroups>;
    // every CTA of the 2.7B shape resident at once (672 CTAs, <= 5 per SM): registers capped by the launch
    // bounds, shared-memory carveout at its maximum
    cudaError_t e = stree::host::smem_attr((const void*)k, (int)smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    const uint32_t fl = stree_launch_flags_get();
    const int early_tree = (fl & STREE_LAUNCH_EARLY_TREE) ? 1 : 0, early_state = (fl & STREE_LAUNCH_EARLY_STATE) ? 1 : 0;
    return launch_k(k, grid, dim3(8 * KC), smem, s, (const IO*)u, weight, bias, (const IO*)state, parent,
                    (IO*)out, T, C, dev_status, early_tree, early_state);
}

template <typename IO, int W>
cudaError_t launch_commit(const stree_conv_dims* d, const void* u, const void* state, const int32_t* parent,
                          const int32_t* path, const int32_t* path_len, void* state_new, int32_t* dev_status,
                          cudaStream_t s) {
    constexpr int V = Pack<IO>::V;
    const int C = d->channels, T = d->n_nodes;
    dim3 grid((C / V + kChunks - 1) / kChunks, d->batch);
    return launch_k(conv_commit_kernel<IO, W>, grid, dim3(32), 0, s, (const IO*)u, (const IO*)state, parent, path,
                    path_len, (IO*)state_new, T, C, dev_status);
}

template <typename IO>
cudaError_t dispatch_conv(const stree_conv_dims* d, const void* u, const float* weight, const float* bias,
                          const void* state, const int32_t* parent, int act, void* out, int32_t* dev_status,
                          cudaStream_t s) {
    switch (d->width) {
        case 1: return launch_conv<IO, 1>(d, u, weight, bias, state, parent, act, out, dev_status, s);
        case 2: return launch_conv<IO, 2>(d, u, weight, bias, state, parent, act, out, dev_status, s);
        case 3: return launch_conv<IO, 3>(d, u, weight, bias, state, parent, act, out, dev_status, s);
        default: return launch_conv<IO, 4>(d, u, weight, bias, state, parent, act, out, dev_status, s);
    }
}

template <typename IO>
cudaError_t dispatch_commit(const stree_conv_dims* d, const void* u, const void* state, const int32_t* parent,
                            const int32_t* path, const int32_t* path_len, void* state_new, int32_t* dev_status,
                            cudaStream_t s) {
    switch (d->width) {
        case 2: return launch_commit<IO, 2>(d, u, state, parent, path, path_len, state_new, dev_status, s);
        case 3: return launch_commit<IO, 3>(d, u, state, parent, path, path_len, state_new, dev_status, s);
        default: return launch_commit<IO, 4>(d, u, state, parent, path, path_len, state_new, dev_status, s);
    }
}

}  // namespace conv
}  // namespace stree

extern "C" int stree_launch_tree_conv(const stree_conv_dims* d, const void* u, const float* weight, const float* bias,
                                      const void* state, const int32_t* parent, int act, void* out,
                                      int32_t* dev_status, cudaStream_t s) {
    cudaError_t e = d->io_dtype == STREE_BF16
                        ? stree::conv::dispatch_conv<__nv_bfloat16>(d, u, weight, bias, state, parent, act, out,
                                                                    dev_status, s)
                        : stree::conv::dispatch_conv<float>(d, u, weight, bias, state, parent, act, out, dev_status, s);
    if (e != cudaSuccess) return (int)e;
    return (int)cudaGetLastError();
}

extern "C" int stree_launch_conv_commit(const stree_conv_dims* d, const void* u, const void* state,
                                        const int32_t* parent, const int32_t* path, const int32_t* path_len,
                                        void* state_new, int32_t* dev_status, cudaStream_t s) {
    if (d->width <= 1) return 0;   // no state
    cudaError_t e = d->io_dtype == STREE_BF16
                        ? stree::conv::dispatch_commit<__nv_bfloat16>(d, u, state, parent, path, path_len, state_new,
                                                                      dev_status, s)
                        : stree::conv::dispatch_commit<float>(d, u, state, parent, path, path_len, state_new,
                                                              dev_status, s);
    if (e != cudaSuccess) return (int)e;
    return (int)cudaGetLastError();
}
