// K5 stree_tree_conv / K6 stree_conv_commit: tree-causal depthwise conv1d over the xBC channels
// and its conv-state commit (reading R-conv).
//
//   seq_i        = conv_state[b] (W-1 rows, oldest first) ++ u[b][root .. i]
//   out[b][i][c] = act( bias[c] + sum_{w<W} weight[c][w] * seq_i[len - W + w][c] )
//
// HBM-bound (intensity ~W FLOP per 4 bytes).  One CTA per (tree, block of 32 16-byte channel
// chunks): the tree's rows of that channel block (and the conv state) are read once, coalesced,
// into shared memory; every node then reads its W-1 ancestors from there (the ancestor chain is
// walked in shared memory, stepping into the state rows above the root), and the output row is
// written once, coalesced.
#include "stree_common.cuh"
#include "stree_host.cuh"

namespace stree {
namespace conv {

constexpr int kThreads = 256;   // 8 warps: lane = channel chunk, warp = node (strided by 8)
constexpr int kChunks = 32;     // 16-byte channel chunks per CTA

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

__host__ __device__ constexpr size_t tree_conv_smem(int T, int W) {
    return (size_t)kMaxNodes * 4 + (size_t)((W - 1) + T) * kChunks * 16;
}

// SiLU: bf16 outputs take x·σ(x) with σ(x) = ½ tanh(x/2) + ½ (one MUFU op; tanh.approx's 2^-11 error is
// far below the bf16 rounding of the output); fp32 outputs keep the exp + division form (the 1e-4 path)
template <typename IO>
__device__ __forceinline__ float silu(float z);
template <>
__device__ __forceinline__ float silu<__nv_bfloat16>(float z) {
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * z));
    return z * fmaf(0.5f, t, 0.5f);
}
template <>
__device__ __forceinline__ float silu<float>(float z) { return __fdividef(z, 1.f + __expf(-z)); }

template <typename IO, int W>
__global__ void __launch_bounds__(kThreads, 3) tree_conv_kernel(const IO* __restrict__ u, const float* __restrict__ weight,
                                                             const float* __restrict__ bias, const IO* __restrict__ state,
                                                             const int32_t* __restrict__ parent, int act,
                                                             IO* __restrict__ out, int T, int C, int32_t* dev_status) {
    constexpr int V = Pack<IO>::V;
    extern __shared__ __align__(16) unsigned char sm[];
    int* sp = reinterpret_cast<int*>(sm);                                   // parent[T]
    uint4* rows = reinterpret_cast<uint4*>(sm + kMaxNodes * 4);             // [(W-1) + T][kChunks]
    __shared__ int s_bad;
    const int b = blockIdx.y, c0 = blockIdx.x * kChunks * V;
    const int tid = threadIdx.x, lane = tid & 31, wy = tid >> 5;
    const bool cv = c0 + lane * V < C;                                     // this lane's chunk exists
    if (tid == 0) s_bad = 0;
    // the block's weights and bias: coalesced loads issued together with the parent and staging loads below
    // (one memory latency for all of them), then through shared memory, [w][v][lane] so the per-thread reads
    // are conflict-free
    __shared__ float s_w[4 * 8 * kChunks];
    __shared__ float s_b[8 * kChunks];
    pdl_wait();
    const int nc = min(kChunks * V, C - c0);   // channels of this block (nc * W <= 4 * kThreads)
    float wv[4], bv;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int k = tid + q * kThreads;
        wv[q] = k < nc * W ? __ldg(weight + (size_t)c0 * W + k) : 0.f;
    }
    bv = (tid < nc && bias) ? __ldg(bias + c0 + tid) : 0.f;
    for (int i = tid; i < T; i += kThreads) sp[i] = parent[(size_t)b * T + i];
    // stage the state rows and the tree's rows of this channel block (one coalesced pass)
    // batches of kBatch independent 16-byte loads per thread in flight (one latency per batch, not per
    // row): addresses are clamped to valid rows so the loads are unconditional, zeros selected after
    constexpr int kBatch = 9, kWy = kThreads / 32;   // 9 x 8 warps = 72 >= 3 + 64 rows: one batch at T = 64
    const int nrows = (W - 1) + T;
    const size_t cofs = (size_t)c0 + (cv ? lane * V : 0);
    for (int r0 = wy; r0 < nrows; r0 += kWy * kBatch) {
        uint4 v[kBatch];
#pragma unroll
        for (int k = 0; k < kBatch; ++k) {
            const int r = min(r0 + kWy * k, nrows - 1);
            const IO* src = (r < W - 1) ? (state ? state + ((size_t)b * (W - 1) + r) * C : u + (size_t)b * T * C)
                                        : u + ((size_t)b * T + (r - (W - 1))) * C;
            v[k] = __ldg(reinterpret_cast<const uint4*>(src + cofs));
        }
#pragma unroll
        for (int k = 0; k < kBatch; ++k) {
            const int r = r0 + kWy * k;
            const bool zero = !cv || (r < W - 1 && !state);
            if (r < nrows) rows[r * kChunks + lane] = zero ? make_uint4(0, 0, 0, 0) : v[k];
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int k = tid + q * kThreads;
        if (k < nc * W) {
            const int cl = k / W, w = k % W;
            s_w[(w * V + cl % V) * kChunks + cl / V] = wv[q];
        }
    }
    if (tid < nc) s_b[(tid % V) * kChunks + tid / V] = bv;
    __syncthreads();
    float wt[W][V], bs[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
#pragma unroll
        for (int w = 0; w < W; ++w) wt[w][v] = cv ? s_w[(w * V + v) * kChunks + lane] : 0.f;
        bs[v] = cv ? s_b[v * kChunks + lane] : 0.f;
    }
    // PAPER.md:90 precondition: parent[0] = -1, 0 <= parent[i] < i (root error takes precedence); the same
    // pass tabulates every node's window rows (oldest first: ancestors at distance W-1 .. 1, then the node;
    // above the root the chain continues into the state rows W-2, W-3, ...) so the main loop's shared-memory
    // loads are independent
    __shared__ int s_win[kMaxNodes * 4];
    for (int i = tid; i < T; i += kThreads) {
        const int p = sp[i];
        if (i == 0 ? p != -1 : (p < 0 || p >= i)) atomicMax(&s_bad, i == 0 ? 2 : 1);
        int v = i, srow = W - 1;
        s_win[i * W + W - 1] = (W - 1) + i;
#pragma unroll
        for (int k = 1; k < W; ++k) {
            if (v >= 0) {
                const int pv = sp[v];
                v = (pv >= 0 && pv < v) ? pv : -1;
            }
            s_win[i * W + W - 1 - k] = v >= 0 ? (W - 1) + v : --srow;
        }
    }
    __syncthreads();
    const int bad = s_bad;
    if (bad && tid == 0 && blockIdx.x == 0) report(dev_status, bad == 2 ? 1 : 2);
#pragma unroll 2
    for (int i = wy; i < T; i += kThreads / 32) {
        int rw[W];
#pragma unroll
        for (int k = 0; k < W; ++k) rw[k] = s_win[i * W + k];
        float z[V];
#pragma unroll
        for (int q = 0; q < V; ++q) z[q] = bs[q];
#pragma unroll
        for (int w = 0; w < W; ++w) {
            float f[V];
            Pack<IO>::unpack(rows[rw[w] * kChunks + lane], f);
#pragma unroll
            for (int q = 0; q < V; ++q) z[q] = fmaf(wt[w][q], f[q], z[q]);
        }
        if (act) {
#pragma unroll
            for (int q = 0; q < V; ++q) z[q] = silu<IO>(z[q]);
        }
        if (bad) {
#pragma unroll
            for (int q = 0; q < V; ++q) z[q] = 0.f;
        }
        if (cv) *reinterpret_cast<uint4*>(out + ((size_t)b * T + i) * C + c0 + lane * V) = Pack<IO>::pack(z);
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
    constexpr int V = Pack<IO>::V;
    const int C = d->channels, T = d->n_nodes;
    dim3 grid((C / V + kChunks - 1) / kChunks, d->batch);
    const size_t smem = tree_conv_smem(T, W);
    auto k = tree_conv_kernel<IO, W>;
    // one wave at the 2.7B shape (336 CTAs over 148 SMs needs 3 resident per SM): registers capped by the
    // launch bounds, shared-memory carveout at its maximum
    cudaError_t e = stree::host::smem_attr((const void*)k, (int)smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    return launch_k(k, grid, dim3(kThreads), smem, s, (const IO*)u, weight, bias, (const IO*)state, parent, act,
                    (IO*)out, T, C, dev_status);
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
