// K4 stree_commit — activation replay of the accepted path (PAPER.md:113,
// Alg. 1 l.123):  h_new = e^{Λ_k} h0 + Σ_{s∈path} e^{Λ_k-Λ_s} dt_s x_s B_sᵀ.
//
// HBM-bound streaming kernel (intensity ≈ r/4 FLOP/B): one CTA per (tree, head)
// state block (P x N fp32, 32 KB at P=64, N=128), 256 threads.  Every thread
// issues its 16-byte state loads at kernel entry — before the dependent
// path_len -> path -> dt chain of the prologue — so the state stream overlaps
// the prologue latency; the rank-r update uses the path rows of x and B staged in
// shared memory; results are written with streaming stores.
#include "stree_common.cuh"

namespace stree {

constexpr int kCommitThreads = 256;
constexpr int kCommitVec = 8;        // float4 per thread held in registers (P*N <= 8192 fp32)
constexpr int kCommitChunk = 16;     // path nodes staged per smem round

template <typename IO>
__global__ void __launch_bounds__(kCommitThreads) commit_kernel(int T, int H, int P, int N, int G,
                                                                const IO* __restrict__ x, const float* __restrict__ dt,
                                                                const float* __restrict__ A,
                                                                const IO* __restrict__ Bm, const float* h0,
                                                                const int32_t* __restrict__ parent,
                                                                const int32_t* __restrict__ path,
                                                                const int32_t* __restrict__ path_len, float* h_new,
                                                                int32_t* dev_status) {
    extern __shared__ float smem[];
    const int h = blockIdx.x, b = blockIdx.y;
    const int g = h / (H / G);
    __shared__ int s_path[kMaxNodes];
    __shared__ float s_coef[kMaxNodes];
    __shared__ float s_decay;
    __shared__ int s_ok;
    const int tid = threadIdx.x;
    const size_t off = ((size_t)b * H + h) * (size_t)P * N;
    const float* src = h0 ? h0 + off : nullptr;
    float* dst = h_new + off;
    const int total = P * N;
    const bool vec = (N % 4 == 0) && (total <= kCommitThreads * kCommitVec * 4);
    const int nvec = total / 4;

    // ---- 1. state loads first (independent of the path) ----
    float4 acc[kCommitVec];
    if (vec) {
#pragma unroll
        for (int q = 0; q < kCommitVec; ++q) {
            const int e = tid + q * kCommitThreads;
            acc[q] = (e < nvec && src) ? __ldcs(reinterpret_cast<const float4*>(src) + e) : make_float4(0, 0, 0, 0);
        }
    }
    // ---- 2. path validation + coefficients (warp 0) ----
    if (tid < 32) {
        const int r = path_len[b];
        int ok = (r >= 1 && r <= T);
        if (ok) {
            for (int m = tid; m < r; m += 32) {
                const int v = path[(size_t)b * T + m];
                s_path[m] = v;
                bool good = (v >= 0 && v < T);
                if (m == 0) good = good && v == 0;
                else {
                    const int u = path[(size_t)b * T + m - 1];
                    good = good && v > u;
                    if (parent && good) good = parent[(size_t)b * T + v] == u;
                }
                if (!good) ok = 0;
            }
        }
        ok = __all_sync(0xffffffffu, ok);
        if (ok) {
            // path-cumsum of log-decays lam_m = Σ_{q<=m} dt_q A_h (PAPER.md:86-90 on the path);
            // c_m = e^{lam_{r-1} - lam_m} dt_m,  decay = e^{lam_{r-1}}
            const float Ah = A[h];
            float carry = 0.f;
            for (int base = 0; base < r; base += 32) {
                const int m = base + tid;
                float a = (m < r) ? dt[((size_t)b * T + s_path[m]) * H + h] * Ah : 0.f;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const float t = __shfl_up_sync(0xffffffffu, a, o);
                    if (tid >= o) a += t;
                }
                a += carry;
                if (m < r) s_coef[m] = a;
                carry = __shfl_sync(0xffffffffu, a, 31);
            }
            __syncwarp();
            for (int m = tid; m < r; m += 32)
                s_coef[m] = expf(carry - s_coef[m]) * dt[((size_t)b * T + s_path[m]) * H + h];
            if (tid == 0) s_decay = expf(carry);
        }
        if (tid == 0) s_ok = ok ? r : 0;
    }
    __syncthreads();
    const int r = s_ok;
    if (r == 0) {
        if (tid == 0 && h == 0) report(dev_status, STREE_DEV_BAD_PATH);
        if (src != dst) {
            if (vec) {
#pragma unroll
                for (int q = 0; q < kCommitVec; ++q) {
                    const int e = tid + q * kCommitThreads;
                    if (e < nvec) __stcs(reinterpret_cast<float4*>(dst) + e, acc[q]);
                }
            } else {
                for (int k = tid; k < total; k += kCommitThreads) dst[k] = src ? src[k] : 0.f;
            }
        }
        return;
    }
    const float decay = s_decay;
    float* s_u = smem;                           // [chunk][P]  c_m * x_m[p]
    float* s_B = smem + kCommitChunk * P;        // [chunk][N]
    if (vec) {
#pragma unroll
        for (int q = 0; q < kCommitVec; ++q)
            acc[q] = make_float4(decay * acc[q].x, decay * acc[q].y, decay * acc[q].z, decay * acc[q].w);
        for (int m0 = 0; m0 < r; m0 += kCommitChunk) {
            const int mc = min(kCommitChunk, r - m0);
            if (m0) __syncthreads();
            for (int k = tid; k < mc * P; k += kCommitThreads) {
                const int m = k / P, p = k % P;
                s_u[m * P + p] = s_coef[m0 + m] * to_f32(x[(((size_t)b * T + s_path[m0 + m]) * H + h) * P + p]);
            }
            for (int k = tid; k < mc * N; k += kCommitThreads) {
                const int m = k / N, n = k % N;
                s_B[m * N + n] = to_f32(Bm[(((size_t)b * T + s_path[m0 + m]) * G + g) * N + n]);
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < kCommitVec; ++q) {
                const int e = tid + q * kCommitThreads;
                if (e < nvec) {
                    const int p = (e * 4) / N, n = (e * 4) % N;
                    float4 a = acc[q];
                    for (int m = 0; m < mc; ++m) {
                        const float u = s_u[m * P + p];
                        const float4 bb = *reinterpret_cast<const float4*>(&s_B[m * N + n]);
                        a.x = fmaf(u, bb.x, a.x); a.y = fmaf(u, bb.y, a.y);
                        a.z = fmaf(u, bb.z, a.z); a.w = fmaf(u, bb.w, a.w);
                    }
                    acc[q] = a;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < kCommitVec; ++q) {
            const int e = tid + q * kCommitThreads;
            if (e < nvec) __stcs(reinterpret_cast<float4*>(dst) + e, acc[q]);
        }
    } else {
        // generic fallback (N % 4 != 0 or a state block larger than 32 K fp32)
        for (int e = tid; e < total; e += kCommitThreads) {
            const int p = e / N, n = e % N;
            float a = decay * (src ? src[e] : 0.f);
            for (int m = 0; m < r; ++m) {
                const int s = s_path[m];
                a = fmaf(s_coef[m] * to_f32(x[(((size_t)b * T + s) * H + h) * P + p]),
                         to_f32(Bm[(((size_t)b * T + s) * G + g) * N + n]), a);
            }
            dst[e] = a;
        }
    }
}

}  // namespace stree

extern "C" int stree_launch_commit(const stree_dims* d, const void* x, const float* dt, const float* A,
                                   const void* Bm, const float* h0, const int32_t* parent,
                                   const int32_t* path, const int32_t* path_len, float* h_new,
                                   int32_t* dev_status, cudaStream_t s) {
    const int P = d->head_dim, N = d->d_state;
    dim3 grid(d->n_heads, d->batch);
    size_t smem = (size_t)stree::kCommitChunk * (P + N) * sizeof(float);
    if (smem > 200 * 1024) return (int)cudaErrorInvalidValue;
    cudaError_t e;
    if (d->io_dtype == STREE_BF16) {
        auto k = stree::commit_kernel<__nv_bfloat16>;
        if (smem > 48 * 1024 && (e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                          (int)smem)) != cudaSuccess)
            return (int)e;
        k<<<grid, stree::kCommitThreads, smem, s>>>(d->n_nodes, d->n_heads, P, N, d->n_groups,
                                                     (const __nv_bfloat16*)x, dt, A, (const __nv_bfloat16*)Bm, h0,
                                                     parent, path, path_len, h_new, dev_status);
    } else {
        auto k = stree::commit_kernel<float>;
        if (smem > 48 * 1024 && (e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                          (int)smem)) != cudaSuccess)
            return (int)e;
        k<<<grid, stree::kCommitThreads, smem, s>>>(d->n_nodes, d->n_heads, P, N, d->n_groups, (const float*)x, dt,
                                                     A, (const float*)Bm, h0, parent, path, path_len, h_new,
                                                     dev_status);
    }
    return (int)cudaGetLastError();
}
