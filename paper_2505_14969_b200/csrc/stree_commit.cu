// K4 stree_commit — activation replay of the accepted path (PAPER.md:113,
// Alg. 1 l.123):  h_new = e^{Λ_k} h0 + Σ_{s∈path} e^{Λ_k-Λ_s} dt_s x_s B_sᵀ.
//
// HBM-bound streaming kernel: every (b, h) state block (P x N fp32) is read
// once and written once with 16-byte vector accesses; the rank-r update uses
// the r path coefficients and the path's x / B rows staged in shared memory
// (r is small: 3-10 for the drafted trees of the paper).  Grid: (H, B, P/16),
// 128 threads; each CTA streams a 16 x N slab (8 KB at N = 128).
#include "stree_common.cuh"

namespace stree {

constexpr int kCommitRows = 16;      // state rows (p) per CTA
constexpr int kCommitChunk = 32;     // path nodes staged per smem round

template <typename IO>
__global__ void __launch_bounds__(128) commit_kernel(int T, int H, int P, int N, int G,
                                                     const IO* __restrict__ x, const float* __restrict__ dt,
                                                     const float* __restrict__ A, const IO* __restrict__ Bm,
                                                     const float* h0, const int32_t* __restrict__ parent,
                                                     const int32_t* __restrict__ path,
                                                     const int32_t* __restrict__ path_len, float* h_new,
                                                     int32_t* dev_status) {
    extern __shared__ float smem[];
    const int h = blockIdx.x, b = blockIdx.y, p0 = blockIdx.z * kCommitRows;
    const int g = h / (H / G);
    const int rows = min(kCommitRows, P - p0);
    __shared__ int s_path[kMaxNodes];
    __shared__ float s_coef[kMaxNodes];
    __shared__ float s_decay;
    __shared__ int s_ok;
    const int tid = threadIdx.x;
    const int r = path_len[b];
    // ---- validate path (root-anchored, increasing, parent-linked) ----
    if (tid < 32) {
        int ok = (r >= 1 && r <= T);
        if (ok) {
            for (int m = tid; m < r; m += 32) {
                int v = path[(size_t)b * T + m];
                s_path[m] = v;
                bool good = (v >= 0 && v < T);
                if (m == 0) good = good && v == 0;
                else {
                    int u = path[(size_t)b * T + m - 1];
                    good = good && v > u;
                    if (parent && good) good = parent[(size_t)b * T + v] == u;
                }
                if (!good) ok = 0;
            }
        }
        ok = __all_sync(0xffffffffu, ok);
        // path-cumsum of log-decays along the path: lam_m = Σ_{q<=m} dt_q A_h
        // (PAPER.md:86-90 restricted to the accepted path), coefficients
        // c_m = e^{lam_{r-1} - lam_m} dt_m and decay = e^{lam_{r-1}}.
        if (ok) {
            const float Ah = A[h];
            float carry = 0.f;
            float lam_last = 0.f;
            // two passes: first total, then coefficients (r <= 256)
            for (int base = 0; base < r; base += 32) {
                int m = base + tid;
                float a = (m < r) ? dt[((size_t)b * T + s_path[m]) * H + h] * Ah : 0.f;
                for (int o = 1; o < 32; o <<= 1) {
                    float t = __shfl_up_sync(0xffffffffu, a, o);
                    if (tid >= o) a += t;
                }
                a += carry;
                if (m < r) s_coef[m] = a;  // inclusive prefix lam_m
                carry = __shfl_sync(0xffffffffu, a, 31);
            }
            lam_last = carry;
            __syncwarp();
            for (int m = tid; m < r; m += 32) {
                float dtm = dt[((size_t)b * T + s_path[m]) * H + h];
                s_coef[m] = expf(lam_last - s_coef[m]) * dtm;
            }
            if (tid == 0) s_decay = expf(lam_last);
        }
        if (tid == 0) s_ok = ok;
    }
    __syncthreads();
    const size_t base_off = ((size_t)b * H + h) * (size_t)P * N + (size_t)p0 * N;
    const float* src = h0 ? h0 + base_off : nullptr;
    float* dst = h_new + base_off;
    const int total = rows * N;
    if (!s_ok) {
        if (tid == 0 && h == 0 && blockIdx.z == 0) report(dev_status, STREE_DEV_BAD_PATH);
        if (src != dst)
            for (int k = tid; k < total; k += blockDim.x) dst[k] = src ? src[k] : 0.f;
        return;
    }
    const float decay = s_decay;
    float* s_u = smem;                                  // [chunk][rows]   c_m * x_m[p]
    float* s_B = smem + kCommitChunk * kCommitRows;     // [chunk][N]
    const bool vec = (N % 4 == 0) && (N <= 256);
    if (vec) {
        const int nvec = total / 4;                     // float4 elements of the slab
        constexpr int kPer = 8;                         // up to 8 float4 per thread (16 x 256 / 4 / 128)
        float4 acc[kPer];
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            int e = tid + q * 128;
            if (e < nvec) {
                float4 v = src ? reinterpret_cast<const float4*>(src)[e] : make_float4(0, 0, 0, 0);
                acc[q] = make_float4(decay * v.x, decay * v.y, decay * v.z, decay * v.w);
            }
        }
        for (int m0 = 0; m0 < r; m0 += kCommitChunk) {
            const int mc = min(kCommitChunk, r - m0);
            __syncthreads();
            for (int k = tid; k < mc * rows; k += 128) {
                int m = k / rows, pp = k % rows;
                int s = s_path[m0 + m];
                s_u[m * kCommitRows + pp] =
                    s_coef[m0 + m] * to_f32(x[(((size_t)b * T + s) * H + h) * P + p0 + pp]);
            }
            for (int k = tid; k < mc * N; k += 128) {
                int m = k / N, n = k % N;
                s_B[m * N + n] = to_f32(Bm[(((size_t)b * T + s_path[m0 + m]) * G + g) * N + n]);
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < kPer; ++q) {
                int e = tid + q * 128;
                if (e < nvec) {
                    int pp = (e * 4) / N, n = (e * 4) % N;
                    float4 a = acc[q];
                    for (int m = 0; m < mc; ++m) {
                        float u = s_u[m * kCommitRows + pp];
                        float4 bb = *reinterpret_cast<const float4*>(&s_B[m * N + n]);
                        a.x = fmaf(u, bb.x, a.x); a.y = fmaf(u, bb.y, a.y);
                        a.z = fmaf(u, bb.z, a.z); a.w = fmaf(u, bb.w, a.w);
                    }
                    acc[q] = a;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            int e = tid + q * 128;
            if (e < nvec) reinterpret_cast<float4*>(dst)[e] = acc[q];
        }
    } else {
        // scalar fallback (N % 4 != 0): one element at a time
        for (int e = tid; e < total; e += 128) {
            int pp = e / N, n = e % N;
            float a = decay * (src ? src[e] : 0.f);
            for (int m = 0; m < r; ++m) {
                int s = s_path[m];
                a = fmaf(s_coef[m] * to_f32(x[(((size_t)b * T + s) * H + h) * P + p0 + pp]),
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
    dim3 grid(d->n_heads, d->batch, (d->head_dim + stree::kCommitRows - 1) / stree::kCommitRows);
    const bool vec = (d->d_state % 4 == 0) && (d->d_state <= 256);
    size_t smem = vec ? (size_t)stree::kCommitChunk * (stree::kCommitRows + d->d_state) * sizeof(float) : 0;
    if (d->io_dtype == STREE_BF16)
        stree::commit_kernel<__nv_bfloat16><<<grid, 128, smem, s>>>(
            d->n_nodes, d->n_heads, d->head_dim, d->d_state, d->n_groups, (const __nv_bfloat16*)x, dt, A,
            (const __nv_bfloat16*)Bm, h0, parent, path, path_len, h_new, dev_status);
    else
        stree::commit_kernel<float><<<grid, 128, smem, s>>>(
            d->n_nodes, d->n_heads, d->head_dim, d->d_state, d->n_groups, (const float*)x, dt, A,
            (const float*)Bm, h0, parent, path, path_len, h_new, dev_status);
    return (int)cudaGetLastError();
}
