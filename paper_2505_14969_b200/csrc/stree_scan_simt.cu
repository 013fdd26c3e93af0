// K2' stree_tree_scan, generic SIMT (FP32 FMA) kernel.
//
// Serves every shape (any T <= 256, P, N, G) and both io dtypes; it is the
// fp32 parity path (rel-err 1e-4) and the fallback for shapes the tcgen05
// kernel does not take.  One CTA per (head, tree), 256 threads; per 64-row x
// 64-column output tile it computes, entirely on chip:
//   Y0  = C · h0_hᵀ                      (carry-in, PAPER.md:100 M_x), N-chunked
//   y  = e^{Λ_i} Y0  +  Σ_{j∈path(i)} e^{Λ_i-Λ_j} dt_j (C_i·B_j) x_j  +  D_h x_i
// with Λ = L·(dt A_h) the tree segsum and the decay mask
// applied before exp (off-path entries are never exponentiated).
#include "stree_common.cuh"
#include "stree_host.cuh"

namespace stree {

constexpr int kTile = 64;   // rows (nodes) / cols (p) / n per smem chunk
constexpr int kPitch = 68;  // smem pitch of 64-wide tiles (16-byte aligned rows)

struct SimtSmem {
    // byte offsets into dynamic smem
    size_t sp, jmp, jmp2, rows, rows2, lam, dtv, cst, hst, ms, xs, total;
    int W, Tpad, mpitch;
    __host__ __device__ SimtSmem(int T) {
        W = (T + 31) / 32;
        Tpad = (T + 3) & ~3;
        mpitch = Tpad + 1;
        size_t o = 0;
        auto take = [&](size_t bytes) { size_t r = o; o += (bytes + 15) & ~size_t(15); return r; };
        sp = take(sizeof(int) * T); jmp = take(sizeof(int) * T); jmp2 = take(sizeof(int) * T);
        rows = take(sizeof(uint32_t) * T * W); rows2 = take(sizeof(uint32_t) * T * W);
        lam = take(sizeof(float) * T); dtv = take(sizeof(float) * T);
        cst = take(sizeof(float) * kTile * kPitch); hst = take(sizeof(float) * kTile * kPitch);
        ms = take(sizeof(float) * kTile * mpitch); xs = take(sizeof(float) * Tpad * kPitch);
        total = o;
    }
};

template <typename IO>
__global__ void __launch_bounds__(256) scan_simt_kernel(int T, int H, int P, int N, int G,
                                                        const IO* __restrict__ x, const float* __restrict__ dt,
                                                        const float* __restrict__ A, const IO* __restrict__ Bm,
                                                        const IO* __restrict__ Cm, const float* __restrict__ D,
                                                        const float* __restrict__ h0,
                                                        const int32_t* __restrict__ parent, IO* __restrict__ y,
                                                        int32_t* dev_status, DtX dtx, int d_pc) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const SimtSmem L(T);
    int* sp = (int*)(smem_raw + L.sp);
    uint32_t* rows = (uint32_t*)(smem_raw + L.rows);
    float* lam = (float*)(smem_raw + L.lam);
    float* dtv = (float*)(smem_raw + L.dtv);
    float* CsT = (float*)(smem_raw + L.cst);   // [n][row]
    float* HsT = (float*)(smem_raw + L.hst);   // [n][p]
    float* Ms = (float*)(smem_raw + L.ms);     // [row][j]
    float* Xs = (float*)(smem_raw + L.xs);     // [j][p]
    const int W = L.W, mp = L.mpitch;
    const int h = blockIdx.x, b = blockIdx.y, g = h / (H / G);
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    pdl_wait();

    for (int i = tid; i < T; i += 256) sp[i] = parent[(size_t)b * T + i];
    __syncthreads();
    const int code = build_tree_rows(sp, T, W, rows, (uint32_t*)(smem_raw + L.rows2), (int*)(smem_raw + L.jmp),
                                     (int*)(smem_raw + L.jmp2));
    if (code) {
        if (tid == 0 && h == 0 && blockIdx.z == 0) report(dev_status, code);
        for (int k = tid; k < T * P; k += 256) {
            int i = k / P, p = k % P;
            if ((i / kTile) % (int)gridDim.z == (int)blockIdx.z) y[(((size_t)b * T + i) * H + h) * P + p] = from_f32<IO>(0.f);
        }
        return;
    }
    const float Ah = A[h];
    const float Dh = D ? D[h] : 0.f;   // (d_pc: D[h][p] per output column below)
    for (int i = tid; i < T; i += 256) dtv[i] = dt_eff(dtx, dt[((size_t)b * T + i) * H + h], h);
    __syncthreads();
    // tree segsum Λ_i = Σ_{j∈path(i)} dt_j A_h   (A_tree = L A_log)
    for (int i = tid; i < T; i += 256) {
        float s = 0.f;
        for (int w = 0; w < W; ++w) {
            uint32_t bits = rows[i * W + w];
            while (bits) {
                int j = (w << 5) + __ffs(bits) - 1;
                bits &= bits - 1;
                s += dtv[j] * Ah;
            }
        }
        lam[i] = s;
    }
    __syncthreads();

    // row tiles are spread over blockIdx.z (one 64-node tile of rows per CTA) so that a single tree still
    // fills the machine; every CTA rebuilds the (cheap) tree prologue
    for (int pc = 0; pc < P; pc += kTile) {
        for (int rc = blockIdx.z * kTile; rc < T; rc += kTile * gridDim.z) {
            const int jmax = min(T, rc + kTile);   // columns j <= i < rc + 64
            float acc[4][4];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[r][c] = 0.f;
            // ---- carry-in Y0 = C · h0_hᵀ over N chunks ----
            if (h0) {
                for (int nc = 0; nc < N; nc += kTile) {
                    for (int k = tid; k < kTile * kTile; k += 256) {
                        int rr = k / kTile, nn = k % kTile;
                        int i = rc + rr, n = nc + nn, p = pc + rr;
                        CsT[nn * kPitch + rr] =
                            (i < T && n < N) ? to_f32(Cm[(((size_t)b * T + i) * G + g) * N + n]) : 0.f;
                        HsT[nn * kPitch + rr] =
                            (p < P && n < N) ? h0[(((size_t)b * H + h) * P + p) * N + n] : 0.f;
                    }
                    __syncthreads();
#pragma unroll 8
                    for (int nn = 0; nn < kTile; ++nn) {
                        float4 a = *reinterpret_cast<const float4*>(&CsT[nn * kPitch + ty * 4]);
                        float4 bb = *reinterpret_cast<const float4*>(&HsT[nn * kPitch + tx * 4]);
                        float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
                        for (int r = 0; r < 4; ++r)
#pragma unroll
                            for (int c = 0; c < 4; ++c) acc[r][c] = fmaf(av[r], bv[c], acc[r][c]);
                    }
                    __syncthreads();
                }
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    int i = rc + ty * 4 + r;
                    float e = (i < T) ? expf(lam[i]) : 0.f;
#pragma unroll
                    for (int c = 0; c < 4; ++c) acc[r][c] *= e;
                }
            }
            // ---- decay-masked weights M[i][j] = L_ij e^{Λ_i-Λ_j} dt_j (C_i·B_j) ----
            // G = C·Bᵀ for this row tile, 64 x 64 register-tiled over N chunks staged in shared memory
            // (the same pattern as Y0; CsT holds C chunk [n][row], HsT is reused for B chunk [n][j])
            for (int jc = 0; jc < jmax; jc += kTile) {
                float gacc[4][4];
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int c = 0; c < 4; ++c) gacc[r][c] = 0.f;
                for (int nc = 0; nc < N; nc += kTile) {
                    __syncthreads();
                    for (int k = tid; k < kTile * kTile; k += 256) {
                        int rr = k / kTile, nn = k % kTile;
                        int i = rc + rr, j = jc + rr, n = nc + nn;
                        CsT[nn * kPitch + rr] =
                            (i < T && n < N) ? to_f32(Cm[(((size_t)b * T + i) * G + g) * N + n]) : 0.f;
                        HsT[nn * kPitch + rr] =
                            (j < jmax && n < N) ? to_f32(Bm[(((size_t)b * T + j) * G + g) * N + n]) : 0.f;
                    }
                    __syncthreads();
#pragma unroll 8
                    for (int nn = 0; nn < kTile; ++nn) {
                        float4 a = *reinterpret_cast<const float4*>(&CsT[nn * kPitch + ty * 4]);
                        float4 bb = *reinterpret_cast<const float4*>(&HsT[nn * kPitch + tx * 4]);
                        float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
                        for (int r = 0; r < 4; ++r)
#pragma unroll
                            for (int c = 0; c < 4; ++c) gacc[r][c] = fmaf(av[r], bv[c], gacc[r][c]);
                    }
                }
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int rr = ty * 4 + r, i = rc + rr;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const int j = jc + tx * 4 + c;
                        if (j < jmax) {
                            float w = 0.f;
                            if (i < T && mask_bit(rows, W, i, j))
                                w = expf(fminf(lam[i] - lam[j], 0.f)) * dtv[j] * gacc[r][c];
                            Ms[rr * mp + j] = w;
                        }
                    }
                }
            }
            for (int k = tid; k < jmax * kTile; k += 256) {
                int j = k / kTile, pp = k % kTile, p = pc + pp;
                Xs[j * kPitch + pp] = (p < P) ? to_f32(x[(((size_t)b * T + j) * H + h) * P + p]) : 0.f;
            }
            __syncthreads();
            // ---- masked contraction Y += M · X_h (PAPER.md:96 M_u u) ----
            for (int j = 0; j < jmax; ++j) {
                float4 xv = *reinterpret_cast<const float4*>(&Xs[j * kPitch + tx * 4]);
                float xa[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    float m = Ms[(ty * 4 + r) * mp + j];
#pragma unroll
                    for (int c = 0; c < 4; ++c) acc[r][c] = fmaf(m, xa[c], acc[r][c]);
                }
            }
            // ---- epilogue: + D_h x_i, store ----
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                int i = rc + ty * 4 + r;
                if (i >= T) continue;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    int p = pc + tx * 4 + c;
                    if (p < P) {
                        const float dd = d_pc ? (D ? D[(size_t)h * P + p] : 0.f) : Dh;
                        float v = acc[r][c] + dd * Xs[i * kPitch + tx * 4 + c];
                        y[(((size_t)b * T + i) * H + h) * P + p] = from_f32<IO>(v);
                    }
                }
            }
            __syncthreads();
        }
    }
}

}  // namespace stree

extern "C" size_t stree_simt_smem_bytes(int T) { return stree::SimtSmem(T).total; }

extern "C" int stree_launch_scan_simt(const stree_dims* d, const void* x, const float* dt, const float* A,
                                      const void* Bm, const void* Cm, const float* D, const float* h0,
                                      const int32_t* parent, void* y, int32_t* dev_status, cudaStream_t s) {
    const int T = d->n_nodes;
    size_t smem = stree::SimtSmem(T).total;
    dim3 grid(d->n_heads, d->batch, (T + stree::kTile - 1) / stree::kTile);
    cudaError_t e;
    if (d->io_dtype == STREE_BF16) {
        auto k = stree::scan_simt_kernel<__nv_bfloat16>;
        e = stree::host::smem_attr((const void*)k, (int)smem);
        if (e != cudaSuccess) return (int)e;
        e = stree::launch_k(k, grid, dim3(256), smem, s, T, d->n_heads, d->head_dim, d->d_state, d->n_groups,
                            (const __nv_bfloat16*)x, dt, A, (const __nv_bfloat16*)Bm, (const __nv_bfloat16*)Cm, D, h0,
                            parent, (__nv_bfloat16*)y, dev_status, stree::DtX::from(stree_scan_opts_get()),
                            (stree_scan_opts_get() && stree_scan_opts_get()->d_per_channel) ? 1 : 0);
        if (e != cudaSuccess) return (int)e;
    } else {
        auto k = stree::scan_simt_kernel<float>;
        e = stree::host::smem_attr((const void*)k, (int)smem);
        if (e != cudaSuccess) return (int)e;
        e = stree::launch_k(k, grid, dim3(256), smem, s, T, d->n_heads, d->head_dim, d->d_state, d->n_groups,
                            (const float*)x, dt, A, (const float*)Bm, (const float*)Cm, D, h0, parent, (float*)y,
                            dev_status, stree::DtX::from(stree_scan_opts_get()),
                            (stree_scan_opts_get() && stree_scan_opts_get()->d_per_channel) ? 1 : 0);
        if (e != cudaSuccess) return (int)e;
    }
    return (int)cudaGetLastError();
}
